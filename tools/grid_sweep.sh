# C1 (1M rows) probe time by grid size: GACE_ROWS_PER_CTA = minimum rows per CTA (0 = one CTA per SM)
for per in 0 8192 16384 32768 65536; do
  r=$(GACE_ROWS_PER_CTA=$per python bench.py --config C1 --steps 100 --warmup 3 --no-cpu-baseline --no-e2e --cold-batches 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']; print('step %.4f scan %.4f fin %.4f p50 %.4f' % (d['ms_per_step'], s['scan_ms'], s['finalize_ms'], d['latency_ms']['p50']))")
  echo "C1 rows_per_cta=$per $r"
done
