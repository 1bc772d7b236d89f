# C1 (latency config): generic vs specialised scan kernels, and the per-stage times
for m in "" 1; do
  r=$(GACE_JIT_MIN_ROWS=$m python bench.py --config C1 --steps 200 --warmup 3 --no-cpu-baseline --no-e2e --cold-batches 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']; print('kernel %s step %.4f scan %.4f fin %.4f p50 %.4f' % (d['roofline']['kernel'], d['ms_per_step'], s['scan_ms'], s['finalize_ms'], d['latency_ms']['p50']))")
  echo "C1 GACE_JIT_MIN_ROWS=[$m] $r"
done
