# scan time of the specialised kernel by CTA size (GACE_JIT_THREADS: 1024 / 768 / 512)
for c in C4 C5 C5_i64; do for th in 1024 768 512; do
  r=$(GACE_JIT_THREADS=$th python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --cold-batches 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('scan %.4f step %.4f %s' % (d['stages_ms']['scan_ms'], d['ms_per_step'], d['roofline']['kernel']))")
  echo "$c threads=$th $r"
done; done
