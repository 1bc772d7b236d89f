# L2 prefetch distance sweep (design experiment): scan time per config and distance.
mkdir -p gpurun_out
for c in C5 C5_i64 C4; do for d in 1 2 3 4 6; do
  GACE_JIT_DEFS=GACE_L2_PF_DIST=$d timeout 300 python bench.py --config $c --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/pf_${c}_$d.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/pf_${c}_$d.json').read().strip().splitlines()[-1]); print('$c', 'dist=$d', 'scan_ms=%.4f' % d['stages_ms']['scan_ms'], 'frac=%.3f' % d['roofline']['frac'], d['clocks']['reasons'])"
done; done 2>&1 | tee gpurun_out/pf_sweep.txt
