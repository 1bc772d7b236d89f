for c in C5 C5_i64; do for m in 2 13; do for pf in 1 0; do
  r=$(GACE_JIT_DEFS="GACE_L2_PREFETCH=$pf" GACE_ORIENT_MASK=$m python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --cold-batches 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f'%d['stages_ms']['scan_ms'])")
  echo "$c mask=$m l2pf=$pf scan_ms=$r"
done; done; done
for pf in 1 0; do r=$(GACE_JIT_DEFS="GACE_L2_PREFETCH=$pf" python bench.py --config C4 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --cold-batches 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f'%d['stages_ms']['scan_ms'])"); echo "C4 l2pf=$pf scan_ms=$r"; done
