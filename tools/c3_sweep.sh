# C3 scan time by load-pipelining variant (GACE_JIT_DEFS design switches)
for d in "" "GACE_L2_PREFETCH_U=1" "GACE_PREFETCH=1" "GACE_PREFETCH=1,GACE_L2_PREFETCH_U=1"; do
  r=$(GACE_JIT_DEFS="$d" python bench.py --config C3 --steps 50 --warmup 3 --no-cpu-baseline --no-e2e --cold-batches 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('scan %.4f step %.4f' % (d['stages_ms']['scan_ms'], d['ms_per_step']))")
  echo "C3 defs=[$d] $r"
done
