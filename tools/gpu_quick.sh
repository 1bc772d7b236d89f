# GPU tests + C5 bench (+ optional extra configs): bash tools/gpu_quick.sh [tag] [configs...]
set -x
TAG=${1:-q}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_$TAG.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gputests_$TAG.log
timeout 300 python bench.py --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_C5_$TAG.json 2> gpurun_out/bench_C5_$TAG.err; echo "bench rc=$?"
for c in "$@"; do timeout 300 python bench.py --config $c --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/bench_${c}_$TAG.json 2>gpurun_out/bench_${c}_$TAG.err; echo "$c rc=$?"; done
GACE_NO_T1=1 timeout 300 python bench.py --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/bench_C5_${TAG}_not1.json 2>&1
TAG=$TAG python - <<'PY'
import json,glob,os
for f in sorted(glob.glob('gpurun_out/bench_*_'+os.environ['TAG']+'*.json')):
    try:
        d=json.load(open(f)); print(f, 'scan_ms %.3f'%d['stages_ms']['scan_ms'], 'frac %.3f'%d['roofline']['frac'])
    except Exception as e: print(f, 'ERR', e)
PY
