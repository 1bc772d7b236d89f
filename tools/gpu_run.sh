set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "bench rc=$?"
cat gpurun_out/bench_C5.json
for c in C1 C2 C3 C4; do timeout 300 python bench.py --config $c --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; echo "$c rc=$?"; cat gpurun_out/bench_$c.json; done
