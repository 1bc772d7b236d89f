# Zero-copy result write: all GPU tests, smoke, then C1/C3/C5 bench lines with and without it.
set -x
mkdir -p gpurun_out
TAG=${1:-zc1}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log
for c in C1 C3; do
  GACE_NO_ZERO_COPY=1 timeout 300 python bench.py --config $c --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_copy_$TAG.json 2>gpurun_out/bench_${c}_copy_$TAG.err; echo "$c copy rc=$?"
  timeout 300 python bench.py --config $c --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_zc_$TAG.json 2>gpurun_out/bench_${c}_zc_$TAG.err; echo "$c zc rc=$?"
  timeout 300 python bench.py --config $c --steps 200 --no-cpu-baseline --no-e2e --graphs > gpurun_out/bench_${c}_zcg_$TAG.json 2>gpurun_out/bench_${c}_zcg_$TAG.err; echo "$c zc+graphs rc=$?"
done
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; echo "bench rc=$?"
