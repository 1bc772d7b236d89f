# CUDA-graph replay: GPU tests, then C1/C3/C5 bench lines with and without --graphs.
set -x
mkdir -p gpurun_out
TAG=${1:-g1}
timeout 600 python -m pytest tests/test_gpu_graphs.py -x -q > gpurun_out/gputests_graphs_$TAG.log 2>&1; echo "graph tests rc=$?"; tail -3 gpurun_out/gputests_graphs_$TAG.log
for c in C1 C3 C5; do
  timeout 300 python bench.py --config $c --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_eager_$TAG.json 2>gpurun_out/bench_${c}_eager_$TAG.err; echo "$c eager rc=$?"
  timeout 300 python bench.py --config $c --steps 100 --no-cpu-baseline --no-e2e --graphs > gpurun_out/bench_${c}_graphs_$TAG.json 2>gpurun_out/bench_${c}_graphs_$TAG.err; echo "$c graphs rc=$?"
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_all_$TAG.log 2>&1; echo "all gpu tests rc=$?"; tail -2 gpurun_out/gputests_all_$TAG.log
