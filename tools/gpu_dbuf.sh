# Double-buffered accumulators: all GPU tests, smoke, C1/C3/C5 lines with and without.
set -x
mkdir -p gpurun_out
TAG=${1:-db1}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
for c in C1 C3; do
  GACE_NO_ACC_DBUF=1 timeout 300 python bench.py --config $c --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_memset_$TAG.json 2>/dev/null; echo "$c memset rc=$?"
  timeout 300 python bench.py --config $c --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_dbuf_$TAG.json 2>/dev/null; echo "$c dbuf rc=$?"
done
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; echo "bench rc=$?"
