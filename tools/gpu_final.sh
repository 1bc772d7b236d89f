# Round-end evidence: GPU tests, smoke, default bench, C1/C3 lines, reference arm, launch list.
set -x
mkdir -p gpurun_out
TAG=${1:-fin}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; echo "bench rc=$?"
for c in C1 C2 C3 C4 C5_i64 D; do timeout 300 python bench.py --config $c --steps 100 --no-cpu-baseline > gpurun_out/bench_${c}_$TAG.json 2>gpurun_out/bench_${c}_$TAG.err; echo "$c rc=$?"; done
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_$TAG.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'gace|fin_|probe|minmax|sample' -c 200 --csv --log-file gpurun_out/launches_C5_$TAG.csv $B > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu rc=$?"
