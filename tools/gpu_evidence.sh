# Round evidence on one GPU: GPU tests, smoke, the default bench line, every config's bench
# line, the reference arm, and an ncu launch list of the default bench command.
set -x
mkdir -p gpurun_out
TAG=${1:-ev}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_$TAG.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; echo "bench rc=$?"
for c in C1 C2 C3 C3B C4 C5_i64 D D_m1_k16; do timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline > gpurun_out/bench_${c}_$TAG.json 2>gpurun_out/bench_${c}_$TAG.err; echo "$c rc=$?"; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1; echo "ref rc=$?"
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_$TAG.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'gace|fin_|probe|minmax|sample' -c 200 --csv --log-file gpurun_out/launches_C5_$TAG.csv $B > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu rc=$?"
G="python tools/gpu_debug.py C5 0"
GACE_JIT_DUMP=gpurun_out/jit_C5_$TAG.cubin $G > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:probe -c 1 -o gpurun_out/prof_C5_$TAG $G > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
bash tools/gpu_prof_sets.sh
