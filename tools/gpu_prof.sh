# ncu evidence for one config: launch list of a short bench run + one --set full capture
# of the probe kernel.  Usage (under gpurun): bash tools/gpu_prof.sh C5 <tag>
set -x
C=${1:-C5}; TAG=${2:-r01}
mkdir -p gpurun_out
B="python bench.py --config $C --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'gace|fin_|probe|minmax|sample' -c 200 --csv \
    --log-file gpurun_out/launches_${C}_$TAG.csv $B > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
G="python tools/gpu_debug.py $C 0"
GACE_JIT_DUMP=gpurun_out/jit_${C}_$TAG.cubin $G > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:probe -c 1 \
    -o gpurun_out/prof_${C}_$TAG $G > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
