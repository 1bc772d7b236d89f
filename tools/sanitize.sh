#!/bin/bash
# compute-sanitizer evidence for the probe (one tool per gpurun call, per the
# B200 profiling recipe).  Usage, on the GPU box:  tools/sanitize.sh <memcheck|racecheck|synccheck|initcheck>
# Runs the tool over small probes -- C1 at 200,003 rows and C5 at 4,000,003 rows, each sampled
# and unsampled, with the generic kernel (GACE_JIT=0) and the plan-specialised ones (GACE_JIT=1:
# structure-keyed, then layout-keyed after tools/profile_probe.py's jit_sync) -- and writes
# gpurun_out/sanitize_<tool>.log.  Exit code: the tool's (nonzero on any reported error).
set -u
tool=${1:-memcheck}
out=gpurun_out/sanitize_${tool}.log
mkdir -p gpurun_out
extra=""
case $tool in
  memcheck) extra="--leak-check full" ;;
  racecheck) extra="--racecheck-report hazard" ;;
esac
rc=0
: > "$out"
for args in "--config C1 --rows 200003 --probes 3" "--config C1 --rows 200003 --probes 3 --rate 0.05" \
            "--config C5 --rows 4000003 --probes 3" "--config C5 --rows 4000003 --probes 3 --rate 0.01"; do
  for jit in 0 1; do        # generic kernel; plan-specialised kernels (structure, then layout)
    echo "=== GACE_JIT=$jit compute-sanitizer --tool $tool $extra python tools/profile_probe.py $args" >> "$out"
    GACE_JIT=$jit timeout 1200 compute-sanitizer --tool "$tool" $extra --error-exitcode 9 \
        python tools/profile_probe.py $args >> "$out" 2>&1
    r=$?
    echo "=== exit $r" >> "$out"
    [ $r -ne 0 ] && rc=$r
  done
done
exit $rc
