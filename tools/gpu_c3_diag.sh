# C3 (Zipf head) diagnosis: ablations of the full-size probe and one ncu --set full capture.
set -x
mkdir -p gpurun_out
for ab in 0 2 8 10; do
  echo "== GACE_ABLATE=$ab"
  GACE_ABLATE=$ab timeout 300 python tools/ablate.py C3 2>&1 | tail -8
done > gpurun_out/c3_ablate.log 2>&1
G="python tools/gpu_debug.py C3 0"
timeout 300 $G > gpurun_out/c3_plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:probe -c 1 -o gpurun_out/prof_C3 $G > gpurun_out/ncu_C3.log 2>&1
echo "full rc=$?"
