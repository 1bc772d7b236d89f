# design exploration on one GPU: smem microbenchmark + ablations of the full-size probe
mkdir -p gpurun_out build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/microbench tools/microbench.cu && ./build/microbench
for ab in 0 1 4 8 12 14; do
  echo "== GACE_ABLATE=$ab"
  GACE_ABLATE=$ab python tools/ablate.py ${1:-C5} 2>&1 | grep -E "nothing|hll only|preds only|preds \+ pairs|all  "
done
