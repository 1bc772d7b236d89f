#!/bin/bash
# design-exploration driver: microbench + ablation runs of the full-size C5 probe
./build/microbench
for ab in 0 1 8 2 6 14 15; do
  echo "== GACE_ABLATE=$ab"
  GACE_ABLATE=$ab python tools/ablate.py ${1:-C5} 2>&1 | grep -E "hll only|preds only|preds \+ pairs|all  "
done
