#!/bin/bash
# C5 (or $CFG) bench line under design switches (env assignments per variant), one after the other:
#   tools/variants.sh "label|ENV=VAL ENV2=VAL" ...   -> gpurun_out/var_<label>.json
mkdir -p gpurun_out
cfg=${CFG:-C5}
for v in "$@"; do
  label=${v%%|*}; envs=${v#*|}
  env $envs python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --cold-batches 0 \
      > gpurun_out/var_${cfg}_$label.json 2> gpurun_out/var_${cfg}_$label.err
  python - "$label" "gpurun_out/var_${cfg}_$label.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"{sys.argv[1]:24s} scan {d['stages_ms']['scan_ms']:.4f} ms  step {d['ms_per_step']:.4f}  frac {d['roofline']['frac']:.3f}  clk {d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
