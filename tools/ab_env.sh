#!/bin/bash
# A/B of library variants / engine switches under gpurun: tools/ab_env.sh <shape c2|c4> "<label>|<env assignments>" ...
# Prints one summary line per config (tokens/s, ms/step, tau, expert-GEMM HBM fraction by pass, clocks).
shape=$1; shift
if [ "$shape" = c4 ]; then args="--shape c4 --batch 32"; else args=""; fi
for cfg in "$@"; do
  label=${cfg%%|*}; envs=${cfg#*|}
  env $envs timeout 600 python bench.py $args --no-cpu-baseline --no-offload-section --no-sections --steps 8 \
    --e2e-tokens 8 > gpurun_out/ab.json 2> gpurun_out/ab.err
  python - "$label" "$shape" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[2], sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 3), round(d["tau"], 4), round(r["frac"], 3),
          {k: round(v["hbm_frac"], 3) for k, v in r.get("by_pass", {}).items()}, d["clocks"]["sm_mhz"], flush=True)
except Exception as ex:
    print(sys.argv[2], sys.argv[1], "failed", ex, open("gpurun_out/ab.err").read()[-500:])
PY
done
