#!/bin/bash
# Per-batch A/B of engine switches on the bench (run under gpurun): tools/ab_batches.sh "<B list>" "<env cfg>"...
bl=$1; shift
for B in $bl; do
  for cfg in "$@"; do
    env $cfg timeout 600 python bench.py --batch $B --no-offload-section --no-cpu-baseline --steps 6 > gpurun_out/ab.json 2>/dev/null
    python - "$B" "$cfg" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print("B", sys.argv[1], sys.argv[2], round(d["value"], 1), round(d["ms_per_step"], 2), round(d["tau"], 4), d["clocks"]["sm_mhz"], flush=True)
PY
  done
done
