#!/bin/bash
# C4 (fine-grained E64 K6, B=32) split-K sweep: tools/ab_c4.sh "<env cfg>"...
for cfg in "$@"; do
  env $cfg timeout 600 python bench.py --shape c4 --batch 32 --no-offload-section --no-cpu-baseline --steps 6 --e2e-tokens 8 > gpurun_out/ab.json 2>/dev/null
  python - "$cfg" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 2), round(d["tau"], 4), round(d["roofline"]["frac"], 3), d["clocks"]["sm_mhz"], flush=True)
PY
done
