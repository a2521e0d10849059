#!/bin/bash
# A/B of library variants on the default bench (run under gpurun): tools/ab_bench.sh <rounds> <lib|default>...
rounds=$1; shift
for i in $(seq 1 $rounds); do
  for v in "$@"; do
    if [ "$v" = default ]; then unset SMOE_LIB; else export SMOE_LIB=$v; fi
    timeout 600 python bench.py --no-offload-section --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    python - "$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 2), round(d["tau"], 4), round(d["roofline"]["frac"], 3),
      round(d["e2e"]["value"], 1), d["clocks"]["sm_mhz"], flush=True)
PY
  done
done
unset SMOE_LIB
