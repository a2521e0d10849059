#!/bin/bash
# A/B of engine switches / library variants on the default bench (run under gpurun):
#   tools/ab_env.sh <rounds> <variant>...   variant = "default" | "VAR=v[,VAR=v...]" | "lib:<path.so>[,VAR=v...]"
rounds=$1; shift
for i in $(seq 1 $rounds); do
  for v in "$@"; do
    (
      for kv in ${v//,/ }; do
        case $kv in
          default) ;;
          lib:*) export SMOE_LIB=${kv#lib:} ;;
          *) export "$kv" ;;
        esac
      done
      timeout 600 python bench.py --no-offload-section --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ab.json 2>/dev/null
    )
    python - "$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 2), round(d["tau"], 4), round(d["roofline"]["frac"], 3),
      round(d["e2e"]["value"], 1), d["clocks"]["sm_mhz"], flush=True)
PY
  done
done
