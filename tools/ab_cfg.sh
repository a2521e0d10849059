#!/bin/bash
# A/B of engine switches on several bench configs (run under gpurun):
#   tools/ab_cfg.sh "<cfg args>|<cfg args>..." "<env>" "<env>"...
# cfg args are bench.py arguments; "-" as env = defaults.  Prints one line per (cfg, env).
IFS='|' read -ra CFGS <<< "$1"; shift
for cfg in "${CFGS[@]}"; do
  for v in "$@"; do
    e=""; [ "$v" != "-" ] && e="$v"
    env $e timeout 600 python bench.py $cfg --no-sections --no-offload-section --no-cpu-baseline --e2e-tokens 4 \
      > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python - "$cfg" "$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
bp = d["roofline"]["by_pass"]
print(f"{sys.argv[1]:<34} {sys.argv[2]:<40} tok/s {d['value']:8.1f} ms {d['ms_per_step']:7.2f} tau {d['tau']:.3f} "
      f"draft {bp['draft']['hbm_frac']:.3f} verify {bp['verify']['hbm_frac']:.3f}/{bp['verify']['tensor_frac']:.3f} "
      f"e2e {(d.get('e2e') or {}).get('value')} mhz {(d.get('clocks') or {}).get('sm_mhz')}", flush=True)
PY
  done
done
