#!/bin/bash
# Quick A/B under gpurun: GPU parity suite, then C4 and C2 headline bench lines (no sections).
mkdir -p gpurun_out
tag=${1:-ab}
[ -n "$NO_TESTS" ] || timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gputest.txt 2>&1
timeout 600 python bench.py --shape c4 --batch 32 --no-cpu-baseline --no-offload-section --steps 6 --e2e-tokens 8 \
  > gpurun_out/${tag}_c4.json 2> gpurun_out/${tag}_c4.err
timeout 600 python bench.py --no-cpu-baseline --no-offload-section --no-sections --steps 8 \
  > gpurun_out/${tag}_c2.json 2> gpurun_out/${tag}_c2.err
python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
for s in ("c4", "c2"):
    try:
        d = json.loads(open(f"gpurun_out/{t}_{s}.json").read().strip().splitlines()[-1])
        r = d["roofline"]
        print(s, round(d["value"], 1), "tok/s", round(d["ms_per_step"], 2), "ms/step tau", round(d["tau"], 3),
              "frac", round(r["frac"], 3), {k: round(v["hbm_frac"], 3) for k, v in r.get("by_pass", {}).items()},
              "e2e", round(d["e2e"]["value"], 1), d["clocks"])
    except Exception as ex:
        print(s, "failed", ex)
PY
