#!/bin/bash
# Round profile capture (run under gpurun): launch list of one default bench step, ncu --set full of the
# fused MoE GEMM in a draft pass and in a verify pass, then the timed bench line.
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv \
  --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  --no-offload-section > gpurun_out/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm_tc --launch-skip 1 -c 1 \
  -o gpurun_out/moe_draft python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-offload-section \
  > gpurun_out/ncu_moe_draft.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm_tc --launch-skip 261 -c 1 \
  -o gpurun_out/moe_verify python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-offload-section \
  > gpurun_out/ncu_moe_verify.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -c 3000 gpurun_out/bench_default.json
