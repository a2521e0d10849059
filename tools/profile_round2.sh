#!/bin/bash
# Round-2 profile capture (run under gpurun): launch list of the default bench, ncu --set full of the
# persistent pass kernel in one draft pass and one verify pass of the bench configuration.
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  --no-offload-section > gpurun_out/ncu_launch_bench.log 2>&1
# bench --steps 1 --warmup 1: pass kernels 0-4 = warm-up step, 5-8 = draft passes, 9 = verify pass
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pass_tc --launch-skip 5 -c 1 \
  -o gpurun_out/pass_draft python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-offload-section \
  > gpurun_out/ncu_pass_draft.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pass_tc --launch-skip 9 -c 1 \
  -o gpurun_out/pass_verify python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-offload-section \
  > gpurun_out/ncu_pass_verify.log 2>&1
