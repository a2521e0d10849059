#!/bin/bash
# Round-4 profile captures under gpurun (one GPU): ncu --set full of the fused MoE launch
# (k_gemm_tc<SwiGLU, StoreF32>) at C2 gamma=4 (draft + verify), C2 gamma=8 (verify: the tensor-pipe case)
# and C4 (draft + verify), plus the launch list of the default bench step.  Launch indices count only the
# matching kernel: 32 per C2 pass (28 per C4 pass); --steps 1 --warmup 1.
set -x
mkdir -p gpurun_out
K='regex:k_gemm_tc<.int.3'
N="ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k $K -c 1"
C2="python bench.py --no-cpu-baseline --no-offload-section --no-sections --steps 1 --warmup 1 --e2e-tokens 2"
C4="python bench.py --shape c4 --batch 32 --no-cpu-baseline --no-offload-section --steps 1 --warmup 1 --e2e-tokens 2"
timeout 900 $N --launch-skip 165 -o gpurun_out/r04_c2_draft -f $C2 > gpurun_out/r04_ncu_c2_draft.log 2>&1
timeout 900 $N --launch-skip 293 -o gpurun_out/r04_c2_verify -f $C2 > gpurun_out/r04_ncu_c2_verify.log 2>&1
timeout 900 $N --launch-skip 549 -o gpurun_out/r04_c2g8_verify -f $C2 --gamma 8 > gpurun_out/r04_ncu_c2g8.log 2>&1
timeout 900 $N --launch-skip 145 -o gpurun_out/r04_c4_draft -f $C4 > gpurun_out/r04_ncu_c4_draft.log 2>&1
timeout 900 $N --launch-skip 257 -o gpurun_out/r04_c4_verify -f $C4 > gpurun_out/r04_ncu_c4_verify.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/r04_launches_default.csv $C2 > gpurun_out/r04_ncu_launch.log 2>&1
