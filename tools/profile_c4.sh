#!/bin/bash
# C4 (fine-grained E64 K6, B=32, N=8) profile capture under gpurun: bench line, launch list, ncu --set full of
# the fused MoE launch (k_gemm_tc<SwiGLU, StoreF32>) in one draft pass and one verify pass.
# bench --steps 1 --warmup 1: 28 k_gemm_tc<SwiGLU> launches per pass (the dense layer 0 up projection + 27 fused
# MoE layers); warm-up step = launches 0-139, timed step 140-279 (draft passes 140-251, verify 252-279).
# MoE layer 5 of the first timed draft pass / of the verify pass.
set -x
mkdir -p gpurun_out
B="python bench.py --shape c4 --batch 32 --no-cpu-baseline --no-offload-section --e2e-tokens 4"
[ -n "$SKIP_BENCH" ] || timeout 600 $B --steps 6 --warmup 3 > gpurun_out/c4_bench.json 2> gpurun_out/c4_bench.err
[ -n "$SKIP_BENCH" ] || timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv \
  --log-file gpurun_out/c4_launches.csv $B --steps 1 --warmup 1 > gpurun_out/c4_ncu_launch.log 2>&1
for spec in "draft 145" "verify 257"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_gemm_tc<.int.3" --launch-skip $2 -c 1 \
    -o gpurun_out/c4_moe_$1 -f $B --steps 1 --warmup 1 > gpurun_out/c4_ncu_$1.log 2>&1
done
