#!/bin/bash
# compute-sanitizer over small-shape GPU tests of every kernel family (run under gpurun).
# usage: tools/sanitize.sh  -> gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
SEL="test_f32_forward_matches_reference or test_bf16_fine_grained_lossless or test_bf16_lossless_and_batch_invariant or test_tcgen05_matches_cuda_core_gemm or (test_expert_parallel_bitexact_bf16 and 2-)"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python -m pytest tests/test_engine_gpu.py -q -x -k "$SEL" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $? : $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
