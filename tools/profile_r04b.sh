#!/bin/bash
# Round-4 follow-up captures under gpurun (one GPU): ncu --set full of the row-group gate (k_gate_rg) of a
# C4 draft pass (T=32) and verify pass (T=160), and the launch list of the default C2 bench restricted to
# the speculative phases (NVTX range "smoe speculative phase"), so init kernels do not dilute the shares.
set -x
mkdir -p gpurun_out
C4="python bench.py --shape c4 --batch 32 --no-cpu-baseline --no-offload-section --no-sections --steps 1 --warmup 1 --e2e-tokens 2"
C2="python bench.py --no-cpu-baseline --no-offload-section --no-sections --steps 1 --warmup 1 --e2e-tokens 2"
N="ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:k_gate_rg -c 1"
timeout 900 $N --launch-skip 140 -o gpurun_out/r04_c4_gate_draft -f $C4 > gpurun_out/r04_ncu_c4_gate_draft.log 2>&1
timeout 900 $N --launch-skip 245 -o gpurun_out/r04_c4_gate_verify -f $C4 > gpurun_out/r04_ncu_c4_gate_verify.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "smoe speculative phase/" --metrics gpu__time_duration.sum --clock-control none \
  -c 1400 --csv --log-file gpurun_out/r04_launches_phases.csv $C2 > gpurun_out/r04_ncu_launch_phases.log 2>&1
