bash tools/sanitize.sh > gpurun_out/sanitize_summary.txt 2>&1
bash tools/ab_batches.sh "1 8 16 32 64" "SMOE_PDL=1" > gpurun_out/batches.txt 2>&1
bash tools/ab_c4.sh "SMOE_PDL=1" "SMOE_S_DOWN=2" "SMOE_PDL=1" "SMOE_S_DOWN=2" > gpurun_out/c4.txt 2>&1
cat gpurun_out/sanitize_summary.txt gpurun_out/batches.txt gpurun_out/c4.txt
