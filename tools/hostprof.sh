SMOE_HOST_PROF=1 timeout 300 python bench.py --shape c4 --batch 32 --no-cpu-baseline --no-offload-section --steps 3 --warmup 2 --e2e-tokens 4 > gpurun_out/c4_hostprof.json 2> gpurun_out/c4_hostprof.err
SMOE_HOST_PROF=1 timeout 300 python bench.py --no-cpu-baseline --no-offload-section --no-sections --steps 3 --warmup 2 --e2e-tokens 4 > gpurun_out/c2_hostprof.json 2> gpurun_out/c2_hostprof.err
