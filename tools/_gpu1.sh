timeout 1100 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest.log
tools/ab_env.sh 3 default SMOE_GATE_STAGE=0
bash tools/ab_c4.sh "SMOE_PDL=1"
