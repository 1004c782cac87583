timeout 600 python -m pytest tests/test_gpu_filter.py -x -q > gpurun_out/pytest_f2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f2.log; tail -3 gpurun_out/pytest_f2.log
bash scripts/env_sweep.sh f2 c2 "FKB_L2PF=0" "FKB_L2PF=1" "FKB_L2PF=2" "FKB_L2PF=3" "FKB_FUSED_CHAIN=0 FKB_L2PF=0" "FKB_L2PF=0"
bash scripts/env_sweep.sh f2c3 c3 "FKB_L2PF=0" "FKB_L2PF=3"
bash scripts/env_sweep.sh f2c4 c4 "FKB_L2PF=0" "FKB_L2PF=3"
