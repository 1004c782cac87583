timeout 600 python -m pytest tests/test_gpu_filter.py -x -q > gpurun_out/pytest_f3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f3.log; tail -3 gpurun_out/pytest_f3.log
FKB_FUSED_CHAIN=2 timeout 600 python -m pytest tests/test_gpu_filter.py -x -q -k "fused or unverified or singular or fallback or parity" > gpurun_out/pytest_f3b.log 2>&1; echo "pytest2 rc=$?" >> gpurun_out/pytest_f3b.log; tail -3 gpurun_out/pytest_f3b.log
bash scripts/env_sweep.sh f3 c2 "FKB_FUSED_CHAIN=1" "FKB_FUSED_CHAIN=2" "FKB_FUSED_CHAIN=0" "FKB_FUSED_CHAIN=1" "FKB_FUSED_CHAIN=2"
bash scripts/env_sweep.sh f3c3 c3 "FKB_UQ_ROWS=2" "FKB_UQ_ROWS=1" "FKB_UQ_ROWS=2 FKB_FUSED_CHAIN=2"
bash scripts/env_sweep.sh f3c4 c4 "FKB_FUSED_CHAIN=1" "FKB_FUSED_CHAIN=2"
