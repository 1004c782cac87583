timeout 600 python -m pytest tests/test_gpu_filter.py -x -q -k "c2 or fused or run_" > gpurun_out/pytest_f13.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f13.log; tail -2 gpurun_out/pytest_f13.log
bash scripts/env_sweep.sh f13 c2 "FKB_UFORK=1" "FKB_UFORK=2" "FKB_UFORK=3" "FKB_UFORK=2 FKB_UPASS_CTAS=2" "FKB_UFORK=1" "FKB_UFORK=2"
