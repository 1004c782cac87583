FKB_UQ_SHAPE=9 timeout 900 python -m pytest tests/test_gpu_filter.py -x -q -k "uq or c3" > gpurun_out/pytest_f16.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f16.log; tail -3 gpurun_out/pytest_f16.log
bash scripts/env_sweep.sh f16 c3 "FKB_UQ_SHAPE=0" "FKB_UQ_SHAPE=9" "FKB_UQ_SHAPE=0" "FKB_UQ_SHAPE=9"
timeout 1500 python scripts/parity_full.py --out gpurun_out/parity_r02.json > gpurun_out/parity_f16.log 2>&1; tail -8 gpurun_out/parity_f16.log
