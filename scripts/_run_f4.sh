timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_f4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f4.log; tail -3 gpurun_out/pytest_f4.log
bash scripts/env_sweep.sh f4c3 c3 "FKB_UQ_SHAPE=116" "FKB_UQ_SHAPE=208"
for qu in 0 216 208 232 408 508 504; do FKB_SPMM_QU=$qu timeout 300 python scripts/spmm_time.py c2 2>&1 | tail -1; done
timeout 300 python scripts/spmm_time.py c4 2>&1 | tail -1
