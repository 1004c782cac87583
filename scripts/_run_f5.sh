timeout 900 python -m pytest tests/test_gpu_filter.py -x -q > gpurun_out/pytest_f5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f5.log; tail -3 gpurun_out/pytest_f5.log
bash scripts/env_sweep.sh f5 c2 "FKB_PDL=0" "FKB_PDL=1" "FKB_PDL=2" "FKB_PDL=3" "FKB_PDL=0" "FKB_PDL=3"
bash scripts/env_sweep.sh f5c3 c3 "FKB_UQ_SHAPE=0" "FKB_UQ_SHAPE=208"
for qu in 0 216 208 232 408 504; do FKB_SPMM_QU=$qu timeout 300 python scripts/spmm_time.py c2 2>&1 | tail -1; done
timeout 300 python scripts/spmm_time.py c4 2>&1 | tail -1
