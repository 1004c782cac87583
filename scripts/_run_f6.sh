for qu in 0 1008 1016 2008 2016 5004 5008; do FKB_SPMM_QU=$qu timeout 300 python scripts/spmm_time.py c2 2>&1 | tail -1; done
bash scripts/gpu_ncu.sh r2 > gpurun_out/ncu_run.log 2>&1; tail -45 gpurun_out/ncu_run.log
