timeout 900 python -m pytest tests/test_gpu_tdeig.py tests/test_gpu_ekf.py -x -q > gpurun_out/pytest_f11.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f11.log; tail -3 gpurun_out/pytest_f11.log
FKB_EKF_TRACE=1 FKB_TDEIG_TRACE=1 timeout 600 python scripts/profile.py fekf c2 3 > gpurun_out/fekf_f11.log 2>&1; tail -32 gpurun_out/fekf_f11.log
