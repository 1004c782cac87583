# Round-end evidence on one B200: GPU tests, bench lines (c2, c3, c4, reference arm), the c2
# step launch list and ncu --set full captures of the top kernels.  Each ncu run follows a
# clean run of the same command.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-widened > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --config c4 --no-cpu-baseline --no-widened --steps 20 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python scripts/profile.py step c2 > /dev/null 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_c2.csv python scripts/profile.py step c2 > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_c2.csv > gpurun_out/launches_c2.txt 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_gemv_rowmajor \
    -o gpurun_out/step_gemv -f python scripts/profile.py step c2 > gpurun_out/ncu_gemv.log 2>&1
NE=1000 timeout 300 python scripts/profile.py enkf c2 > /dev/null 2>&1 && \
NE=1000 ncu --set full --clock-control none -k regex:k_samp_cols512 -s 1 -c 1 \
    -o gpurun_out/enkf_full -f python scripts/profile.py enkf c2 > gpurun_out/ncu_enkf.log 2>&1
for r in step_gemv enkf_full; do python scripts/ncu_summary.py gpurun_out/$r.ncu-rep $r > gpurun_out/$r.txt 2>&1; done
tail -2 gpurun_out/pytest_gpu.log
