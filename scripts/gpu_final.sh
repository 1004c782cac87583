# Final evidence run on one B200: full GPU suite + smoke, bench lines (c2 with widened paths,
# c3 fused UQ, c4, reference arm), the c2 step launch list and an ncu --set full of the U pass.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
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
python scripts/ncu_summary.py gpurun_out/step_gemv.ncu-rep step_gemv > gpurun_out/step_gemv.txt 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
