timeout 900 python -m pytest tests/test_gpu_filter.py -x -q > gpurun_out/pytest_f9.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f9.log; tail -3 gpurun_out/pytest_f9.log
FKB_RUN_TRACE=1 timeout 300 python bench.py --no-cpu-baseline --no-widened > gpurun_out/bench_c2_f9.json 2> gpurun_out/bench_c2_f9.err; grep "\[run\]" gpurun_out/bench_c2_f9.err | tail -4
FKB_RUN_TRACE=1 timeout 300 python bench.py --config c3 --no-cpu-baseline --no-widened > gpurun_out/bench_c3_f9.json 2> gpurun_out/bench_c3_f9.err; grep "\[run\]" gpurun_out/bench_c3_f9.err | tail -4
FKB_RUN_TRACE=1 timeout 600 python bench.py --config c4 --no-cpu-baseline --no-widened --steps 10 > gpurun_out/bench_c4_f9.json 2> gpurun_out/bench_c4_f9.err; grep "\[run\]" gpurun_out/bench_c4_f9.err | tail -4
for c in c2 c3 c4; do python -c "
import json
d=json.loads(open('gpurun_out/bench_${c}_f9.json').read().strip().splitlines()[-1])
print('$c', round(d['value']), 'e2e', round(d['e2e']['value']), 'per_call', round(d['e2e']['per_call']['value']), 'us', round(d['ms_per_step']*1e3,1))
"; done
FKB_EKF_TRACE=1 FKB_TDEIG_TRACE=1 timeout 600 python scripts/profile.py fekf c2 2 > gpurun_out/fekf_tdeig.log 2>&1; grep -v "^\[ekf\]   ghep" gpurun_out/fekf_tdeig.log | tail -24
FKB_CORE_EIG=jacobi FKB_EKF_TRACE=1 timeout 600 python scripts/profile.py fekf c2 2 > gpurun_out/fekf_jac.log 2>&1; grep "eig\|fekf step" gpurun_out/fekf_jac.log | tail -8
