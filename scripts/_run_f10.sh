timeout 900 python -m pytest tests/test_gpu_tdeig.py tests/test_gpu_ekf.py tests/test_gpu_filter.py -x -q > gpurun_out/pytest_f10.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f10.log; tail -3 gpurun_out/pytest_f10.log
for c in c2 c3; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-widened > gpurun_out/bench_${c}_f10.json 2> gpurun_out/bench_${c}_f10.err; done
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-widened --steps 20 > gpurun_out/bench_c4_f10.json 2> gpurun_out/bench_c4_f10.err
for c in c2 c3 c4; do python -c "
import json
d=json.loads(open('gpurun_out/bench_${c}_f10.json').read().strip().splitlines()[-1])
print('$c', round(d['value']), 'e2e', round(d['e2e']['value']), 'per_call', round(d['e2e']['per_call']['value']), 'us', round(d['ms_per_step']*1e3,1))
"; done
FKB_EKF_TRACE=1 FKB_TDEIG_TRACE=1 timeout 600 python scripts/profile.py fekf c2 3 > gpurun_out/fekf_f10.log 2>&1; grep -v "^\[ekf\]   ghep: [sg]" gpurun_out/fekf_f10.log | tail -26
