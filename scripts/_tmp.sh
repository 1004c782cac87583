timeout 900 python -m pytest tests/test_gpu_filter.py tests/test_gpu_errors.py tests/test_gpu_cpp_shim.py tests/test_gpu_driver_verbatim.py -x -q 2>&1 | tail -5
timeout 300 python bench.py --no-cpu-baseline --no-widened > gpurun_out/bench_c2_zc.json 2> gpurun_out/bench_c2_zc.err
FKB_RUN_MAPPED=0 timeout 300 python bench.py --no-cpu-baseline --no-widened > gpurun_out/bench_c2_nozc.json 2> gpurun_out/bench_c2_nozc.err
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-widened --steps 20 > gpurun_out/bench_c4_zc.json 2> gpurun_out/bench_c4_zc.err
for c in c2_zc c2_nozc c4_zc; do python -c "
import json
d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1])
print('$c', round(d['value']), 'e2e', round(d['e2e']['value']), 'us', round(d['ms_per_step']*1e3,1), 'lat_us', round(d['step_latency']['ms_per_step']*1e3,1), d['roofline']['kernel'], round(d['roofline']['frac'],3))
"; tail -2 gpurun_out/bench_$c.err; done
