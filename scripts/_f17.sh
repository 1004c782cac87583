timeout 1200 python -m pytest tests/test_gpu_filter.py tests/test_gpu_cpp_shim.py tests/test_gpu_driver_verbatim.py -x -q > gpurun_out/pytest_f17.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f17.log; tail -3 gpurun_out/pytest_f17.log
timeout 600 python scripts/parity_full.py --configs c1 --extra "" --out gpurun_out/parity_c1.json > gpurun_out/parity_c1.log 2>&1; python -c "
import json
d=json.load(open('gpurun_out/parity_c1.json'))
for r in d['runs']: print(r['config'], r['worst'], 'fallbacks', sum(bool(x) for x in r['cap_fallback']))
"
for c in c2 c3; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-widened > gpurun_out/bench_${c}_f17.json 2> gpurun_out/bench_${c}_f17.err; done
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-widened --steps 20 > gpurun_out/bench_c4_f17.json 2> gpurun_out/bench_c4_f17.err
for c in c2 c3 c4; do python -c "
import json
d=json.loads(open('gpurun_out/bench_${c}_f17.json').read().strip().splitlines()[-1])
print('$c', round(d['value']), 'e2e', round(d['e2e']['value']), 'us', round(d['ms_per_step']*1e3,1), d['roofline']['kernel'], round(d['roofline']['frac'],3), {k: round(v*1e3,1) for k,v in d['kernel_ms_in_graph'].items()})
"; done
