for cpc in 0 2 1; do
FKB_COLDOT_CPC=$cpc timeout 600 python bench.py --no-cpu-baseline --no-widened > gpurun_out/bench_c2_cpc$cpc.json 2> gpurun_out/bench_c2_cpc$cpc.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_c2_cpc$cpc.json').read().strip().splitlines()[-1])
print('c2 cpc$cpc', round(d['value']), 'e2e', round(d['e2e']['value']), 'us', round(d['ms_per_step']*1e3,1), 'lat', round(d['step_latency']['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['phases_ms_serial'].items()})
"; tail -2 gpurun_out/bench_c2_cpc$cpc.err; done
FKB_COLDOT_CPC=2 timeout 600 python bench.py --config c4 --no-cpu-baseline --no-widened --steps 20 > gpurun_out/bench_c4_cpc2.json 2> gpurun_out/bench_c4_cpc2.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_c4_cpc2.json').read().strip().splitlines()[-1])
print('c4 cpc2', round(d['value']), 'e2e', round(d['e2e']['value']), 'us', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['phases_ms_serial'].items()})
"
for cpc in 0 2; do
FKB_COLDOT_CPC=$cpc timeout 600 python bench.py --config c3 --no-cpu-baseline --no-widened > gpurun_out/bench_c3_cpc$cpc.json 2> gpurun_out/bench_c3_cpc$cpc.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_c3_cpc$cpc.json').read().strip().splitlines()[-1])
print('c3 cpc$cpc', round(d['value']), 'e2e', round(d['e2e']['value']), 'us', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['phases_ms_serial'].items()})
"; done
