# Development round trip for the pipelined batch: filter tests, batch parity, bench lines.
#   bash scripts/gpu_piped.sh TAG
set -x
tag=${1:-dev}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_filter.py tests/test_gpu_errors.py tests/test_gpu_pcg.py -x -q > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
timeout 1500 python -m pytest tests/test_gpu_parity_full.py -q -k "pipelined or default_solver" > gpurun_out/parity_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/parity_$tag.log
timeout 300 python bench.py --no-cpu-baseline --no-widened > gpurun_out/bench_c2_$tag.json 2> gpurun_out/bench_c2_$tag.err
FKB_PIPED=0 timeout 300 python bench.py --no-cpu-baseline --no-widened > gpurun_out/bench_c2np_$tag.json 2> gpurun_out/bench_c2np_$tag.err
timeout 300 python bench.py --config c3 --no-cpu-baseline --no-widened > gpurun_out/bench_c3_$tag.json 2> gpurun_out/bench_c3_$tag.err
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-widened --steps 20 > gpurun_out/bench_c4_$tag.json 2> gpurun_out/bench_c4_$tag.err
tail -15 gpurun_out/pytest_$tag.log
tail -25 gpurun_out/parity_$tag.log
for c in c2 c2np c3 c4; do python -c "
import json,sys
try:
    d=json.loads(open('gpurun_out/bench_${c}_$tag.json').read().strip().splitlines()[-1])
    print('$c', round(d['value']), 'e2e', round(d['e2e']['value']), 'batch', d.get('device_batch') and round(d['device_batch']['value']), 'ms', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d.get('kernel_ms_in_graph',{}).items()})
except Exception as e: print('$c', 'ERR', e)
"; tail -2 gpurun_out/bench_${c}_$tag.err; done
