# Quick round trip for the pipelined batch: timeline, batch parity at c2/c3, bench c2.
set -x
tag=${1:-dev}
mkdir -p gpurun_out
timeout 300 python scripts/timeline.py c2 8 batch > gpurun_out/tl_$tag.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity_full.py -q -x -k "pipelined and (c0 or c2 or c1)" > gpurun_out/parity_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/parity_$tag.log
timeout 300 python bench.py --no-cpu-baseline --no-widened > gpurun_out/bench_c2_$tag.json 2> gpurun_out/bench_c2_$tag.err
FKB_EARLY_PCG=0 timeout 300 python bench.py --no-cpu-baseline --no-widened > gpurun_out/bench_c2ne_$tag.json 2> gpurun_out/bench_c2ne_$tag.err
tail -5 gpurun_out/parity_$tag.log
for c in c2 c2ne; do python -c "
import json,sys
try:
    d=json.loads(open('gpurun_out/bench_${c}_$tag.json').read().strip().splitlines()[-1])
    print('$c', round(d['value']), 'e2e', round(d['e2e']['value']), 'batch', d.get('device_batch') and round(d['device_batch']['value']), 'ms', round(d['ms_per_step']*1e3,1))
except Exception as e: print('$c', 'ERR', e)
"; tail -2 gpurun_out/bench_${c}_$tag.err; done
cat gpurun_out/tl_$tag.txt | tail -45
