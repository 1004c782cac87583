# The pipelined batch (FKB_PIPED=1) against the default full step graphs: CUPTI timelines of an
# 8-step batch, batch parity, c2 bench lines.   bash scripts/gpu_piped.sh TAG
set -x
tag=${1:-dev}
mkdir -p gpurun_out
timeout 300 python scripts/timeline.py c2 8 batch > gpurun_out/tl_full_$tag.txt 2>&1
FKB_PIPED=1 timeout 300 python scripts/timeline.py c2 8 batch > gpurun_out/tl_piped_$tag.txt 2>&1
FKB_PIPED=1 FKB_EARLY_PCG=0 timeout 300 python scripts/timeline.py c2 8 batch > gpurun_out/tl_piped_late_pcg_$tag.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity_full.py -q -k "batch" > gpurun_out/parity_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/parity_$tag.log
timeout 300 python bench.py --no-cpu-baseline --no-widened > gpurun_out/bench_c2_$tag.json 2> gpurun_out/bench_c2_$tag.err
FKB_PIPED=1 timeout 300 python bench.py --no-cpu-baseline --no-widened > gpurun_out/bench_c2piped_$tag.json 2> gpurun_out/bench_c2piped_$tag.err
tail -5 gpurun_out/parity_$tag.log
for c in c2 c2piped; do python -c "
import json
d=json.loads(open('gpurun_out/bench_${c}_$tag.json').read().strip().splitlines()[-1])
print('$c', round(d['value']), 'e2e', round(d['e2e']['value']), 'us', round(d['ms_per_step']*1e3,1), 'lat_us', round(d['step_latency']['ms_per_step']*1e3,1))
"; done
head -4 gpurun_out/tl_full_$tag.txt gpurun_out/tl_piped_$tag.txt gpurun_out/tl_piped_late_pcg_$tag.txt | grep batch
