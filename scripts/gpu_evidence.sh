# Round evidence on one B200: the full GPU suite + smoke, bench lines (c2 with the CPU baseline
# and the widened rows, c3, c4, the reference arm), launch lists of one step per config and
# ncu --set full captures (scripts/gpu_ncu.sh).   bash scripts/gpu_evidence.sh TAG
set -x
tag=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c2_$tag.json 2> gpurun_out/bench_c2_$tag.err
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-widened > gpurun_out/bench_c3_$tag.json 2> gpurun_out/bench_c3_$tag.err
timeout 900 python bench.py --config c4 --no-cpu-baseline --no-widened --steps 20 > gpurun_out/bench_c4_$tag.json 2> gpurun_out/bench_c4_$tag.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
bash scripts/gpu_ncu.sh $tag > gpurun_out/ncu_run_$tag.log 2>&1
tail -3 gpurun_out/pytest_$tag.log; tail -2 gpurun_out/smoke_$tag.log
for c in c2 c3 c4; do python -c "
import json
d=json.loads(open('gpurun_out/bench_${c}_$tag.json').read().strip().splitlines()[-1])
print('$c', round(d['value']), 'e2e', round(d['e2e']['value']), 'per_call', round(d['e2e']['per_call']['value']), 'us', round(d['ms_per_step']*1e3,1), 'lat_us', round(d['step_latency']['ms_per_step']*1e3,1), d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks'])
"; done
cut -c1-400 gpurun_out/bench_ref_$tag.json
