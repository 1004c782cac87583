# c2 bench lines (device value, e2e, in-graph phases) under environment variants.
#   bash scripts/env_sweep.sh TAG CONFIG "VAR=a VAR2=b" "VAR=c" ...
tag=$1; cfg=$2; shift 2
mkdir -p gpurun_out
for v in "$@"; do
  env $v timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-widened > gpurun_out/sweep_$tag.json 2> gpurun_out/sweep_$tag.err
  python -c "
import json
try:
    d=json.loads(open('gpurun_out/sweep_$tag.json').read().strip().splitlines()[-1])
    print('$cfg [$v]', round(d['value']), 'e2e', round(d['e2e']['value']), 'us', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d.get('kernel_ms_in_graph',{}).items()}, flush=True)
except Exception as e: print('$v', 'ERR', e)
"
  tail -1 gpurun_out/sweep_$tag.err
done
