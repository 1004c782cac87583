timeout 900 python -m pytest tests/test_gpu_filter.py -x -q > gpurun_out/pytest_f7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f7.log; tail -3 gpurun_out/pytest_f7.log
timeout 600 python bench.py > gpurun_out/bench_c2_f7.json 2> gpurun_out/bench_c2_f7.err; tail -2 gpurun_out/bench_c2_f7.err
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-widened > gpurun_out/bench_c3_f7.json 2> gpurun_out/bench_c3_f7.err; tail -2 gpurun_out/bench_c3_f7.err
timeout 900 python bench.py --config c4 --no-cpu-baseline --no-widened --steps 20 > gpurun_out/bench_c4_f7.json 2> gpurun_out/bench_c4_f7.err; tail -2 gpurun_out/bench_c4_f7.err
for c in c2 c3 c4; do python -c "
import json
d=json.loads(open('gpurun_out/bench_${c}_f7.json').read().strip().splitlines()[-1])
print('$c', round(d['value']), 'e2e', round(d['e2e']['value']), 'per_call', round(d['e2e']['per_call']['value']), 'us', round(d['ms_per_step']*1e3,1), d['roofline']['kernel'], round(d['roofline']['frac'],3))
"; done
F="--set full --clock-control none --import-source on --profile-from-start off"
timeout 300 python scripts/profile.py step c3 > gpurun_out/prof_c3.log 2>&1 && timeout 600 ncu $F -k regex:"k_mean_uq|k_cap_pcg|k_coldot" -o gpurun_out/step_c3_f7 -f python scripts/profile.py step c3 > gpurun_out/ncu_c3.log 2>&1
python scripts/ncu_summary.py gpurun_out/step_c3_f7.ncu-rep step_c3_f7 > gpurun_out/ncu_step_c3_f7.txt 2>&1
FKB_EKF_TRACE=1 timeout 600 python scripts/profile.py fekf c2 3 > gpurun_out/fekf_trace.log 2>&1; tail -60 gpurun_out/fekf_trace.log
