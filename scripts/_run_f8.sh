timeout 900 python -m pytest tests/test_gpu_filter.py -x -q -k "run_ or unverified" > gpurun_out/pytest_f8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f8.log; tail -3 gpurun_out/pytest_f8.log
python - <<'PY'
import torch, time
for mb in (0.5, 2, 8, 64):
    n = int(mb * 2**20 / 8)
    d = torch.randn(n, dtype=torch.float64, device="cuda"); h = torch.empty(n, dtype=torch.float64).pin_memory()
    for _ in range(3): h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [h.copy_(d, non_blocking=True) for _ in range(10)]; b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    a.record(); [d.copy_(h, non_blocking=True) for _ in range(10)]; b.record(); torch.cuda.synchronize()
    ms2 = a.elapsed_time(b) / 10
    print(f"pinned {mb} MB: D2H {mb * 2**20 / ms / 1e6:.1f} GB/s ({ms*1e3:.1f} us), H2D {mb * 2**20 / ms2 / 1e6:.1f} GB/s")
PY
FKB_RUN_TRACE=1 timeout 300 python bench.py --no-cpu-baseline --no-widened > gpurun_out/bench_c2_f8.json 2> gpurun_out/bench_c2_f8.err; grep "\[run\]" gpurun_out/bench_c2_f8.err | tail -8
FKB_RUN_TRACE=1 timeout 600 python bench.py --config c4 --no-cpu-baseline --no-widened --steps 10 > gpurun_out/bench_c4_f8.json 2> gpurun_out/bench_c4_f8.err; grep "\[run\]" gpurun_out/bench_c4_f8.err | tail -8
for c in c2 c4; do python -c "
import json
d=json.loads(open('gpurun_out/bench_${c}_f8.json').read().strip().splitlines()[-1])
print('$c', round(d['value']), 'e2e', round(d['e2e']['value']), 'per_call', round(d['e2e']['per_call']['value']), 'us', round(d['ms_per_step']*1e3,1))
"; done
timeout 300 python scripts/pcg_stamps.py c2 2>&1 | tail -4
