# Round-2 GPU check: full GPU suite + smoke, bench lines c2 (widened), c3, c4 and the reference arm.
#   bash scripts/gpu_r2.sh TAG
set -x
tag=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2_$tag.json 2> gpurun_out/bench_c2_$tag.err
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-widened > gpurun_out/bench_c3_$tag.json 2> gpurun_out/bench_c3_$tag.err
timeout 900 python bench.py --config c4 --no-cpu-baseline --no-widened --steps 20 > gpurun_out/bench_c4_$tag.json 2> gpurun_out/bench_c4_$tag.err
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
tail -3 gpurun_out/pytest_$tag.log; cat gpurun_out/smoke_$tag.log | tail -3
for c in c2 c3 c4; do cut -c1-400 gpurun_out/bench_${c}_$tag.json; tail -3 gpurun_out/bench_${c}_$tag.err; done
