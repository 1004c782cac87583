# GPU round-trip used during development: tests, a c2 bench line, optional extras.
#   bash scripts/gpu_check.sh [tag] [pytest-args...]
set -x
tag=${1:-dev}; shift || true
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -x -q -m gpu "$@" > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
timeout 600 python bench.py --no-cpu-baseline --no-widened > gpurun_out/bench_c2_$tag.json 2> gpurun_out/bench_c2_$tag.err
tail -3 gpurun_out/pytest_$tag.log; cut -c1-600 gpurun_out/bench_c2_$tag.json; tail -5 gpurun_out/bench_c2_$tag.err
