# c2 bench line under a list of environment settings (one per argument, e.g. "FKB_FUSE_RHS=0")
mkdir -p gpurun_out
i=0
for spec in "$@"; do
  i=$((i+1))
  env $spec timeout 300 python bench.py --no-cpu-baseline --no-widened ${BENCH_ARGS:-} > gpurun_out/env_$i.json 2>gpurun_out/env_$i.err
  python - "$i" "$spec" <<'PY'
import json, sys
try:
    d = json.load(open(f"gpurun_out/env_{sys.argv[1]}.json"))
except Exception as e:
    print(sys.argv[2], "FAILED", e); sys.exit()
k = d["kernel_ms_in_graph"]
print(f"[{sys.argv[2]}]", round(d["value"]), round(d["e2e"]["value"]), " ".join(f"{a}={1e3*b:.1f}" for a, b in k.items()))
PY
done
