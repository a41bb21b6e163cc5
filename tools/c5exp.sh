cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for DI in 6 1; do
  for W in C5s C3 C4; do
    SPH_DENS_INNER=$DI timeout 600 python bench.py --workload $W --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/x_${W}_${DI}.json 2>/dev/null
    python - "$W" "$DI" gpurun_out/x_${W}_${DI}.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
print(sys.argv[1], "inner", sys.argv[2], round(d["ms_per_step"], 2), {k: (round(v["ms_per_step"], 2), v["launches_per_step"]) for k, v in d["kernels"].items()}, d["config"]["density_passes_mean"])
PY
  done
done
