#!/bin/bash
# One gpurun call: the default bench line (C4), the other configs' lines (C2, C3, C5s), and the
# oracle on every config family (--cpu-baseline-all).  Output in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
TAG=${TAG:-all}
timeout 900 python bench.py > gpurun_out/bench_${TAG}_C4.json 2> gpurun_out/bench_${TAG}_C4.err; echo C4 rc=$?
for W in C2 C3 C5s; do
  timeout 600 python bench.py --workload $W --no-cpu-baseline > gpurun_out/bench_${TAG}_$W.json 2> gpurun_out/bench_${TAG}_$W.err; echo $W rc=$?
done
if [ "${CPU:-1}" = "1" ]; then timeout 1200 python bench.py --cpu-baseline-all gpurun_out/cpu_baseline_${TAG}.json > gpurun_out/cpu_${TAG}.log 2>&1; echo cpu rc=$?; fi
for f in gpurun_out/bench_${TAG}_*.json; do python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["config"]["workload"], round(d["ms_per_step"], 3), "%.4g" % d["value"], {k: round(v["ms_per_step"], 3) for k, v in d["kernels"].items()}, "frac", round(d["roofline"]["frac"], 4))
PY
done
