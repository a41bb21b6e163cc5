#!/bin/bash
# GPU tests (optional) + a short bench printing ms/step and per-kernel ms.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONUNBUFFERED=1
if [ "${TESTS:-1}" = "1" ]; then timeout 900 python -m pytest tests -q -m gpu -x --tb=short 2>&1 | tail -5; fi
timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/qb.json 2> gpurun_out/qb.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/qb.json").read().strip().splitlines()[-1])
print("ms/step", round(d["ms_per_step"], 3), "value", "%.4g" % d["value"], {k: round(v["ms_per_step"], 3) for k, v in d["kernels"].items()})
PY
