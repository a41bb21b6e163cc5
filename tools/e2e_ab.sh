#!/bin/bash
# e2e (pipelined host I/O) ms per step, three runs each with uploads on the copy engines and by kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for mode in ce kernel ce kernel; do
  if [ $mode = ce ]; then export SPH_H2D_CE=1; else unset SPH_H2D_CE; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_ab.json 2>/dev/null
  python - $mode <<'PY'
import json, sys
d = json.loads(open("gpurun_out/e2e_ab.json").read().strip().splitlines()[-1])
print(sys.argv[1], round(d["ms_per_step"], 3), round(d["e2e"]["ms_per_step"], 3), d["e2e"]["device_ms_per_step"])
PY
done
