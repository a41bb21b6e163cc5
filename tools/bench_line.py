"""One-line summary of a bench.py JSON line: ms/step, interactions/s, per-phase ms (launches)."""
import json
import sys

try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2] if len(sys.argv) > 2 else sys.argv[1], round(d["ms_per_step"], 2), "%.4g" % d["value"],
          {k: (round(v["ms_per_step"], 2), v["launches_per_step"]) for k, v in d["kernels"].items()},
          "passes", d["config"]["density_passes_mean"], "regrids", d["config"]["density_regrids_mean"])
except Exception as e:  # noqa: BLE001
    print(sys.argv[1], "no bench line:", e)
