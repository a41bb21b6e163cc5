#!/bin/bash
# A/B timing of in-tree library variants (SPH_LIB): one short C4 bench per variant, ms per step
# and per-kernel ms.  LIBS="base f256 ..." names paper_2505_14538_b200/libsph_<v>.so ("" = libsph.so).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for v in ${LIBS}; do
  lib=paper_2505_14538_b200/libsph_$v.so; [ "$v" = "main" ] && lib=paper_2505_14538_b200/libsph.so
  SPH_LIB=$PWD/$lib timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
    print(v, "ms/step", round(d["ms_per_step"], 3), {k: round(x["ms_per_step"], 3) for k, x in d["kernels"].items()}, "frac", round(d["roofline"]["frac"], 4))
except Exception as e:
    print(v, "FAILED", e, open(f"gpurun_out/ab_{v}.err").read()[-800:])
PY
done
