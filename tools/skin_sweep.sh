#!/bin/bash
# C4 step time vs the list skin (bench.py --skin): the loop cost of a larger skin, which list reuse
# over several steps would need.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for S in ${SKINS:-0.05 0.1 0.15 0.2}; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --skin $S > gpurun_out/skin_$S.json 2> gpurun_out/skin_$S.err
  python tools/bench_line.py gpurun_out/skin_$S.json "skin $S"
done
