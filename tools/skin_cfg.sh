#!/bin/bash
# Step time of every config at two list skins.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for S in ${SKINS:-0.05 0.08}; do
  for W in ${WLS:-C4 C2 C3 C5s}; do
    timeout 600 python bench.py --workload $W --no-cpu-baseline --no-e2e --steps 5 --skin $S > gpurun_out/sk_${W}_$S.json 2> gpurun_out/sk_${W}_$S.err
    python tools/bench_line.py gpurun_out/sk_${W}_$S.json "$W skin $S"
  done
done
