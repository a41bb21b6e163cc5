#!/bin/bash
# Adaptive-grid configs at several sparse-block thresholds (SPH_SPARSE_WIDE).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for K in ${KS:-0 8 16 32}; do
  for W in C5s C3; do
    SPH_SPARSE_WIDE=$K timeout 600 python bench.py --workload $W --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/sp_${W}_${K}.json 2> gpurun_out/sp_${W}_${K}.err
    python tools/bench_line.py gpurun_out/sp_${W}_${K}.json "$W sparse $K"
  done
done
