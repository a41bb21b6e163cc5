#!/bin/bash
# Adaptive-grid configs (C3 Sedov, C5s clustered) at several wide margins (SPH_WIDE_MARGIN).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for M in ${MARGINS:-0 0.2}; do
  for W in C5s C3; do
    SPH_WIDE_MARGIN=$M timeout 600 python bench.py --workload $W --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/m_${W}_${M}.json 2> gpurun_out/m_${W}_${M}.err
    python tools/bench_line.py gpurun_out/m_${W}_${M}.json "$W margin $M"
  done
done
