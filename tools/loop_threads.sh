#!/bin/bash
# Tuning experiment: k_density / k_gradient block sizes (rebuilds libsph.so with -DSPH_DENS_T/-DSPH_GRAD_T).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for T in ${THREADS:-256 288 320}; do
  SPH_NVCC_EXTRA="-DSPH_DENS_T=$T -DSPH_GRAD_T=$T" python paper_2505_14538_b200/build.py --force > gpurun_out/build_$T.log 2>&1 || tail -3 gpurun_out/build_$T.log
  grep -A2 "k_densityENS\|k_gradientENS" paper_2505_14538_b200/ptxas.log | grep "Used\|spill" | tr '\n' ' '; echo
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 6 > gpurun_out/lt_$T.json 2> gpurun_out/lt_$T.err
  python tools/bench_line.py gpurun_out/lt_$T.json "loop threads $T"
done
