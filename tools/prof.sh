#!/bin/bash
# One short bench run with grid debug output, then an ncu --set full capture of the loop kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
SPH_DEBUG=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep "sph rank" | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_force|k_density|k_gradient|k_lists}" -s ${SKIP:-4} -c ${COUNT:-4} -o gpurun_out/prof_${TAG:-x} python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${TAG:-x}.log 2>&1; echo ncu rc=$?
python tools/ncu_summary.py gpurun_out/prof_${TAG:-x}.ncu-rep
