#!/bin/bash
# One gpurun call: ncu launch list of a short bench run and one `ncu --set full` capture of the
# kernels matching $KERNELS (default: the loop kernels).  Scratch output in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-prof}
KERNELS=${KERNELS:-"^k_force$|^k_density$|^k_gradient$|^k_lists$|^k_bank$"}
WL=${WL:-}
if [ "${LAUNCHES:-1}" = "1" ]; then echo "== ncu launches"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline $WL > gpurun_out/ncu_bench_$TAG.log 2>&1; echo rc=$?; fi
echo "== ncu full"; timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$KERNELS" -s ${SKIP:-5} -c ${COUNT:-5} -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline $WL > gpurun_out/ncu_full_$TAG.log 2>&1; echo rc=$?
ls -la gpurun_out
