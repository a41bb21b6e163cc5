#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list and a full capture of the top kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
STEPS=${STEPS:-10}
if [ "${TESTS:-1}" = "1" ]; then echo "== pytest -m gpu"; timeout 900 python -m pytest tests -q -m gpu --tb=line 2>&1 | tail -25; fi
if [ "${TESTS:-1}" = "1" ]; then echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3; fi
echo "== bench"; timeout 900 python bench.py --steps $STEPS --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
if [ "${NCU:-1}" = "1" ]; then
echo "== ncu launches"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo rc=$?
echo "== ncu full"; timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_force|k_density|k_gradient|k_lists|k_bank" -s 5 -c 5 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo rc=$?
fi
ls -la gpurun_out
