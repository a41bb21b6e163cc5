cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${WL:-C5s}.csv python bench.py --workload ${WL:-C5s} --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c5s.log 2>&1; echo rc=$?
python tools/launch_summary.py gpurun_out/launches_${WL:-C5s}.csv 25
SPH_DEBUG=1 timeout 300 python bench.py --workload ${WL:-C5s} --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep -i "wide\|sph rank" | tail -5
