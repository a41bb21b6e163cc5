#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py (one gpurun call).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 3 --print-limit 20 python tools/sanitize_run.py \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?"
  tail -4 gpurun_out/sanitize_$tool.log
done
