#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py (each tool in turn, logs to gpurun_out/)
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1 || exit 1
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 7 --print-limit 50 python tools/sanitize_cases.py > gpurun_out/san_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/san_$tool.log
done
