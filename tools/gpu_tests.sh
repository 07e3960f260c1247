#!/bin/bash
# GPU-box session: the GPU test suite (optionally a -k filter) + smoke
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
K=${1:-}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "$K" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
