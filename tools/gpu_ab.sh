#!/bin/bash
# A/B: bench lines for the given variants on a config (default c4) + optional parity subset
# usage: [PARITY=<pytest -k expr>] gpu_ab.sh TAG CONFIG V1 [V2 ...]
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
TAG=$1; CFG=$2; shift 2
for v in "$@"; do
  timeout 600 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu --variant $v > gpurun_out/${TAG}_${CFG}_v$v.json 2> gpurun_out/${TAG}_${CFG}_v$v.err
done
if [ -n "$PARITY" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "$PARITY" > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
fi
