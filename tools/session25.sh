cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for c in c1 c2 c3; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/r01c_$c.json 2>&1; done
timeout 1200 python bench.py --config c5 --steps 1 --warmup 3 > gpurun_out/r01c_c5.json 2>&1
timeout 600 python bench.py > gpurun_out/r01c_c4.json 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/r01c_ref.json 2>&1
