cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/mr2.log 2>&1
echo "rc=$?" >> gpurun_out/mr2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/mr2_ref.log 2>&1
echo "rc=$?" >> gpurun_out/mr2_ref.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref1.log 2>&1
echo "rc=$?" >> gpurun_out/ref1.log
