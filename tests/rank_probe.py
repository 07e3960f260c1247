"""One rank of a launcher test (tests/test_sharded_gloo.py): joins the job
from the torchrun-style environment bench.launch_ranks sets, runs
run_sharded on c1 with the C oracle as the per-rank runner over gloo, and
rank 0 prints the ensemble sums as JSON (hex of the float64 bits)."""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def main():
    import torch.distributed as dist
    from paper_1810_03047_b200 import configs
    from paper_1810_03047_b200.engine import run_sharded
    from test_sharded_gloo import _oracle_runner
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    res = run_sharded(configs.build("c1"), int(sys.argv[1]), 77, rank=rank, world_size=world,
                      runner=_oracle_runner)
    if rank == 0:
        print(json.dumps({"world": world, "n": res.n_trajectories,
                          "sum": (res.values * res.n_trajectories).tobytes().hex(),
                          "sumsq": res.sumsq.tobytes().hex()}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
