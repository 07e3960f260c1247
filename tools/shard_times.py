"""Per-shard device times of a config's multi-GPU split, measured one shard at a
time on ONE B200: each rank of run_sharded integrates its block-aligned shard
with no data-path dependence on the others, so T(N) = max over the N shards'
times (+ one all-reduce of the block partials, tens of microseconds over
NVLink, not included).  This pool has single-GPU boxes only; this is the
measured stand-in for the 1/2/4/8-GPU scaling run.

    python tools/shard_times.py c4 [variant] > profiles/r2_shard_times_c4.json
"""
import json, os, sys
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)
from paper_1810_03047_b200 import configs, native
from paper_1810_03047_b200.configs import N_TRAJECTORIES
from paper_1810_03047_b200.engine import DeviceProblem, shard_range
from paper_1810_03047_b200.packing import pack_problem

name = sys.argv[1]
variant = int(sys.argv[2]) if len(sys.argv) > 2 else -1
n_total = int(sys.argv[3]) if len(sys.argv) > 3 else N_TRAJECTORIES[name]
pk = pack_problem(configs.build(name))
SEED = 987654321
REPS = int(os.environ.get("SHARD_REPS", "2"))
rows = []
with DeviceProblem(pk, variant=variant) as dp:
    dp.run(1, 0, 64, resident=True)
    t1 = None
    for world in (1, 2, 4, 8):
        shards = []
        for rank in range(world):
            b, e = shard_range(n_total, world, rank)
            ms = min(dp.run(SEED, b, e, resident=True).total_ms for _ in range(REPS)) if e > b else 0.0
            shards.append({"rank": rank, "begin": b, "end": e, "ms": round(ms, 3)})
        t = max(s["ms"] for s in shards)
        t1 = t1 or t
        rows.append({"n_gpus": world, "t_max_ms": t, "trajectories_per_s": n_total / (t * 1e-3),
                     "efficiency_vs_1": t1 / (world * t), "shards": shards})
print(json.dumps({"config": name, "trajectories": n_total, "variant": native.variants()[variant] if variant >= 0 else "auto",
                  "order": os.environ.get("QTM_ORDER", "1"),
                  "method": "each shard run alone on one B200 (total device time of qtm_run incl. the reductions); "
                            "T(N) = max over shards; the all-reduce is not included",
                  "scaling": rows}, indent=1))
