"""Event-driven model of the persistent trajectory grid on 1..8 B200s.

Inputs measured on one B200 (tools/gpu_scale_inputs.sh writes them):
  * the per-trajectory work of a config's full ensemble (attempt counts from the
    device's per-trajectory counters);
  * the time per unit of work of a trajectory CTA that has its SM to itself (tau1)
    and of one that shares it with a second CTA (tau2), from two timed launches of
    148 and 296 trajectories.

Model: every GPU runs `sms * ctas_per_sm` persistent CTAs (CTA j on SM j % sms);
a CTA pulls the next trajectory from its queue when it finishes one and exits when
the queue is empty; a CTA progresses at 1/tau1 work units per second while alone on
its SM and at 1/tau2 while its neighbour is still running.  Queues:
  static  -- contiguous block-aligned shards per GPU (engine.shard_range), one
             counter per GPU: what run_sharded does;
  global  -- one counter for all GPUs (a cross-GPU work queue).
Reports the makespan, the strong-scaling efficiency T(1) / (N T(N)), and the same for
a static split with the trajectories dealt longest-first (a lower bound on what any
reordering can reach).

    python tools/scale_sim.py gpurun_out/scale_inputs_c4.npz [--sms 148] [--ctas 2]
"""
from __future__ import annotations

import argparse
import heapq
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def shard_ranges(n_total: int, world: int):
    from paper_1810_03047_b200.engine import shard_range
    return [shard_range(n_total, world, r) for r in range(world)]


def simulate(work_by_gpu, sms: int, ctas: int, tau1: float, tau2: float, shared_queue=None) -> float:
    """Makespan (seconds).  work_by_gpu: list of per-GPU work lists in pull order, or,
    with shared_queue (one list), every GPU pulls from that list."""
    n_gpu = len(work_by_gpu) if shared_queue is None else work_by_gpu
    queues = [list(reversed(w)) for w in work_by_gpu] if shared_queue is None else None
    shared = list(reversed(shared_queue)) if shared_queue is not None else None

    def pull(g):
        if shared is not None:
            return shared.pop() if shared else None
        return queues[g].pop() if queues[g] else None

    # state per (gpu, sm): remaining work of each resident CTA
    t = 0.0
    # event loop over all SMs: each SM is independent given the pull order, but the
    # pull order couples them -> global event queue keyed by finish time
    rem = {}      # (g, sm) -> list of remaining work of active CTAs
    last = {}     # (g, sm) -> time of last update
    heap = []
    ver = {}

    def rate(k):
        return 1.0 / (tau1 if k <= 1 else tau2)

    def schedule(key, now):
        ver[key] = ver.get(key, 0) + 1
        r = rem[key]
        if not r:
            return
        k = len(r)
        dt = min(r) / rate(k)
        heapq.heappush(heap, (now + dt, ver[key], key))

    def advance(key, now):
        r = rem[key]
        k = len(r)
        if k:
            done = (now - last[key]) * rate(k)
            rem[key] = [x - done for x in r]
        last[key] = now

    # initial fill: CTA j of GPU g pulls in launch order (breadth-first over SMs)
    for g in range(n_gpu):
        for s in range(sms):
            rem[(g, s)] = []
            last[(g, s)] = 0.0
    for c in range(ctas):
        for s in range(sms):
            for g in range(n_gpu):
                w = pull(g)
                if w is not None:
                    rem[(g, s)].append(float(w))
    for key in rem:
        schedule(key, 0.0)
    while heap:
        now, v, key = heapq.heappop(heap)
        if ver.get(key) != v:
            continue
        advance(key, now)
        t = now
        r = rem[key]
        # the CTA with the least remaining work is the one this event finishes
        # (ties and rounding: everything within a relative 1e-12 of it too)
        lim = min(r) + 1e-12 * abs(max(r)) + 1e-9
        keep = []
        for x in r:
            if x <= lim:
                w = pull(key[0])
                if w is not None:
                    keep.append(float(w))
            else:
                keep.append(x)
        rem[key] = keep
        schedule(key, now)
    return t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("inputs")
    ap.add_argument("--sms", type=int, default=148)
    ap.add_argument("--ctas", type=int, default=2)
    ap.add_argument("--gpus", type=int, nargs="*", default=[1, 2, 4, 8])
    a = ap.parse_args()
    z = np.load(a.inputs)
    work = z["attempts"].astype(np.float64)
    n = work.size
    t148, t296 = float(z["t_alone_ms"]) * 1e-3, float(z["t_pair_ms"]) * 1e-3
    w148, w296 = z["work_alone"].astype(np.float64), z["work_pair"].astype(np.float64)
    # a launch ends with its longest CTA: tau = launch time / the largest per-CTA work
    tau1 = t148 / w148.max()
    # tau2 from the two-per-SM launch: the value at which the model reproduces its time
    lo, hi = tau1, 4.0 * tau1
    for _ in range(50):
        mid = 0.5 * (lo + hi)
        if simulate([w296], a.sms, a.ctas, tau1, mid) > t296:
            hi = mid
        else:
            lo = mid
    tau2 = 0.5 * (lo + hi)
    print(f"{n} trajectories, work/trajectory mean {work.mean():.0f} (min {work.min():.0f}, max {work.max():.0f}) attempts")
    print(f"tau1 {tau1 * 1e6:.3f} us/attempt alone on an SM, tau2 {tau2 * 1e6:.3f} us/attempt sharing it "
          f"(pair throughput {2 * tau1 / tau2:.2f}x)")
    full = float(z["t_full_ms"]) * 1e-3 if "t_full_ms" in z.files else None
    base = None
    for g in a.gpus:
        ranges = shard_ranges(n, g)
        static = simulate([work[b:e] for b, e in ranges], a.sms, a.ctas, tau1, tau2)
        glob = simulate(g, a.sms, a.ctas, tau1, tau2, shared_queue=work)
        lpt = simulate([np.sort(work[b:e])[::-1] for b, e in ranges], a.sms, a.ctas, tau1, tau2)
        glpt = simulate(g, a.sms, a.ctas, tau1, tau2, shared_queue=np.sort(work)[::-1])
        if base is None:
            base = static
            if full:
                print(f"model check: simulated 1-GPU launch {static * 1e3:.1f} ms vs measured {full * 1e3:.1f} ms")
        ideal = work.sum() * tau2 / (g * a.sms * a.ctas)
        print(f"N={g}: static {static * 1e3:7.2f} ms (eff {base / (g * static):.3f})   "
              f"global queue {glob * 1e3:7.2f} ms (eff {base / (g * glob):.3f})   "
              f"static longest-first {lpt * 1e3:7.2f} ms (eff {base / (g * lpt):.3f})   "
              f"global longest-first {glpt * 1e3:7.2f} ms (eff {base / (g * glpt):.3f})   "
              f"[no-tail bound {ideal * 1e3:.2f} ms]")


if __name__ == "__main__":
    main()
