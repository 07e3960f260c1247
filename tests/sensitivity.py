"""The reference algorithm's own one-ulp sensitivity (parity-test helper).

How far the reference algorithm's trajectories move when its first step
size is perturbed by one ulp: the floor for any implementation that is not
bit-identical to it (tree reductions, CUDA hypot).  Measured with the C
restatement (oracle/, pinned to the reference by tests/test_oracle_golden.py)
on exactly the sample under test.  c5 -- 29k attempts per trajectory over
t in [0, 40] -- moves its jump times by ~3e-6; every other config stays
below 1e-6.
"""

import dataclasses

import numpy as np

import goldens

MAXJ = 256
_SENS: dict = {}


def self_sensitivity(oracle_lib, pk, n, stream="philox", begin=0):
    """(oracle run, max |dt*|, max |dvalue|, max |dmean|) under a one-ulp
    perturbation of the first step (cached per problem and sample)."""
    key = (pk.digest, n, stream, begin)
    if key not in _SENS:
        a = oracle_lib.run(pk, goldens.SEED, begin, begin + n, max_jumps=MAXJ, stream=stream)
        pk2 = dataclasses.replace(pk, h0_first=float(np.nextafter(pk.h0_first, 1.0)))
        b = oracle_lib.run(pk2, goldens.SEED, begin, begin + n, max_jumps=MAXJ, stream=stream)
        same = [i for i in range(n) if a["jump_count"][i] == b["jump_count"][i]
                and a["status"][i] == 0 and b["status"][i] == 0]
        dt = max((float(np.abs(a["jump_t"][i, :a["jump_count"][i]]
                               - b["jump_t"][i, :a["jump_count"][i]]).max(initial=0.0))
                  for i in same), default=0.0)
        ok = (a["status"] == 0) & (b["status"] == 0)
        dv = float(np.abs(a["values"][ok] - b["values"][ok]).max(initial=0.0))
        dmean = float(np.abs(a["values"][ok].mean(axis=0) - b["values"][ok].mean(axis=0)).max())
        _SENS[key] = (a, dt, dv, dmean)
    return _SENS[key]
