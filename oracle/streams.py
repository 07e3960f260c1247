"""Per-trajectory random streams for the parity harness (TEST INFRASTRUCTURE).

This module belongs to the oracle: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline leg may import it.  The product path draws
its numbers on the device (``paper_1810_03047_b200/csrc/qtm_rng.cuh``).

Every stream object exposes ``next_u01() -> (u, self)``, the only contract
the reference trajectory engine needs from its rng state
(/root/reference/pkg/src/mcwf/trajectory.py:194-196, the same duck type as
the reference test oracle ``ScriptedDraws``, tests/oracles.py:60-72).

Three stream kinds, all keyed by the *global* trajectory index k so that a
trajectory's draws do not depend on how the ensemble is sharded:

* ``philox``  -- counter-based Philox4x32-10 (Salmon et al., SC'11).  Draw n
  of trajectory k is word ``n & 3`` of the block
  ``philox(ctr=(n >> 2, k_lo, k_hi, 0), key=(seed_lo, seed_hi))``, scaled by
  2**-32 exactly like the reference LFSR113 output (rng.py:37-48).
* ``lfsr113`` -- the reference's own combined Tausworthe generator, one
  stream per trajectory seeded with ``derive_stream(seed, k)``
  (rng.py:51-60 seeding, rng.py:76-90 derivation).  Restated here from the
  published algorithm; pinned bit-for-bit against the reference in
  tests/test_oracle_rng.py.
* ``scripted`` -- replays a fixed list of draws then a fallback value,
  mirroring tests/oracles.py:60-72.
"""

from __future__ import annotations

M32 = 0xFFFFFFFF
M64 = 0xFFFFFFFFFFFFFFFF
INV_2_32 = 2.3283064365386963e-10  # 2**-32

PHILOX_M0, PHILOX_M1 = 0xD2511F53, 0xCD9E8D57
PHILOX_W0, PHILOX_W1 = 0x9E3779B9, 0xBB67AE85

STREAM_KINDS = {"philox": 0, "lfsr113": 1, "scripted": 2}


def philox4x32_10(ctr, key, rounds=10):
    """Philox4x32 block function; returns four 32-bit words."""
    c0, c1, c2, c3 = (int(x) & M32 for x in ctr)
    k0, k1 = (int(x) & M32 for x in key)
    for r in range(rounds):
        if r:
            k0 = (k0 + PHILOX_W0) & M32
            k1 = (k1 + PHILOX_W1) & M32
        p0 = PHILOX_M0 * c0
        p1 = PHILOX_M1 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0, p1 & M32, (p0 >> 32) ^ c3 ^ k1, p0 & M32)
    return c0, c1, c2, c3


class PhiloxStream:
    """Draw sequence of trajectory ``k`` under master seed ``seed``."""

    def __init__(self, seed: int, k: int):
        if k < 0:
            raise ValueError("trajectory index must be non-negative")
        self.seed = int(seed) & M64
        self.k = int(k) & M64
        self.n = 0
        self._block = None

    def next_u01(self):
        n = self.n
        if n & 3 == 0 or self._block is None:
            self._block = philox4x32_10((n >> 2, self.k & M32, self.k >> 32, 0),
                                        (self.seed & M32, self.seed >> 32))
        u = self._block[n & 3] * INV_2_32
        self.n = n + 1
        return u, self


# -- LFSR113 (restated from the published combined Tausworthe routine) --------

_LFSR_MIN = (1, 7, 15, 127)


def lfsr113_seed(words):
    """Legalise four seed words: a word at or below its bound gets bound+1
    OR-ed in (reference rng.py:51-60)."""
    out = []
    for w, lo in zip(words, _LFSR_MIN):
        w = int(w) & M32
        if w <= lo:
            w |= lo + 1
        out.append(w)
    return out


def lfsr113_next(z):
    """Advance the four-word state in place; return the 32-bit output."""
    z1, z2, z3, z4 = z
    b = (((z1 << 6) & M32) ^ z1) >> 13
    z1 = (((z1 & 0xFFFFFFFE) << 18) & M32) ^ b
    b = (((z2 << 2) & M32) ^ z2) >> 27
    z2 = (((z2 & 0xFFFFFFF8) << 2) & M32) ^ b
    b = (((z3 << 13) & M32) ^ z3) >> 21
    z3 = (((z3 & 0xFFFFFFF0) << 7) & M32) ^ b
    b = (((z4 << 3) & M32) ^ z4) >> 12
    z4 = (((z4 & 0xFFFFFF80) << 13) & M32) ^ b
    z[:] = [z1, z2, z3, z4]
    return z1 ^ z2 ^ z3 ^ z4


def _splitmix_mix(x):
    x &= M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def lfsr113_derive(master_seed: int, index: int):
    """Per-index state: avalanche (seed, index) into four words, legalise,
    discard 16 draws (reference rng.py:76-90)."""
    if index < 0:
        raise ValueError("rank must be non-negative")
    golden = 0x9E3779B97F4A7C15
    x = (int(master_seed) & M64) ^ (((index + 1) * golden) & M64)
    words = []
    for _ in range(2):
        x = _splitmix_mix(x + golden)
        words += [x & M32, (x >> 32) & M32]
    z = lfsr113_seed(words)
    for _ in range(16):
        lfsr113_next(z)
    return z


class Lfsr113Stream:
    def __init__(self, seed: int, k: int):
        self.z = lfsr113_derive(seed, k)

    @property
    def words(self):
        return tuple(self.z)

    def next_u01(self):
        return lfsr113_next(self.z) * INV_2_32, self


class ScriptedStream:
    """Replays ``draws`` then returns ``fallback`` forever."""

    def __init__(self, draws, fallback=0.999999):
        self.draws = [float(x) for x in draws]
        self.fallback = float(fallback)
        self.n = 0

    def next_u01(self):
        u = self.draws[self.n] if self.n < len(self.draws) else self.fallback
        self.n += 1
        return u, self


def make_stream(kind: str, seed: int, k: int, script=None, fallback=0.999999):
    if kind == "philox":
        return PhiloxStream(seed, k)
    if kind == "lfsr113":
        return Lfsr113Stream(seed, k)
    if kind == "scripted":
        return ScriptedStream(script if script is not None else [], fallback)
    raise ValueError(f"unknown stream kind {kind!r}")
