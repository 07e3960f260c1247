"""Random streams: Philox4x32-10 known-answer vectors, the LFSR113 stream
derivation against the reference's bits, and the C oracle's streams
against the Python restatement."""

import os

import numpy as np

import goldens
from oracle import streams

# Random123 known-answer vectors for philox4x32_10 (ctr, key) -> out
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def test_philox_known_answers():
    for ctr, key, want in KAT:
        assert streams.philox4x32_10(ctr, key) == want


def test_philox_stream_layout():
    s = streams.PhiloxStream(0x1234567890ABCDEF, 77)
    draws = [s.next_u01()[0] for _ in range(9)]
    for n, u in enumerate(draws):
        blk = streams.philox4x32_10((n >> 2, 77, 0, 0), (0x90ABCDEF, 0x12345678))
        assert u == blk[n & 3] * 2.0 ** -32
    assert all(0.0 <= u < 1.0 for u in draws)


def test_c_oracle_philox_matches_python(oracle_lib):
    for seed, k in ((987654321, 0), (1, 2**33 + 5), (2**64 - 1, 12345)):
        s = streams.PhiloxStream(seed, k)
        for n in range(13):
            assert oracle_lib.philox_u01(seed, k, n) == s.next_u01()[0]


def test_lfsr113_derivation_matches_reference_bits(oracle_lib):
    z = np.load(os.path.join(goldens.GOLDEN_DIR, "lfsr113_streams.npz"))
    seed = int(z["seed"])
    for k in range(z["words"].shape[0]):
        want = tuple(int(w) for w in z["words"][k])
        assert tuple(streams.lfsr113_derive(seed, k)) == want
        assert oracle_lib.lfsr113_words(seed, k) == want
        st = streams.Lfsr113Stream(seed, k)
        got = [st.next_u01()[0] for _ in range(z["draws"].shape[1])]
        np.testing.assert_array_equal(got, z["draws"][k])


def test_lfsr113_seed_legalisation():
    assert streams.lfsr113_seed([2, 8, 16, 128]) == [2, 8, 16, 128]
    z = streams.lfsr113_seed([0, 0, 0, 0])
    assert z[0] > 1 and z[1] > 7 and z[2] > 15 and z[3] > 127


def test_scripted_stream_fallback():
    s = streams.ScriptedStream([0.25, 0.5], 0.75)
    assert [s.next_u01()[0] for _ in range(4)] == [0.25, 0.5, 0.75, 0.75]


def test_philox_uniformity_chi2():
    # 2**16 draws over 64 bins; chi2 with 63 dof well inside 99.9 %
    s = streams.PhiloxStream(2024, 3)
    u = np.array([s.next_u01()[0] for _ in range(1 << 16)])
    counts = np.bincount((u * 64).astype(int), minlength=64)
    exp = len(u) / 64
    assert ((counts - exp) ** 2 / exp).sum() < 110.0
