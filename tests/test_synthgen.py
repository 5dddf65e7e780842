"""The chunked generator is bit-identical to the reference generate_spd_btd (golden hashes)."""

import hashlib

import numpy as np

from paper_2509_03015_b200.synthgen import generate_spd_btd


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_generator_bit_identical(golden):
    for rec in golden["gen_hashes"]:
        key, hd, hs, hb = str(rec).split(":")
        N, n, d, seed = (int(v) for v in key.split(","))
        for chunk in (1, 7, 4096):
            A, B = generate_spd_btd(N, n, d, seed, chunk=chunk)
            assert (_sha(A.diag), _sha(A.sub), _sha(B.blocks)) == (hd, hs, hb), (key, chunk)


def test_slice_generator_bit_identical():
    """generate_spd_btd_slice (each rank's chunk of the one global instance, bench.py N > 1) equals
    the corresponding rows of the full generator, including the first / last rows and tiny N."""
    from paper_2509_03015_b200.synthgen import generate_spd_btd_slice
    for (N, n, d) in [(1000, 5, 3), (2, 3, 1), (1, 2, 2), (300, 8, 1)]:
        A, B = generate_spd_btd(N, n, d, seed=3, chunk=64)
        for f, l in [(0, N - 1), (0, 0), (N - 1, N - 1), (N // 3, N // 2), (1, max(N - 2, 1))]:
            if not 0 <= f <= l < N:
                continue
            dg, sb, rh = generate_spd_btd_slice(N, n, d, 3, f, l, chunk=37)
            assert np.array_equal(dg, A.diag[f:l + 1]) and np.array_equal(sb, A.sub[f:l])
            assert np.array_equal(rh, B.blocks[f:l + 1])
