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
