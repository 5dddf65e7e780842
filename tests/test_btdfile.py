"""BTD1 container (reference btdfile.py): bit-exact round trips, reading a file
written by the real reference, the reference's error classes, and the pinned-memory read feeding
the overlapped host-input factorization."""

import os
import struct

import numpy as np
import pytest

import paper_2509_03015_b200 as pkg

HERE = os.path.dirname(os.path.abspath(__file__))


def test_reads_reference_written_file_bit_exactly():
    A, B = pkg.read_btd(os.path.join(HERE, "golden", "ref_small.btd"))
    G, R = pkg.generate_spd_btd(7, 3, 2, seed=5)  # bit-identical generator
    sub = G.sub.copy()
    sub[2, 1, 1] = -0.0
    assert A.diag.tobytes() == G.diag.tobytes() and A.sub.tobytes() == sub.tobytes()
    assert B.blocks.tobytes() == R.blocks.tobytes()
    assert np.signbit(A.sub[2, 1, 1])


@pytest.mark.parametrize("with_rhs", [True, False])
def test_round_trip(tmp_path, with_rhs):
    A, B = pkg.generate_spd_btd(11, 4, 3, seed=1)
    A.diag[0, 0, 1] = -0.0
    p = tmp_path / "x.btd"
    pkg.write_btd(p, A, B if with_rhs else None)
    assert os.path.getsize(p) == 40 + 8 * (11 * 16 + 10 * 16 + (11 * 4 * 3 if with_rhs else 0))
    A2, B2 = pkg.read_btd(p)
    assert A2.diag.tobytes() == A.diag.tobytes() and A2.sub.tobytes() == A.sub.tobytes()
    assert (B2 is None) == (not with_rhs)
    if with_rhs:
        assert B2.blocks.tobytes() == B.blocks.tobytes()


def test_errors_like_reference(tmp_path):
    A, B = pkg.generate_spd_btd(5, 2, 1, seed=0)
    p = tmp_path / "ok.btd"
    pkg.write_btd(p, A, B)
    raw = p.read_bytes()
    bad = tmp_path / "bad.btd"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(pkg.BadMagic):
        pkg.read_btd(bad)
    bad.write_bytes(raw[:4] + struct.pack("<I", 2) + raw[8:])
    with pytest.raises(pkg.VersionUnsupported):
        pkg.read_btd(bad)
    bad.write_bytes(raw[:-8])
    with pytest.raises(pkg.TruncatedPayload):
        pkg.read_btd(bad)
    bad.write_bytes(raw[:20])
    with pytest.raises(pkg.TruncatedPayload):
        pkg.read_btd(bad)
    bad.write_bytes(raw[:8] + struct.pack("<Q", 0) + raw[16:])
    with pytest.raises(pkg.BtdFormatError):
        pkg.read_btd(bad)
    with pytest.raises(pkg.IoError):
        pkg.read_btd(tmp_path / "missing.btd")
    with pytest.raises(pkg.BtdFormatError):
        pkg.write_btd(tmp_path / "y.btd", A, pkg.BlockRhs(np.zeros((4, 2, 1))))


torch = pytest.importorskip("torch")


@pytest.mark.gpu
def test_pinned_read_feeds_the_gpu_factorization(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    A, B = pkg.generate_spd_btd(20000, 16, 2, seed=4)
    p = tmp_path / "big.btd"
    pkg.write_btd(p, A, B)
    pA, pB = pkg.read_btd(p, pinned=True)
    assert pA.diag.is_pinned()
    X = pkg.recursive_solve(pkg.recursive_factorize(pA), pB)
    ref = pkg.recursive_solve(pkg.recursive_factorize(A), B)
    assert np.array_equal(X.blocks.numpy(), ref.blocks)
