"""CUDA-graph replay of the factor / solve launch sequences (btd_set_graphs, include/blocktri_b200.h).

With device-resident inputs the C ABI captures the whole recursion (every level, assembly and the
base) into one graph per (shape, config, buffer addresses) and replays it.  Replays must be
bitwise identical to direct launches, must read the buffers' current contents, and must report
NotPositiveDefinite with the same coordinates."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_2509_03015_b200 as pkg  # noqa: E402
from paper_2509_03015_b200 import _native  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    prev = _native.lib().btd_set_graphs(1)
    yield
    _native.lib().btd_set_graphs(prev)


def _device(A, B):
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    dB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
    return dA, dB


def _run(dA, dB, cfg=None):
    h = pkg.recursive_factorize(dA, cfg)
    return pkg.recursive_solve(h, dB).blocks.clone()


@pytest.mark.parametrize("N,n,d", [(3000, 64, 1), (20000, 8, 2), (1024, 32, 1), (700, 128, 3), (500, 40, 4)])
def test_graph_replay_bitwise_equals_direct_launches(N, n, d):
    A, B = pkg.generate_spd_btd(N, n, d, seed=5)
    dA, dB = _device(A, B)
    L = _native.lib()
    L.btd_set_graphs(0)
    x_direct = _run(dA, dB)
    c0 = L.btd_launch_count()
    _run(dA, dB)
    direct_launches = L.btd_launch_count() - c0
    L.btd_set_graphs(1)
    xs = [_run(dA, dB) for _ in range(3)]  # capture, then cache hits
    c0 = L.btd_launch_count()
    xs.append(_run(dA, dB))
    graph_launches = L.btd_launch_count() - c0
    for x in xs:
        assert torch.equal(x, x_direct)
    assert graph_launches == direct_launches  # a replay counts the kernels its graph contains


def test_graph_replay_reads_current_buffer_contents():
    A, B = pkg.generate_spd_btd(2000, 32, 1, seed=1)
    A2, B2 = pkg.generate_spd_btd(2000, 32, 1, seed=2)
    dA, dB = _device(A, B)
    _run(dA, dB)
    _run(dA, dB)  # graphs cached for these addresses
    dA.diag.copy_(torch.from_numpy(A2.diag))
    dA.sub.copy_(torch.from_numpy(A2.sub))
    dB.blocks.copy_(torch.from_numpy(B2.blocks))
    x = _run(dA, dB)
    _native.lib().btd_set_graphs(0)
    try:
        x_ref = _run(dA, dB)
    finally:
        _native.lib().btd_set_graphs(1)
    assert torch.equal(x, x_ref)
    _, rres = pkg.residual_report(dA, pkg.BlockRhs(x), dB)
    assert rres <= 1e-12


def test_graph_replay_reports_npd_coordinates():
    A, B = pkg.generate_spd_btd(3000, 64, 1, seed=9)
    diag = A.diag.copy()
    diag[1234, 5, 5] = -10.0
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(diag).cuda(), torch.from_numpy(A.sub).cuda())
    coords = []
    for _ in range(3):
        with pytest.raises(pkg.NotPositiveDefinite) as e:
            pkg.recursive_factorize(dA)
        coords.append((e.value.pivot, e.value.level, e.value.member, e.value.block))
    assert coords[0] == coords[1] == coords[2]
    # a good matrix in the same buffers factors cleanly through the cached graph
    dA.diag.copy_(torch.from_numpy(A.diag))
    h = pkg.recursive_factorize(dA)
    X = pkg.recursive_solve(h, pkg.BlockRhs(torch.from_numpy(B.blocks).cuda()))
    _, rres = pkg.residual_report(dA, X, pkg.BlockRhs(torch.from_numpy(B.blocks).cuda()))
    assert rres <= 1e-12


def test_graphs_replay_on_the_default_stream():
    """torch's default stream is the legacy NULL stream (not capturable): the library records on a
    private stream and replays into the caller's, so steady-state calls are graph replays."""
    A, B = pkg.generate_spd_btd(3000, 64, 1, seed=6)
    dA, dB = _device(A, B)
    for _ in range(3):  # two alternating workspace address sets get captured
        _run(dA, dB)
    L = _native.lib()
    r0 = L.btd_graph_replays()
    _run(dA, dB)
    assert L.btd_graph_replays() - r0 == 2  # the factorization and the solve
