"""The multi-GPU product path with a real communicator: 2 ranks (processes) on one GPU, each
running the CUDA engine (sm_100a partial factor / solve kernels through the C ABI) on its slice of
ONE global instance, the reduced system all-gathered by TorchComm over gloo (NCCL refuses two
ranks on one device).  The gathered solution equals the unsharded single-process solve."""

import os
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import paper_2509_03015_b200 as pkg  # noqa: E402
from paper_2509_03015_b200.sharded import CudaEngine, ShardedSolver, TorchComm, gather_solution, shard_plan  # noqa: E402
from paper_2509_03015_b200.synthgen import generate_spd_btd_slice  # noqa: E402

CASES = [(30000, 64, 2, 64, 8), (20000, 16, 3, 8, 3), (4000, 128, 1, 16, 4)]


def _worker(rank, world, port, out_dir, case):
    N, n, d, cross, rho = case
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        plan = shard_plan(N, world, cross, rho)
        a, b = plan.chunk(rank)
        dg, sb, rh = generate_spd_btd_slice(N, n, d, 7, a, b)
        if rank > 0:  # shared boundary block / rhs panel owned by the left rank
            dg[0] = 0.0
            rh[0] = 0.0
        dev = torch.device("cuda", 0)
        solver = ShardedSolver(plan, rank, TorchComm(), CudaEngine(dev))
        solver.factorize(torch.from_numpy(dg).to(dev), torch.from_numpy(sb).to(dev))
        x = solver.solve(torch.from_numpy(rh).to(dev))
        np.save(os.path.join(out_dir, f"x{rank}.npy"), x.cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
def test_two_ranks_one_gpu_gloo_equals_unsharded(case):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    N, n, d, cross, rho = case
    world = 2
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, 29600 + os.getpid() % 1000, tmp, case), nprocs=world, join=True)
        xs = [np.load(os.path.join(tmp, f"x{g}.npy")) for g in range(world)]
    plan = shard_plan(N, world, cross, rho)
    X = gather_solution(plan, xs)
    A, B = pkg.generate_spd_btd(N, n, d, seed=7)
    ref = pkg.recursive_solve(pkg.recursive_factorize(A, pkg.RecursionConfig(crossover=cross, segment_length=rho)),
                              B).blocks
    assert np.abs(X - ref).max() <= 1e-12 * np.abs(ref).max()
    assert pkg.residual_report(A, pkg.BlockRhs(X), B)[1] <= 1e-12
