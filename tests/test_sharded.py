"""Sharded (multi-GPU) host logic: cut planning is bit-exact with the global plan, and the
G-rank algorithm (all-gathers over gloo, world_size 2 and 3, CPU) reproduces the single-process
solution.  The per-rank math is the CPU oracle engine; the GPU engine is covered by
test_sharded_gpu in test_gpu_parity.py."""

import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import blocktri_port as port
from oracle.sharded_engine import OracleEngine
from paper_2509_03015_b200 import RecursionConfig
from paper_2509_03015_b200.sharded import (ShardedSolver, TorchComm, chunk_inputs, gather_solution,
                                           run_sharded_local, shard_plan)
from paper_2509_03015_b200.synthgen import generate_spd_btd


@pytest.mark.parametrize("N,G", [(1048576, 2), (1048576, 4), (1048576, 8), (65536, 2), (100003, 3), (2000, 2),
                                 (777, 3)])
def test_plan_bit_exact(N, G):
    rho = 8 if N > 10000 else 3
    cross = 64 if N > 10000 else 8
    p = shard_plan(N, G, cross, rho)  # raises if any chunk plan differs from the global one
    assert p.cuts[0] == 0 and p.cuts[-1] == N - 1 and len(p.cuts) == G + 1
    assert sum(p.reduced_sizes) - (G - 1) == p.reduced_N


def _case():
    N, n, d, cross, rho = 2000, 3, 2, 8, 3
    A, B = generate_spd_btd(N, n, d, seed=11)
    return N, n, d, cross, rho, A, B


def test_local_simulation_matches_single_process():
    N, n, d, cross, rho, A, B = _case()
    cfg = RecursionConfig(crossover=cross, segment_length=rho)
    ref = port.solve(port.factorize(A.diag, A.sub, cross, rho), B.blocks)
    for G in (2, 3):
        plan = shard_plan(N, G, cross, rho)
        X = run_sharded_local(plan, OracleEngine(), A.diag, A.sub, B.blocks, cfg)
        assert np.abs(X - ref).max() <= 1e-12 * np.abs(ref).max()


def _worker(rank, world, port_, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N, n, d, cross, rho, A, B = _case()
        cfg = RecursionConfig(crossover=cross, segment_length=rho)
        plan = shard_plan(N, world, cross, rho)
        dg, sg, rg = chunk_inputs(plan, rank, A.diag, A.sub, B.blocks)
        solver = ShardedSolver(plan, rank, TorchComm(), OracleEngine(), cfg).factorize(dg, sg)
        x = solver.solve(rg)
        np.save(os.path.join(out_dir, f"x{rank}.npy"), x)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_world(world):
    N, n, d, cross, rho, A, B = _case()
    ref = port.solve(port.factorize(A.diag, A.sub, cross, rho), B.blocks)
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, 29500 + world + os.getpid() % 1000, tmp), nprocs=world, join=True)
        plan = shard_plan(N, world, cross, rho)
        xs = [np.load(os.path.join(tmp, f"x{g}.npy")) for g in range(world)]
    X = gather_solution(plan, xs)
    assert np.abs(X - ref).max() <= 1e-12 * np.abs(ref).max()
