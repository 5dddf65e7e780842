"""Generate golden fixtures by running the REAL reference (build container only).

    python tests/golden/make_golden.py      # needs /root/reference (read-only); writes tests/golden/*.npz

The reference package is imported from /root/reference/pkg/src without installing or copying it
(sys.dont_write_bytecode keeps the read-only tree untouched).  The fixtures pin the CPU oracle
(oracle/blocktri_port.py) and are the GPU parity targets; nothing at test/bench time reads
/root/reference.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import blocktri as bt  # noqa: E402
from blocktri.schur import _factorize_level  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# (N, n, d, seed, crossover, rho, auto)
SOLVE_CASES = [
    (1, 1, 1, 0, 64, 8, False),
    (2, 3, 2, 1, 64, 8, False),
    (3, 2, 1, 2, 1, 1, False),
    (9, 2, 1, 2, 2, 3, False),
    (10, 3, 2, 3, 2, 3, False),
    (40, 4, 3, 3, 4, 2, False),
    (97, 13, 3, 8, 5, 4, False),
    (100, 8, 2, 6, 64, 8, False),
    (150, 40, 2, 9, 16, 3, False),
    (200, 3, 2, 4, 8, 8, False),
    (257, 5, 1, 5, 64, 8, False),
    (300, 64, 1, 7, 64, 8, False),
    (50, 16, 4, 10, 10, 1, False),
    (500, 6, 1, 11, 64, 8, True),
    (130, 24, 5, 12, 7, 6, False),
    (1024, 32, 1, 0, 64, 8, False),   # BASELINE config 1
    (40, 128, 2, 13, 5, 3, False),     # n > 64 (tiled path)
    (12, 192, 3, 14, 64, 8, False),    # n > 64, serial base only
]

SCHUR_CASES = [  # level-0 Schur complement through the reference's own _factorize_level
    (200, 3, 0, 8),
    (97, 4, 1, 3),
    (50, 2, 2, 1),
    (73, 64, 3, 8),
    (61, 32, 4, 5),
]

NPD_CASES = [  # (N, n, seed, rho, crossover, negated global diag blocks)
    (40, 3, 0, 4, 4, (7,)),
    (40, 3, 0, 4, 4, (3, 7)),
    (40, 3, 0, 4, 4, (5,)),
    (40, 3, 0, 4, 4, (0,)),
    (20, 2, 1, 8, 64, (6,)),
    (300, 8, 2, 8, 64, (250, 251)),
    (30, 128, 3, 4, 4, (7,)),
]

GEN_CASES = [(1000, 8, 3, 0), (257, 5, 1, 7), (64, 64, 4, 1), (1, 3, 2, 5), (2, 1, 1, 9)]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {}
    for i, (N, n, d, seed, cross, rho, auto) in enumerate(SOLVE_CASES):
        A, B = bt.generate_spd_btd(N, n, d, seed)
        cfg = bt.RecursionConfig(crossover=cross, segment_length=rho, auto_crossover=auto)
        h = bt.recursive_factorize(A, cfg)
        X = bt.recursive_solve(h, B)
        out[f"solve{i}_meta"] = np.array([N, n, d, seed, cross, rho, int(auto)], dtype=np.int64)
        out[f"solve{i}_x"] = X.blocks
        out[f"solve{i}_levels"] = np.array([lvl.plan.num_blocks for lvl in h.levels] + [h.base.num_blocks],
                                           dtype=np.int64)
        for li, lvl in enumerate(h.levels):
            out[f"solve{i}_seps{li}"] = np.array(lvl.plan.separators, dtype=np.int64)
        out[f"solve{i}_resid"] = np.array(bt.residual_report(A, X, B))
    for i, (N, n, seed, rho) in enumerate(SCHUR_CASES):
        A, _ = bt.generate_spd_btd(N, n, 1, seed)
        cfg = bt.RecursionConfig(segment_length=rho)
        _, S = _factorize_level(A, cfg, 0)
        out[f"schur{i}_meta"] = np.array([N, n, seed, rho], dtype=np.int64)
        out[f"schur{i}_diag"] = S.diag
        out[f"schur{i}_sub"] = S.sub
    for i, (N, n, seed, rho, cross, bad) in enumerate(NPD_CASES):
        A, _ = bt.generate_spd_btd(N, n, 1, seed)
        for b in bad:
            A.diag[b] = -A.diag[b]
        cfg = bt.RecursionConfig(crossover=cross, segment_length=rho)
        try:
            bt.recursive_factorize(A, cfg)
            coords = [-1, -1, -1, -1]
        except bt.NotPositiveDefinite as e:
            coords = [e.pivot, e.level, e.member, e.block]
        out[f"npd{i}_meta"] = np.array([N, n, seed, rho, cross], dtype=np.int64)
        out[f"npd{i}_bad"] = np.array(bad, dtype=np.int64)
        out[f"npd{i}_coords"] = np.array(coords, dtype=np.int64)
    # plans for every N in [3, 700] and rho in [1, 20]
    seps_all, offs = [], [0]
    for rho in range(1, 21):
        for N in range(3, 701):
            s = bt.plan_partition(N, bt.RecursionConfig(segment_length=rho)).separators
            seps_all.extend(s)
            offs.append(len(seps_all))
    out["plans_seps"] = np.array(seps_all, dtype=np.int32)
    out["plans_offsets"] = np.array(offs, dtype=np.int64)
    # generator hashes
    gh = []
    for (N, n, d, seed) in GEN_CASES:
        A, B = bt.generate_spd_btd(N, n, d, seed)
        gh.append(f"{N},{n},{d},{seed}:{sha(A.diag)}:{sha(A.sub)}:{sha(B.blocks)}")
    out["gen_hashes"] = np.array(gh)
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"))


if __name__ == "__main__":
    main()
