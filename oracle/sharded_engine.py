"""CPU ORACLE engine for the sharded driver -- test infrastructure only.

Implements the per-rank interface of paper_2509_03015_b200.sharded (factor_partial, solve_down,
solve_up, factor_full, solve_full) with the numpy restatement of the reference
(oracle/blocktri_port.py: factor_level = bt/schur.py:329-343 + compute_schur :156-193;
split/fold/boundary/assemble = bt/schur.py:196-286), so the multi-process host logic (cuts,
ownership, reduced-system assembly, all-gathers over gloo) can be checked without a GPU.
"""

from __future__ import annotations

import numpy as np

from . import blocktri_port as port


class OracleEngine:
    def factor_partial(self, diag, sub, L, cfg):
        levels, cd, cs = [], diag, sub
        for lvl in range(L):
            rec, cd, cs = port.factor_level(cd, cs, cfg.segment_length, lvl)
            levels.append(rec)
        return {"levels": levels}, cd, cs

    def solve_down(self, state, rhs):
        b, stack = rhs.copy(), []
        for rec in state["levels"]:
            seps, seg, F = rec["seps"], rec["seg"], rec["F"]
            K, J, n = F.shape[0], F.shape[1], F.shape[2]
            d = b.shape[2]
            interior = np.zeros((K, J, n, d))
            for k, (a, c) in enumerate(seg):
                interior[k, :c - a] = b[a:c]
            bsep = b[seps].copy()
            contrib = np.empty((K, 2 * n, d))
            port.gemm_batch(contrib, F.reshape(K, J * n, 2 * n), interior.reshape(K, J * n, d), ta=True, alpha=-1.0)
            bsep[:-1] += contrib[:, :n]
            bsep[1:] += contrib[:, n:]
            stack.append((rec, interior, b))
            b = bsep
        state["stack"] = stack
        return b

    def solve_up(self, state, rhs, red_x):
        x = np.array(red_x)
        for rec, interior, b in reversed(state["stack"]):
            seps, seg, lengths = rec["seps"], rec["seg"], rec["lengths"]
            interior = interior.copy()
            K = interior.shape[0]
            port.gemm_batch(interior[:, 0], rec["CL"], x[:-1], alpha=-1.0, beta=1.0)
            idx = np.arange(K)
            last = interior[idx, lengths - 1]
            port.gemm_batch(last, rec["CR"], x[1:], ta=True, alpha=-1.0, beta=1.0)
            interior[idx, lengths - 1] = last
            port.block_solve(rec["D"], rec["S"], interior)
            out = np.empty_like(b)
            out[seps] = x
            for k, (a, c) in enumerate(seg):
                out[a:c] = interior[k, :c - a]
            x = out
        return x

    def factor_full(self, diag, sub, cfg):
        return port.factorize(np.ascontiguousarray(diag), np.ascontiguousarray(sub), cfg.crossover,
                              cfg.segment_length, cfg.max_levels, cfg.auto_crossover)

    def solve_full(self, h, rhs):
        return port.solve(h, np.ascontiguousarray(rhs))
