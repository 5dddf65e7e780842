// Streaming level elimination for 32 < n <= 64 (one CTA per segment, 16 warps, 1 CTA / SM).
//
// Same algebra as factor_level_kernel (btd_factor.cuh, "Y-form" of the reference chain
// permute_split / factorize_btd_batch / solve_btd_batch(F) / compute_schur, bt/schur.py:98-193,
// bt/block_cholesky.py:24-68); the schedule removes the triangular inverse and the Pt product from
// the per-step critical path:
//
//   group A (warp 0)     : Cholesky of D_j, panel by panel (single-warp chain, btd_chain.cuh): L
//                          with its 8x8 diagonal tiles inverted ("leaves"); every leaf is published
//                          on its own named barrier (bar.arrive; group B waits with bar.sync) as
//                          soon as it exists.  (Round 1 used mbarriers, which compute-sanitizer's
//                          racecheck does not model; with named barriers racecheck checks it.)
//   group B (warps 4-15) : owns 24 register-resident 8-row tiles of the stacked right-hand side
//                          [X1; Gt; I] (X1 = A_{j+1,j} or C_R, Gt = fill coupling, I = identity)
//                          and runs the blocked triangular solve Pt = [X1; Gt; I] L_j^{-T} one
//                          column block behind the pivot chain:
//                             Pt(:,p) = X(:,p) Linv_pp^T ;  X(:,c) -= Pt(:,p) L_cp^T  (c > p)
//                          (C-fragment -> A-fragment conversion by warp shuffles, no smem round
//                          trip).  Pt1 = L_{j+1,j}, Pt3 = Linv_j^T go straight to HBM (Lsub, packed
//                          Linv); Pt1, Pt2 to shared memory.  Before that, for step j-1:
//                          S_L += Pt2 Pt2^T (global, L2 resident) and the next fill coupling
//                          Gt_j = -Pt2 Pt1^T, computed directly into the Gt tiles' registers.
//   all warps (phase 2)  : D_{j+1} = A_{j+1,j+1} - Pt1 Pt1^T (A prefetched into DN), or S_R at the
//                          last row.
// Per step the critical path is the pivot chain + one column block of the solve + the D update.
#pragma once

#include "btd_factor.cuh"

namespace btd {

#ifdef BTD_PHASE_PROF
#define BTD_SPROF(slot, t0)                                                                        \
  do {                                                                                            \
    if (blockIdx.x == 0) atomicAdd(&g_phase_cycles[slot], (unsigned long long)(clock64() - (t0))); \
  } while (0)
#else
#define BTD_SPROF(slot, t0)
#endif

struct StreamShape {
  static constexpr int NT = 64;
  static constexpr int LD = FactorShape<64>::LD;
  static constexpr int NWA = FactorShape<64>::NWA;  // 4
  static constexpr int NWB = 8;
  static constexpr int NW = NWA + NWB;
  static constexpr int NTHREADS = 32 * NW;
  static constexpr int NB = 32 * NWB;
  // XP (2NT x LD: Pt1 | Pt2) + DL (NT x LD) + DN (NT x LD: prefetched A_{j+1,j+1})
  static constexpr size_t SMEM = (size_t)4 * NT * LD * sizeof(double);
  static_assert(NWA == 4, "potrf group is 4 warps at NT = 64");
};

constexpr int kBarS = 3;      // named barrier of group B (streaming kernel)
constexpr int kBarLeaf0 = 4;  // named barriers 4..11: leaf p published by the pivot chain (warp 0) to group B

// cp.async staging of an n x n row-major block into an NT x LD tile by `nb` threads (index gt).
template <int NT, int LD>
__device__ __forceinline__ void stage_block_async_part(double* sm, const double* g, int n, int gt, int nb) {
  if ((n & 1) == 0) {
    for (int idx = gt; idx < NT * (NT / 2); idx += nb) {
      const int r = idx / (NT / 2), c = (idx % (NT / 2)) * 2;
      const bool ok = r < n && c < n;
      cp_async16(sm + r * LD + c, ok ? (const void*)(g + (size_t)r * n + c) : (const void*)g, ok ? 16 : 0);
    }
  } else {
    for (int idx = gt; idx < NT * NT; idx += nb) {
      const int r = idx / NT, c = idx % NT;
      const bool ok = r < n && c < n;
      cp_async8(sm + r * LD + c, ok ? (const void*)(g + (size_t)r * n + c) : (const void*)g, ok ? 8 : 0);
    }
  }
}

// C fragment (lane: row l/4, cols 2(l%4), 2(l%4)+1) -> A fragments of the two k-halves
// (lane: row l/4, col l%4 and col l%4 + 4).
__device__ __forceinline__ void c2a(double v0, double v1, int lane, double& a0, double& a1) {
  const int base = lane & ~3;
  const int sa = base + ((lane & 3) >> 1), sb = sa + 2;
  const double x0 = __shfl_sync(0xffffffffu, v0, sa), x1 = __shfl_sync(0xffffffffu, v1, sa);
  const double y0 = __shfl_sync(0xffffffffu, v0, sb), y1 = __shfl_sync(0xffffffffu, v1, sb);
  a0 = (lane & 1) ? x1 : x0;
  a1 = (lane & 1) ? y1 : y0;
}

// Load an 8-row tile (rows r0.., all NT columns) of a row-major n x n global block into C-fragment
// registers, zero padded.
__device__ __forceinline__ void load_tile_c(double (&t)[8][2], const double* g, int r0, int n, int lane) {
  const int r = r0 + (lane >> 2);
#pragma unroll
  for (int ct = 0; ct < 8; ++ct) {
    const int c = ct * 8 + 2 * (lane & 3);
    if ((n & 1) == 0) {
      double2 v = make_double2(0.0, 0.0);
      if (r < n && c < n) v = *reinterpret_cast<const double2*>(g + (size_t)r * n + c);
      t[ct][0] = v.x;
      t[ct][1] = v.y;
    } else {
      t[ct][0] = (r < n && c < n) ? g[(size_t)r * n + c] : 0.0;
      t[ct][1] = (r < n && c + 1 < n) ? g[(size_t)r * n + c + 1] : 0.0;
    }
  }
}

// S_L tile t (16x16 tile of the lower triangle) += Pt2 Pt2^T, read-modify-write in its global
// (L2-resident) slot; `first` starts from zero.
__device__ __forceinline__ void sl_tile64(const double* XP, double* sl, int n, bool first, int t, int lane) {
  using S = FactorShape<64>;
  constexpr int TS = S::TS, SUB = S::SUB, HALF = S::HALF;
  int rr, cc;
  tri_decode(t, rr, cc);
  double acc[SUB][SUB][2];
#pragma unroll
  for (int i = 0; i < SUB; ++i)
#pragma unroll
    for (int jj = 0; jj < SUB; ++jj) {
      const int r = rr * TS + i * 8 + (lane >> 2);
      const int c = cc * TS + jj * 8 + 2 * (lane & 3);
      const double* src = sl + (size_t)r * n + c;
      acc[i][jj][0] = (!first && r < n && c < n) ? src[0] : 0.0;
      acc[i][jj][1] = (!first && r < n && c + 1 < n) ? src[1] : 0.0;
    }
  syrk_tile<64>(XP, HALF + rr, HALF + cc, acc, lane);
#pragma unroll
  for (int i = 0; i < SUB; ++i)
#pragma unroll
    for (int jj = 0; jj < SUB; ++jj) {
      if (rr == cc && jj > i) continue;
      const int r = rr * TS + i * 8 + (lane >> 2);
      const int c = cc * TS + jj * 8 + 2 * (lane & 3);
      double* dst = sl + (size_t)r * n + c;
      if (r < n && c < n) dst[0] = acc[i][jj][0];
      if (r < n && c + 1 < n) dst[1] = acc[i][jj][1];
    }
}

// acc(8 x 64, C fragments) = -Pt2[rows 8g..] * Pt1^T  (one tile of the fill product)
__device__ __forceinline__ void fill_tile64(const double* XP, int g, double (&acc)[8][2], int lane) {
  constexpr int LD = StreamShape::LD, NT = 64;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c][0] = acc[c][1] = 0.0;
  const double* pa = XP + (NT + g * 8 + (lane >> 2)) * LD + (lane & 3);
  const double* pb = XP + (lane >> 2) * LD + (lane & 3);
#pragma unroll 1
  for (int k0 = 0; k0 < NT; k0 += 4) {
    const double a0 = -pa[k0];
#pragma unroll
    for (int ct = 0; ct < 8; ++ct) dmma(acc[ct], a0, pb[ct * 8 * LD + k0]);
  }
}

__global__ void __launch_bounds__(StreamShape::NTHREADS, 1) factor_stream_kernel(FactorArgs args) {
  using SS = StreamShape;
  constexpr int NT = 64, LD = SS::LD, NWA = SS::NWA, NB = SS::NB;
  extern __shared__ __align__(16) double smem[];
  double* XP = smem;                // rows 0..63: Pt1, rows 64..127: Pt2 (of the last finished step)
  double* DL = smem + 2 * NT * LD;  // D_j -> L_j (+ leaves)
  double* DN = DL + NT * LD;        // A_{j+1,j+1} (prefetch)
  __shared__ int s_fail_a, s_fail;

  const int k = args.k0 + blockIdx.x;
  if (cta_superseded(args.err, args.level, 0, k)) return;
  const bool coupled = !args.base;
  const long long start = coupled ? (long long)args.seps[k] + 1 : 0;
  const long long stop = coupled ? (long long)args.seps[k + 1] : args.N;
  const int J = (int)(stop - start);
  const int n = args.n;
  const size_t bs = (size_t)n * n;
  const int pk = packed_offset_(n);
  const int tid = threadIdx.x, lane = tid & 31, hw = tid >> 5;
  // Roles by SM sub-partition: group A is warp 0 (the pivot chain) plus the warps that share its
  // sub-partition (read from %warpid), so none of group B's DMMA work is issued next to the chain
  // (a DMMA warp on the chain's sub-partition slows it ~1.6x; tools/chain2_bench.cu).  `warp` is
  // the logical warp index every role below is keyed on; logical warp 0 is hardware warp 0.
  __shared__ int s_smsp[SS::NW];
  {
    unsigned wid;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    if (lane == 0) s_smsp[hw] = (int)(wid & 3);
  }
  __syncthreads();
  int warp = 0;
  {
    const int a0 = s_smsp[0];
    bool inA[SS::NW];
    int na = 0;
#pragma unroll
    for (int w = 0; w < SS::NW; ++w) {
      inA[w] = (w == 0) || (s_smsp[w] == a0 && na < NWA);
      na += inA[w];
    }
#pragma unroll
    for (int w = 1; w < SS::NW; ++w)  // an unexpected warp placement: fill group A in order
      if (!inA[w] && na < NWA) {
        inA[w] = true;
        ++na;
      }
    int pos = 0;
#pragma unroll
    for (int w = 0; w < SS::NW; ++w)
      if (inA[w]) warp = (w == hw) ? pos++ : (pos++, warp);
#pragma unroll
    for (int w = 0; w < SS::NW; ++w)
      if (!inA[w]) warp = (w == hw) ? pos++ : (pos++, warp);
  }
  const bool in_a = warp < NWA;
  const int b = warp - NWA;  // group-B warp index
  double* sl = coupled ? args.Sl + (size_t)k * bs : nullptr;

  // group B warp b owns the 8-row tiles b of X1 (X), of Gt (G) and of the identity (Y)

  // ---- prologue ----
  if (tid == 0) {
    s_fail = 0;
  }
  stage_block_async_part<NT, LD>(DL, args.diag + start * bs, n, tid, SS::NTHREADS);
  if (J > 1) stage_block_async_part<NT, LD>(DN, args.diag + (start + 1) * bs, n, tid, SS::NTHREADS);
  cp_async_commit();
  if (coupled) {
    // Gt_0 = C_L^T (rows 64.. of XP, as if it were the fill output of a step -1)
    stage_block_transposed<NT, LD, SS::NTHREADS>(XP + NT * LD, args.sub + (start - 1) * bs, n);
    copy_block<SS::NTHREADS>(args.Lsub + (start - 1) * bs, args.sub + (start - 1) * bs, n);  // C_L
    copy_block<SS::NTHREADS>(args.Lsub + (stop - 1) * bs, args.sub + (stop - 1) * bs, n);    // C_R
  }
  cp_async_wait_all();
  for (int r = n + tid; r < NT; r += SS::NTHREADS) DL[r * LD + r] = 1.0;
  __syncthreads();

  for (int j = 0; j < J; ++j) {
    const bool last = (j == J - 1);
    const long long tstep = clock64();
    if (in_a) {
      // ======== group A: Cholesky of D_j, leaves published one by one ========
      // single-warp left-looking chain (btd_chain.cuh): no group barriers on the critical path
      const int fail = warp == 0 ? chain_potrf64<LD, NT>(DL, lane, kBarLeaf0, 32 + NB) : 0;
      if (fail && tid == 0) s_fail = fail;
      if (tid == 0) BTD_SPROF(11, tstep);
    } else {
      // ======== group B ========
      {
      double X[8][2], G[8][2], Y[8][2];  // C fragments of the three owned tiles
      const bool has_x = coupled || !last;  // base: no X1 at the last row
      const double* x1src = !last ? args.sub + (start + j) * bs : args.sub + (stop - 1) * bs;
      if (has_x) load_tile_c(X, x1src, 8 * b, n, lane);
#pragma unroll
      for (int c = 0; c < 8; ++c) {  // identity tile b: element (r, c) = (c == 8 b + r)
        const int col = c * 8 + 2 * (lane & 3), row = 8 * b + (lane >> 2);
        Y[c][0] = (col == row) ? 1.0 : 0.0;
        Y[c][1] = (col + 1 == row) ? 1.0 : 0.0;
      }
      if (coupled) {
        if (j > 0) {
          // step j-1: S_L += Pt2 Pt2^T (global) and the fill Gt_j = -Pt2 Pt1^T straight into G
          fill_tile64(XP, b, G, lane);
          for (int u = b; u < FactorShape<64>::NSL; u += SS::NWB) sl_tile64(XP, sl, n, j == 1, u, lane);
        } else {  // Gt_0 = C_L^T from the prologue
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const double* s0 = XP + (NT + 8 * b + (lane >> 2)) * LD + c * 8 + 2 * (lane & 3);
            G[c][0] = s0[0];
            G[c][1] = s0[1];
          }
        }
      }
      named_sync(kBarS, NB);  // XP (step j-1's Pt) fully consumed: the solve may overwrite it
      if (b == 0 && lane == 0) BTD_SPROF(12, tstep);
      // ---- blocked triangular solve [X; G; Y] L_j^{-T}, one column block behind the pivot chain ----
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        named_sync(kBarLeaf0 + p, 32 + NB);  // leaf p and the rows below it (chain_potrf)
        const double* lp = DL + (8 * p + (lane >> 2)) * LD + 8 * p + (lane & 3);
        const double lb0 = lp[0], lb1 = lp[4];  // B = Linv_pp^T
        const bool actY = p >= b;  // the identity tile is zero left of its diagonal block
        double nx0 = 0.0, nx1 = 0.0, ng0 = 0.0, ng1 = 0.0, ny0 = 0.0, ny1 = 0.0;  // -Pt(:,p), A fragments
        if (has_x) {
          double a0, a1, acc[2] = {0.0, 0.0};
          c2a(X[p][0], X[p][1], lane, a0, a1);
          dmma(acc, a0, lb0);
          dmma(acc, a1, lb1);
          X[p][0] = acc[0];
          X[p][1] = acc[1];
          c2a(-acc[0], -acc[1], lane, nx0, nx1);
        }
        if (coupled) {
          double a0, a1, acc[2] = {0.0, 0.0};
          c2a(G[p][0], G[p][1], lane, a0, a1);
          dmma(acc, a0, lb0);
          dmma(acc, a1, lb1);
          G[p][0] = acc[0];
          G[p][1] = acc[1];
          c2a(-acc[0], -acc[1], lane, ng0, ng1);
        }
        if (actY) {
          double a0, a1, acc[2] = {0.0, 0.0};
          c2a(Y[p][0], Y[p][1], lane, a0, a1);
          dmma(acc, a0, lb0);
          dmma(acc, a1, lb1);
          Y[p][0] = acc[0];
          Y[p][1] = acc[1];
          c2a(-acc[0], -acc[1], lane, ny0, ny1);
        }
#pragma unroll
        for (int c = p + 1; c < 8; ++c) {  // B = L_cp^T
          const double* q = DL + (8 * c + (lane >> 2)) * LD + 8 * p + (lane & 3);
          const double b0 = q[0], b1 = q[4];
          if (has_x) {
            dmma(X[c], nx0, b0);
            dmma(X[c], nx1, b1);
          }
          if (coupled) {
            dmma(G[c], ng0, b0);
            dmma(G[c], ng1, b1);
          }
          if (actY) {
            dmma(Y[c], ny0, b0);
            dmma(Y[c], ny1, b1);
          }
        }
      }
      if (b == 0 && lane == 0) BTD_SPROF(13, tstep);
      // ---- results: Pt1 / Pt2 -> XP, L_{j+1,j} = Pt1 -> Lsub, Linv = Pt3^T -> packed HBM ----
      const int rl = lane >> 2, r = 8 * b + rl;
      if (has_x) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<double2*>(XP + r * LD + c * 8 + 2 * (lane & 3)) = make_double2(X[c][0], X[c][1]);
        if (!last) {
          double* g = args.Lsub + (start + j) * bs;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int col = c * 8 + 2 * (lane & 3);
            if (r < n && col < n) g[(size_t)r * n + col] = X[c][0];
            if (r < n && col + 1 < n) g[(size_t)r * n + col + 1] = X[c][1];
          }
        }
      }
      if (coupled) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<double2*>(XP + (NT + r) * LD + c * 8 + 2 * (lane & 3)) = make_double2(G[c][0], G[c][1]);
      }
      {  // Pt3[r][c] = Linv[c][r]: packed row c holds columns 0..c (+ a zero pad for even c)
        double* g = args.Linv + (start + j) * (size_t)pk;
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int col = c * 8 + 2 * (lane & 3) + h;  // Linv row
            const int len = ((col + 2) >> 1) << 1;
            if (col < n && r < len) g[packed_offset_(col) + r] = (r <= col) ? Y[c][h] : 0.0;
          }
      }
      }
    }
    cp_async_wait_all();  // this thread's share of the DN prefetch
    __syncthreads();      // Pt1/Pt2 in XP, leaves consumed, DN landed
    if (s_fail) {
      if (tid == 0 && s_fail <= n) report_npd(args.err, args.level, j, k, s_fail);
      return;
    }
    // ======== phase 2 (all warps): D_{j+1} = A_{j+1,j+1} - Pt1 Pt1^T, or S_R at the last row ========
    if (!coupled && last) break;
    {
      // 36 8x8 tiles of the lower triangle, up to 3 per warp (ILP)
      double acc[3][2];
      int tr[3], tc[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        acc[q][0] = acc[q][1] = 0.0;
        const int u = warp + SS::NW * q;
        tr[q] = -1;
        if (u < 36) tri_decode(u, tr[q], tc[q]);
      }
#pragma unroll 4
      for (int k0 = 0; k0 < NT; k0 += 4) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          if (tr[q] < 0) continue;
          const double a = XP[(tr[q] * 8 + (lane >> 2)) * LD + k0 + (lane & 3)];
          const double bb = XP[(tc[q] * 8 + (lane >> 2)) * LD + k0 + (lane & 3)];
          dmma(acc[q], a, bb);
        }
      }
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        if (tr[q] < 0) continue;
        const int r = tr[q] * 8 + (lane >> 2);
        const int c = tc[q] * 8 + 2 * (lane & 3);
        if (!last) {
          const double* src = DN + r * LD + c;
          double* dst = DL + r * LD + c;
          dst[0] = (r == c && r >= n) ? 1.0 : src[0] - acc[q][0];
          dst[1] = (r == c + 1 && r >= n) ? 1.0 : src[1] - acc[q][1];
        } else if (r < n) {
          double* dst = args.Sr + (size_t)k * bs + (size_t)r * n;
          if (c < n) dst[c] = acc[q][0];
          if (c + 1 < n) dst[c + 1] = acc[q][1];
        }
      }
    }
    __syncthreads();  // DL = D_{j+1}; DN free
    if (tid == 0) BTD_SPROF(14, tstep);
    if (!last && j + 2 < J) {  // A_{j+2,j+2}, waited for one step later
      stage_block_async_part<NT, LD>(DN, args.diag + (start + j + 2) * bs, n, tid, SS::NTHREADS);
      cp_async_commit();
    }
  }
  if (!coupled) return;
  // ---- epilogue: the last row's S_L update and S_sub = -Y_R^T Y_L[last] ----
  if (warp >= 8) {
    for (int u = warp - 8; u < FactorShape<64>::NSL; u += SS::NW - 8) sl_tile64(XP, sl, n, J == 1, u, lane);
  } else {
    const int g = warp;  // 8 tiles of the fill product, one per warp
    double acc[8][2];
    fill_tile64(XP, g, acc, lane);
    const int r = 8 * g + (lane >> 2);
    double* ss = args.Ssub + (size_t)k * bs;
#pragma unroll
    for (int ct = 0; ct < 8; ++ct) {
      const int c = ct * 8 + 2 * (lane & 3);
      if (r < n) {
        if (c < n) ss[(size_t)c * n + r] = acc[ct][0];
        if (c + 1 < n) ss[(size_t)(c + 1) * n + r] = acc[ct][1];
      }
    }
  }
}

}  // namespace btd
