// Fused per-level segment elimination for n <= 64 (one CTA per interior segment).
//
// Replaces, for one recursion level, the reference chain
//   permute_split            bt/schur.py:98-138
//   factorize_btd_batch      bt/block_cholesky.py:24-42,60-68   (potrf / trsm / gemm sweeps)
//   _coupling_panels         bt/schur.py:141-153
//   solve_btd_batch(F)       bt/block_cholesky.py:45-57 via bt/schur.py:339-341
//   compute_schur            bt/schur.py:156-193
// with ONE launch.  Algorithm ("Y-form"): eliminate the segment rows in order,
// carrying the fill coupling G_j between the current row and the left separator:
//
//   Linv_j          = chol(D_j)^{-1}                       (stored; the solve only needs Linv, L_sub)
//   [P1 | P2]       = Linv_j [A_{j+1,j}^T | G_j]            (P1 = L_{j+1,j}^T, P2 = Y_L[j])
//   D_{j+1}         = A_{j+1,j+1} - P1^T P1
//   G_{j+1}         = -P1^T P2
//   S_L            += P2^T P2                              (Schur downdate of the left separator)
// and at the last row, with P1 := Linv C_R^T (= Y_R):
//   S_R = Y_R^T Y_R ,  S_sub = -Y_R^T Y_L[last]
// Everything lives in shared memory in transposed form Pt = [P1^T ; P2^T] so that every product is
// an "A row-major x B col-major" DMMA (mma.sync.m8n8k4.f64):  Pt = Xt Linv^T  and  C = Pt Pt^T.
// The lower triangle of C holds [D-update | G^T | S_L] at once.
#pragma once

#include "btd_device.cuh"

namespace btd {

#ifdef BTD_PHASE_PROF
__device__ unsigned long long g_phase_cycles[16];
#define BTD_PHASE_INIT() long long _ph_last = clock64();
#define BTD_PHASE(i)                                                        \
  do {                                                                      \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                              \
      long long _now = clock64();                                           \
      atomicAdd(&g_phase_cycles[i], (unsigned long long)(_now - _ph_last)); \
      _ph_last = _now;                                                      \
    }                                                                       \
  } while (0)
#else
#define BTD_PHASE_INIT()
#define BTD_PHASE(i)
#endif

struct FactorArgs {
  const double* diag;  // level matrix: (N, n, n)
  const double* sub;   // (N-1, n, n), sub[i] = A_{i+1,i}
  const int* seps;     // (K+1) separators of this level (unused for the base)
  long long N;
  int n;
  int K;        // segments (base: 1)
  int base;     // 1: serial base case, the whole chain is one uncoupled segment
  int level;
  double* Linv;  // (N, n, n) out: inverse Cholesky factor of every interior row
  double* Lsub;  // (N-1, n, n) out: L_{i,i-1} inside segments; coupling copies at segment edges
  double* Sl;    // (K, n, n) out: S_L per segment (written into the next level's diag slots)
  double* Sr;    // (K, n, n) out: S_R per segment
  double* Ssub;  // (K, n, n) out: next level sub block k = -Y_R^T Y_L[last]
  DevErr* err;
};

template <int NT>
struct FactorShape {
  static constexpr int LD = NT + 4;  // +4 doubles: conflict-free DMMA fragment loads
  static constexpr int NTHREADS = NT == 64 ? 256 : NT == 32 ? 128 : NT == 16 ? 64 : 32;
  static constexpr int NW = NTHREADS / 32;
  static constexpr int TS = NT == 8 ? 8 : 16;  // syrk warp tile
  static constexpr int SUB = TS / 8;
  static constexpr int TSR = 2 * NT / TS;
  static constexpr int HALF = TSR / 2;
  static constexpr int NSL = HALF * (HALF + 1) / 2;
  static constexpr int NG = HALF * HALF;
  static constexpr int ND = NSL;
  static constexpr int MAXSL = (NSL + NW - 1) / NW;
  static constexpr int MAXG = (NG + NW - 1) / NW;
  static constexpr int MAXD = (ND + NW - 1) / NW;
  static constexpr size_t SMEM = (size_t)3 * NT * LD * sizeof(double);
  static constexpr int MINB = NT == 64 ? 2 : NT == 32 ? 4 : 8;  // CTAs per SM to overlap pivot latency
  static_assert(NT / 8 == NW, "one trtri leaf per warp");
  static_assert(NTHREADS == 4 * NT, "potrf thread map: 8 panel columns x NT/2 row pairs");
};

__device__ __forceinline__ void tri_decode(int s, int& r, int& c) {
  r = 0;
  while ((r + 1) * (r + 2) / 2 <= s) ++r;
  c = s - r * (r + 1) / 2;
}

// Inverse of one 8x8 lower-triangular diagonal tile, in place (lanes 0..7: one column each).
// 1/L_ii was stored at DL[i][NT] by the panel factorization.
template <int NT>
__device__ __forceinline__ void leaf_inverse(double* DL, int d0, int lane) {
  constexpr int LD = FactorShape<NT>::LD;
  double x[8];
  if (lane < 8) {
    const int c = lane;
    double ri[8], row[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) ri[i] = DL[(d0 + i) * LD + NT];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = (i == c) ? ri[i] : 0.0;
#pragma unroll
    for (int i = 1; i < 8; ++i) {
#pragma unroll
      for (int mm = 0; mm < i; ++mm) row[mm] = DL[(d0 + i) * LD + d0 + mm];
      double s0 = 0.0, s1 = 0.0;  // x[mm] == 0 for mm < c, so no predicate is needed
#pragma unroll
      for (int mm = 0; mm < i; ++mm) {
        if (mm & 1)
          s1 = fma(row[mm], x[mm], s1);
        else
          s0 = fma(row[mm], x[mm], s0);
      }
      if (i > c) x[i] = -(s0 + s1) * ri[i];
    }
  }
  __syncwarp();
  if (lane < 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i) DL[(d0 + i) * LD + d0 + lane] = x[i];
  }
}

// ------------------------------------------------------------------------------------------
// In-place Cholesky + triangular inverse of the NT x NT tile DL (lower triangle is read).
// Returns the 1-based first non-positive pivot (reference _first_bad_pivot, bt/kernels.py:136-152;
// failure test is `pivot <= 0` like the LAPACK/OpenBLAS path, so NaN propagates silently, SURVEY
// §5), or 0.  The result is uniform across the CTA.
//
// Panel-blocked right-looking Cholesky.  Each 8-column panel is factored by ONE warp in
// registers (lane l owns panel rows p0+l and p0+l+32): the pivot chain is latency bound
// (shfl -> rsqrt -> fma per column), so it is kept short in instructions and leaves the issue
// slots to the co-resident CTA.  While warp 0 factors panel p, another warp inverts the
// 8x8 diagonal tile of panel p-1 (trtri leaf).  The trailing update of the lower 8x8 tiles is a
// batched DMMA rank-8 update by all warps; the inverse is finished by recursive doubling on DMMA.
// ------------------------------------------------------------------------------------------
template <int NT>
__device__ int potrf_trtri(double* DL) {
  using S = FactorShape<NT>;
  constexpr int LD = S::LD;
  constexpr int NW = S::NW;
  constexpr int NP = NT / 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ int s_fail;
  BTD_PHASE_INIT();
  __syncthreads();

  for (int p = 0; p < NP; ++p) {
    const int p0 = p * 8;
    if (warp == 0) {
      const int ra = p0 + lane, rb = p0 + lane + 32;
      const bool ha = ra < NT, hb = rb < NT;
      double va[8], vb[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        va[c] = ha ? DL[ra * LD + p0 + c] : 0.0;
        vb[c] = hb ? DL[rb * LD + p0 + c] : 0.0;
      }
      // Branch-free pivot chain: a data-dependent `break` here costs ~40% of the chain latency
      // (measured, tools/panel_bench.cu); a failed pivot only poisons values that are discarded.
      int fail = 0;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const double d = __shfl_sync(0xffffffffu, va[kk], kk);
        double lck[8];
#pragma unroll
        for (int c = kk + 1; c < 8; ++c) lck[c] = __shfl_sync(0xffffffffu, va[kk], c);
        fail = (fail == 0 && d <= 0.0) ? p0 + kk + 1 : fail;
        const double rinv = rsqrt(d);
        const double dinv = rinv * rinv;
#pragma unroll
        for (int c = kk + 1; c < 8; ++c) {
          va[c] = fma(-(va[kk] * lck[c]), dinv, va[c]);
          vb[c] = fma(-(vb[kk] * lck[c]), dinv, vb[c]);
        }
        va[kk] = (lane == kk) ? d * rinv : va[kk] * rinv;
        vb[kk] *= rinv;
        if (lane == kk) DL[(p0 + kk) * LD + NT] = rinv;  // 1 / L_kk for the inverse
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (ha) DL[ra * LD + p0 + c] = va[c];
        if (hb) DL[rb * LD + p0 + c] = vb[c];
      }
      if (lane == 0) s_fail = fail;
    } else if (NW > 1 && p > 0 && warp == 1 + (p - 1) % (NW > 1 ? NW - 1 : 1)) {
      leaf_inverse<NT>(DL, p0 - 8, lane);  // overlaps the pivot chain of panel p
    }
    __syncthreads();
    BTD_PHASE(10);
    if (s_fail) return s_fail;
    // trailing update of the lower 8x8 tiles right of the panel: A22 -= L21 L21^T (k = 8), batched
    const int m = NP - p - 1;
#ifdef BTD_EXP_NO_TRAILING
    const int units = 0;
#else
    const int units = m * (m + 1) / 2;
#endif
#pragma unroll 1
    for (int u = warp; u < units; u += NW) {
      int tr, tc;
      tri_decode(u, tr, tc);
      tr += p + 1;
      tc += p + 1;
      const double* pa = DL + (tr * 8 + (lane >> 2)) * LD + p0 + (lane & 3);
      const double* pb = DL + (tc * 8 + (lane >> 2)) * LD + p0 + (lane & 3);
      double acc[2] = {0.0, 0.0};
      dmma(acc, pa[0], pb[0]);
      dmma(acc, pa[4], pb[4]);
      double* dst = DL + (tr * 8 + (lane >> 2)) * LD + tc * 8 + 2 * (lane & 3);
      dst[0] -= acc[0];
      dst[1] -= acc[1];
    }
    __syncthreads();
    BTD_PHASE(11);
  }
  // remaining leaves: the last panel's (and all of them when the CTA has a single warp)
  for (int lf = (NW > 1 ? NP - 1 : 0) + warp; lf < NP; lf += NW) leaf_inverse<NT>(DL, lf * 8, lane);
  __syncthreads();
  BTD_PHASE(12);

  // ---- recursive doubling: [[A,0],[B,C]]^{-1} = [[Ai,0],[-Ci B Ai, Ci]] on DMMA ----
#pragma unroll
  for (int b = 8; 2 * b <= NT; b *= 2) {
    const int tpb = b / 8;
    const int units = (NT / (2 * b)) * tpb * tpb;
    constexpr int MAXV = (NT / 16 * 1 + NW - 1) / NW > 2 ? 2 : 2;  // <= 2 units per warp at every level
    // phase 1: T = B * Ainv   -> strictly-upper scratch block (rows i0.., cols i0+b..)
    {
      double acc[MAXV][2];
      int i0v[MAXV], trv[MAXV], tcv[MAXV];
      bool ok[MAXV];
#pragma unroll
      for (int q = 0; q < MAXV; ++q) {
        const int u = warp + q * NW;
        ok[q] = u < units;
        const int pair = u / (tpb * tpb), rem = u % (tpb * tpb);
        i0v[q] = pair * 2 * b;
        trv[q] = rem / tpb;
        tcv[q] = rem % tpb;
        acc[q][0] = acc[q][1] = 0.0;
      }
      for (int k0 = 0; k0 < b; k0 += 4) {
#pragma unroll
        for (int q = 0; q < MAXV; ++q) {
          if (!ok[q] || k0 < tcv[q] * 8) continue;  // Ainv[k][c] == 0 for k < c
          const int i0 = i0v[q];
          const double a = DL[(i0 + b + trv[q] * 8 + (lane >> 2)) * LD + i0 + k0 + (lane & 3)];
          const double bb = DL[(i0 + k0 + (lane & 3)) * LD + i0 + tcv[q] * 8 + (lane >> 2)];
          dmma(acc[q], a, bb);
        }
      }
#pragma unroll
      for (int q = 0; q < MAXV; ++q) {
        if (!ok[q]) continue;
        const int i0 = i0v[q];
        double* dst = DL + (i0 + trv[q] * 8 + (lane >> 2)) * LD + i0 + b + tcv[q] * 8 + 2 * (lane & 3);
        dst[0] = acc[q][0];
        dst[1] = acc[q][1];
      }
    }
    __syncthreads();
    // phase 2: B <- -Cinv * T
    {
      double acc[MAXV][2];
      int i0v[MAXV], trv[MAXV], tcv[MAXV];
      bool ok[MAXV];
#pragma unroll
      for (int q = 0; q < MAXV; ++q) {
        const int u = warp + q * NW;
        ok[q] = u < units;
        const int pair = u / (tpb * tpb), rem = u % (tpb * tpb);
        i0v[q] = pair * 2 * b;
        trv[q] = rem / tpb;
        tcv[q] = rem % tpb;
        acc[q][0] = acc[q][1] = 0.0;
      }
      for (int k0 = 0; k0 < b; k0 += 4) {
#pragma unroll
        for (int q = 0; q < MAXV; ++q) {
          if (!ok[q] || k0 > trv[q] * 8 + 4) continue;  // Cinv[r][k] == 0 for k > r
          const int i0 = i0v[q];
          const double a = DL[(i0 + b + trv[q] * 8 + (lane >> 2)) * LD + i0 + b + k0 + (lane & 3)];
          const double bb = DL[(i0 + k0 + (lane & 3)) * LD + i0 + b + tcv[q] * 8 + (lane >> 2)];
          dmma(acc[q], a, bb);
        }
      }
#pragma unroll
      for (int q = 0; q < MAXV; ++q) {
        if (!ok[q]) continue;
        const int i0 = i0v[q];
        double* dst = DL + (i0 + b + trv[q] * 8 + (lane >> 2)) * LD + i0 + tcv[q] * 8 + 2 * (lane & 3);
        dst[0] = -acc[q][0];
        dst[1] = -acc[q][1];
      }
    }
    __syncthreads();
  }
  BTD_PHASE(13);
  return 0;
}

// Pt = Xt * Linv^T, in place on the XP rows owned by this warp (16 rows per warp, two 8-row passes:
// a pass reads only its own rows, so it can overwrite them after a __syncwarp).
template <int NT>
__device__ __forceinline__ void pt_gemm(double* XP, const double* DL, bool coupled, int warp, int lane) {
  using S = FactorShape<NT>;
  constexpr int LD = S::LD;
  constexpr int NCT = NT / 8;
  const int row0 = warp * 16;
  if (!coupled && row0 >= NT) return;
  const double* pb = DL + (lane >> 2) * LD + (lane & 3);
#pragma unroll 1
  for (int rt = 0; rt < 2; ++rt) {
    double acc[NCT][2];
#pragma unroll
    for (int c = 0; c < NCT; ++c) acc[c][0] = acc[c][1] = 0.0;
    const double* pa = XP + (row0 + rt * 8 + (lane >> 2)) * LD + (lane & 3);
#pragma unroll
    for (int k0 = 0; k0 < NT; k0 += 4) {
      const double a0 = pa[k0];
#pragma unroll
      for (int ct = 0; ct < NCT; ++ct) {
        if (ct * 8 + 7 < k0) continue;  // Linv[c][k] == 0 for k > c
        dmma(acc[ct], a0, pb[ct * 8 * LD + k0]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int ct = 0; ct < NCT; ++ct) {
      double2 v;
      v.x = acc[ct][0];
      v.y = acc[ct][1];
      *reinterpret_cast<double2*>(XP + (row0 + rt * 8 + (lane >> 2)) * LD + ct * 8 + 2 * (lane & 3)) = v;
    }
  }
}

// acc += Pt[R-tile] * Pt[C-tile]^T over k = 0..NT (one TS x TS warp tile of the lower 2NT x 2NT product)
template <int NT>
__device__ __forceinline__ void syrk_tile(const double* XP, int R, int C, double (&acc)[FactorShape<NT>::SUB][FactorShape<NT>::SUB][2],
                                          int lane) {
  using S = FactorShape<NT>;
  constexpr int LD = S::LD, TS = S::TS, SUB = S::SUB;
  const bool diag = (R == C);
  const double* pa = XP + (R * TS + (lane >> 2)) * LD + (lane & 3);
  const double* pb = XP + (C * TS + (lane >> 2)) * LD + (lane & 3);
#pragma unroll 4
  for (int k0 = 0; k0 < NT; k0 += 4) {
    double a[SUB], b[SUB];
#pragma unroll
    for (int i = 0; i < SUB; ++i) {
      a[i] = pa[i * 8 * LD + k0];
      b[i] = pb[i * 8 * LD + k0];
    }
#pragma unroll
    for (int i = 0; i < SUB; ++i)
#pragma unroll
      for (int jj = 0; jj < SUB; ++jj)
        if (!diag || jj <= i) dmma(acc[i][jj], a[i], b[jj]);
  }
}

template <int NT>
__global__ void __launch_bounds__(FactorShape<NT>::NTHREADS, FactorShape<NT>::MINB)
    factor_level_kernel(FactorArgs args) {
  using S = FactorShape<NT>;
  constexpr int LD = S::LD, NTHREADS = S::NTHREADS, NW = S::NW, TS = S::TS, SUB = S::SUB;
  constexpr int HALF = S::HALF, NSL = S::NSL, NG = S::NG, ND = S::ND;
  extern __shared__ __align__(16) double smem[];
  double* XP = smem;                // 2NT x LD : [X1 | Pt1] rows 0..NT-1, [Gt | Pt2] rows NT..2NT-1
  double* DL = smem + 2 * NT * LD;  // NT x LD  : D -> L -> Linv

  if (error_raised(args.err)) return;
  const int k = blockIdx.x;
  const bool coupled = !args.base;
  const long long start = coupled ? (long long)args.seps[k] + 1 : 0;
  const long long stop = coupled ? (long long)args.seps[k + 1] : args.N;
  const int J = (int)(stop - start);
  const int n = args.n;
  const size_t bs = (size_t)n * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- prologue: D_0, X1_0 (A_{1,0} or C_R), Gt_0 = C_L^T ----
  stage_block_async<NT, LD, NTHREADS>(DL, args.diag + start * bs, n);
  if (J > 1)
    stage_block_async<NT, LD, NTHREADS>(XP, args.sub + start * bs, n);
  else if (coupled)
    stage_block_async<NT, LD, NTHREADS>(XP, args.sub + (stop - 1) * bs, n);
  cp_async_commit();
  if (coupled) {
    stage_block_transposed<NT, LD, NTHREADS>(XP + NT * LD, args.sub + (start - 1) * bs, n);
    copy_block<NTHREADS>(args.Lsub + (start - 1) * bs, args.sub + (start - 1) * bs, n);  // C_L
    copy_block<NTHREADS>(args.Lsub + (stop - 1) * bs, args.sub + (stop - 1) * bs, n);    // C_R
  }
  cp_async_wait_all();
  for (int r = n + tid; r < NT; r += NTHREADS) DL[r * LD + r] = 1.0;
  BTD_PHASE_INIT();

  for (int j = 0; j < J; ++j) {
    const bool last = (j == J - 1);
    BTD_PHASE(0);
    const int piv = potrf_trtri<NT>(DL);  // begins with a barrier
    BTD_PHASE(1);
    if (piv) {
      if (tid == 0 && piv <= n) report_npd(args.err, args.level, j, k, piv);
      return;
    }
    store_block<NT, LD, NTHREADS>(args.Linv + (start + j) * bs, DL, n, true);
    if (last && !coupled) break;

    cp_async_wait_all();
    __syncthreads();
    BTD_PHASE(2);
    pt_gemm<NT>(XP, DL, coupled, warp, lane);
    __syncthreads();
    BTD_PHASE(3);
    if (!last) {
      store_block<NT, LD, NTHREADS>(args.Lsub + (start + j) * bs, XP, n, false);  // L_{j+1,j}
      stage_block_async<NT, LD, NTHREADS>(DL, args.diag + (start + j + 1) * bs, n);
      cp_async_commit();
    }

    BTD_PHASE(4);
    // ---- C = Pt Pt^T (lower): S_L tiles (persistent) and G tiles (held until XP is free) ----
    double held[S::MAXG][SUB][SUB][2];
    if (coupled) {
      // S_L accumulates across the segment's steps in its global output slot (L2 resident):
      // keeping it in registers would cost 32 registers for the whole kernel.
#pragma unroll
      for (int s = 0; s < S::MAXSL; ++s) {
        const int t = warp + s * NW;
        if (t < NSL) {
          int rr, cc;
          tri_decode(t, rr, cc);
          double acc[SUB][SUB][2];
#pragma unroll
          for (int i = 0; i < SUB; ++i)
#pragma unroll
            for (int jj = 0; jj < SUB; ++jj) {
              const int r = rr * TS + i * 8 + (lane >> 2);
              const int c = cc * TS + jj * 8 + 2 * (lane & 3);
              const double* src = args.Sl + (size_t)k * bs + (size_t)r * n + c;
              acc[i][jj][0] = (j > 0 && r < n && c < n) ? src[0] : 0.0;
              acc[i][jj][1] = (j > 0 && r < n && c + 1 < n) ? src[1] : 0.0;
            }
          syrk_tile<NT>(XP, HALF + rr, HALF + cc, acc, lane);
#pragma unroll
          for (int i = 0; i < SUB; ++i)
#pragma unroll
            for (int jj = 0; jj < SUB; ++jj) {
              if (rr == cc && jj > i) continue;
              const int r = rr * TS + i * 8 + (lane >> 2);
              const int c = cc * TS + jj * 8 + 2 * (lane & 3);
              double* dst = args.Sl + (size_t)k * bs + (size_t)r * n + c;
              if (r < n && c < n) dst[0] = acc[i][jj][0];
              if (r < n && c + 1 < n) dst[1] = acc[i][jj][1];
            }
        }
      }
#pragma unroll
      for (int s = 0; s < S::MAXG; ++s) {
        const int g = ((warp - NSL % NW + NW) % NW) + s * NW;
#pragma unroll
        for (int i = 0; i < SUB; ++i)
#pragma unroll
          for (int jj = 0; jj < SUB; ++jj) held[s][i][jj][0] = held[s][i][jj][1] = 0.0;
        if (g < NG) syrk_tile<NT>(XP, HALF + g / HALF, g % HALF, held[s], lane);
      }
    }
    BTD_PHASE(5);
    cp_async_wait_all();
    __syncthreads();
    BTD_PHASE(6);
    // ---- D tiles: D_{j+1} = A_{j+1,j+1} - P1^T P1  (or S_R at the last row) ----
#pragma unroll
    for (int s = 0; s < S::MAXD; ++s) {
      const int dd = ((warp - (NSL + NG) % NW + NW) % NW) + s * NW;
      if (dd < ND) {
        int rr, cc;
        tri_decode(dd, rr, cc);
        double acc[SUB][SUB][2];
#pragma unroll
        for (int i = 0; i < SUB; ++i)
#pragma unroll
          for (int jj = 0; jj < SUB; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
        syrk_tile<NT>(XP, rr, cc, acc, lane);
#pragma unroll
        for (int i = 0; i < SUB; ++i)
#pragma unroll
          for (int jj = 0; jj < SUB; ++jj) {
            if (rr == cc && jj > i) continue;
            const int r = rr * TS + i * 8 + (lane >> 2);
            const int c = cc * TS + jj * 8 + 2 * (lane & 3);
            if (!last) {
              double* dst = DL + r * LD + c;
              dst[0] = (r == c && r >= n) ? 1.0 : dst[0] - acc[i][jj][0];
              dst[1] = (r == c + 1 && r >= n) ? 1.0 : dst[1] - acc[i][jj][1];
            } else if (r < n) {
              double* dst = args.Sr + (size_t)k * bs + (size_t)r * n;
              if (c < n) dst[c] = acc[i][jj][0];
              if (c + 1 < n) dst[c + 1] = acc[i][jj][1];
            }
          }
      }
    }
    BTD_PHASE(7);
    __syncthreads();  // every read of XP (Pt) is complete
    BTD_PHASE(8);
    if (coupled) {
#pragma unroll
      for (int s = 0; s < S::MAXG; ++s) {
        const int g = ((warp - NSL % NW + NW) % NW) + s * NW;
        if (g >= NG) continue;
        const int R = HALF + g / HALF, C = g % HALF;
#pragma unroll
        for (int i = 0; i < SUB; ++i)
#pragma unroll
          for (int jj = 0; jj < SUB; ++jj) {
            const int r = R * TS + i * 8 + (lane >> 2);  // in [NT, 2NT)
            const int c = C * TS + jj * 8 + 2 * (lane & 3);
            if (!last) {
              XP[r * LD + c] = -held[s][i][jj][0];
              XP[r * LD + c + 1] = -held[s][i][jj][1];
            } else {
              // S_sub (row s_{k+1}, col s_k) = -Y_R^T Y_L  = transpose of the held -Y_L^T Y_R
              const int rr = r - NT;
              if (rr < n) {
                if (c < n) args.Ssub[(size_t)k * bs + (size_t)c * n + rr] = -held[s][i][jj][0];
                if (c + 1 < n) args.Ssub[(size_t)k * bs + (size_t)(c + 1) * n + rr] = -held[s][i][jj][1];
              }
            }
          }
      }
    }
    if (!last) {
      if (j + 1 < J - 1)
        stage_block_async<NT, LD, NTHREADS>(XP, args.sub + (start + j + 1) * bs, n);
      else if (coupled)
        stage_block_async<NT, LD, NTHREADS>(XP, args.sub + (stop - 1) * bs, n);  // C_R -> Y_R
      cp_async_commit();
    }
  }

}

// Next-level diagonal: S_diag[p] = (A[s_p] - S_L[p]) - S_R[p-1]  (reference order, bt/schur.py:186-188).
// S_L[p] already sits in next_diag[p]; only the lower triangle is formed (the kernels never read
// the upper triangle of a diagonal block).
__global__ void assemble_schur_diag_kernel(const double* diag, const int* seps, double* next_diag,
                                           const double* Sr, int K, int n, const DevErr* err) {
  if (error_raised(err)) return;
  const int p = blockIdx.x;
  const size_t bs = (size_t)n * n;
  const double* a = diag + (size_t)seps[p] * bs;
  double* out = next_diag + (size_t)p * bs;
  const double* sr = p > 0 ? Sr + (size_t)(p - 1) * bs : nullptr;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int r = e / n, c = e % n;
    if (c > r) continue;
    double v = a[e];
    if (p < K) v -= out[e];
    if (sr) v -= sr[e];
    out[e] = v;
  }
}

__global__ void fill_separators_kernel(int* seps, int P, int N, int step) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < P) seps[k] = (k == P - 1) ? N - 1 : k * step;
}

__global__ void init_err_kernel(DevErr* err) {
  err->key = kNoErr;
  err->level = 0x7fffffff;
  err->pad = 0;
}

}  // namespace btd
