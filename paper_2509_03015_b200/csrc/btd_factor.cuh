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
  static_assert(NT / 8 == NW, "one trtri leaf per warp");
};

__device__ __forceinline__ void tri_decode(int s, int& r, int& c) {
  r = 0;
  while ((r + 1) * (r + 2) / 2 <= s) ++r;
  c = s - r * (r + 1) / 2;
}

// ------------------------------------------------------------------------------------------
// In-place Cholesky + triangular inverse of the NT x NT tile DL (lower triangle is read).
// Panel-blocked (8 columns): unblocked elimination inside the panel, DMMA trailing update.
// Returns the 1-based first non-positive pivot (reference _first_bad_pivot, bt/kernels.py:136-152;
// failure test is `pivot <= 0` like the LAPACK/OpenBLAS path, so NaN propagates silently),
// or 0. The result is uniform across the CTA.
// ------------------------------------------------------------------------------------------
template <int NT>
__device__ int potrf_trtri(double* DL) {
  using S = FactorShape<NT>;
  constexpr int LD = S::LD;
  constexpr int NTHREADS = S::NTHREADS;
  constexpr int NW = S::NW;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (int p = 0; p < NT / 8; ++p) {
    const int p0 = p * 8;
    double sprev = 1.0;
    for (int kk = 0; kk < 8; ++kk) {
      const int k = p0 + kk;
      __syncthreads();
      const double d = DL[k * LD + k];
      // deferred scaling of the previous panel column (nobody reads it in this phase)
      if (kk > 0) {
        const double rs = 1.0 / sprev;
        for (int i = k - 1 + tid; i < NT; i += NTHREADS)
          DL[i * LD + k - 1] = (i == k - 1) ? sprev : DL[i * LD + k - 1] * rs;
      }
      if (d <= 0.0) return k + 1;
      const double dinv = 1.0 / d;
      // update the panel columns c in (k, p0+8), rows i >= c
      const int ncols = p0 + 7 - k;  // columns k+1 .. p0+7
      if (ncols > 0) {
        const int nrows = NT - k - 1;  // rows k+1 .. NT-1
        for (int e = tid; e < nrows * ncols; e += NTHREADS) {
          const int i = k + 1 + e / ncols;
          const int c = k + 1 + e % ncols;
          if (c <= i) DL[i * LD + c] -= DL[i * LD + k] * DL[c * LD + k] * dinv;
        }
      }
      sprev = sqrt(d);
    }
    __syncthreads();
    {
      const int k = p0 + 7;
      const double rs = 1.0 / sprev;
      for (int i = k + tid; i < NT; i += NTHREADS) DL[i * LD + k] = (i == k) ? sprev : DL[i * LD + k] * rs;
    }
    __syncthreads();
    // trailing update of the lower 8x8 tiles right of the panel: A22 -= L21 L21^T (k = 8)
    const int m = NT / 8 - p - 1;
    const int units = m * (m + 1) / 2;
    for (int u = warp; u < units; u += NW) {
      int tr, tc;
      tri_decode(u, tr, tc);
      tr += p + 1;
      tc += p + 1;
      double acc[2] = {0.0, 0.0};
#pragma unroll
      for (int ks = 0; ks < 8; ks += 4) {
        const double a = DL[(tr * 8 + (lane >> 2)) * LD + p0 + ks + (lane & 3)];
        const double b = DL[(tc * 8 + (lane >> 2)) * LD + p0 + ks + (lane & 3)];
        dmma(acc, a, b);
      }
      double* dst = DL + (tr * 8 + (lane >> 2)) * LD + tc * 8 + 2 * (lane & 3);
      dst[0] -= acc[0];
      dst[1] -= acc[1];
    }
  }
  __syncthreads();

  // ---- triangular inverse: 8x8 leaves (one warp each), then recursive doubling with DMMA ----
  {
    const int d0 = warp * 8;
    double x[8];
    if (lane < 8) {
      const int c = lane;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i < c) {
          x[i] = 0.0;
        } else if (i == c) {
          x[i] = 1.0 / DL[(d0 + i) * LD + d0 + i];
        } else {
          double s = 0.0;
#pragma unroll
          for (int mm = 0; mm < i; ++mm)
            if (mm >= c) s += DL[(d0 + i) * LD + d0 + mm] * x[mm];
          x[i] = -s / DL[(d0 + i) * LD + d0 + i];
        }
      }
    }
    __syncwarp();
    if (lane < 8) {
#pragma unroll
      for (int i = 0; i < 8; ++i) DL[(d0 + i) * LD + d0 + lane] = x[i];
    }
  }
  __syncthreads();
#pragma unroll
  for (int b = 8; 2 * b <= NT; b *= 2) {
    const int tpb = b / 8;
    const int units = (NT / (2 * b)) * tpb * tpb;
    // phase 1: T = B * Ainv   -> strictly-upper scratch block (rows i0.., cols i0+b..)
    for (int u = warp; u < units; u += NW) {
      const int pair = u / (tpb * tpb), rem = u % (tpb * tpb), tr = rem / tpb, tc = rem % tpb;
      const int i0 = pair * 2 * b;
      double acc[2] = {0.0, 0.0};
      for (int k0 = tc * 8; k0 < b; k0 += 4) {
        const double a = DL[(i0 + b + tr * 8 + (lane >> 2)) * LD + i0 + k0 + (lane & 3)];
        const double bb = DL[(i0 + k0 + (lane & 3)) * LD + i0 + tc * 8 + (lane >> 2)];
        dmma(acc, a, bb);
      }
      double* dst = DL + (i0 + tr * 8 + (lane >> 2)) * LD + i0 + b + tc * 8 + 2 * (lane & 3);
      dst[0] = acc[0];
      dst[1] = acc[1];
    }
    __syncthreads();
    // phase 2: B <- -Cinv * T
    for (int u = warp; u < units; u += NW) {
      const int pair = u / (tpb * tpb), rem = u % (tpb * tpb), tr = rem / tpb, tc = rem % tpb;
      const int i0 = pair * 2 * b;
      double acc[2] = {0.0, 0.0};
      for (int k0 = 0; k0 <= tr * 8 + 4; k0 += 4) {
        const double a = DL[(i0 + b + tr * 8 + (lane >> 2)) * LD + i0 + b + k0 + (lane & 3)];
        const double bb = DL[(i0 + k0 + (lane & 3)) * LD + i0 + b + tc * 8 + (lane >> 2)];
        dmma(acc, a, bb);
      }
      double* dst = DL + (i0 + b + tr * 8 + (lane >> 2)) * LD + i0 + tc * 8 + 2 * (lane & 3);
      dst[0] = -acc[0];
      dst[1] = -acc[1];
    }
    __syncthreads();
  }
  return 0;
}

// Pt = Xt * Linv^T, in place on the XP rows owned by this warp (16 rows per warp).
template <int NT>
__device__ __forceinline__ void pt_gemm(double* XP, const double* DL, bool coupled, int warp, int lane) {
  using S = FactorShape<NT>;
  constexpr int LD = S::LD;
  constexpr int NCT = NT / 8;
  const int row0 = warp * 16;
  if (!coupled && row0 >= NT) return;
  double acc[2][NCT][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int c = 0; c < NCT; ++c) acc[i][c][0] = acc[i][c][1] = 0.0;
  const double* pa = XP + (row0 + (lane >> 2)) * LD + (lane & 3);
  const double* pb = DL + (lane >> 2) * LD + (lane & 3);
#pragma unroll
  for (int k0 = 0; k0 < NT; k0 += 4) {
    const double a0 = pa[k0];
    const double a1 = pa[8 * LD + k0];
#pragma unroll
    for (int ct = 0; ct < NCT; ++ct) {
      if (ct * 8 + 7 < k0) continue;  // Linv[c][k] == 0 for k > c
      const double b = pb[ct * 8 * LD + k0];
      dmma(acc[0][ct], a0, b);
      dmma(acc[1][ct], a1, b);
    }
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int ct = 0; ct < NCT; ++ct) {
      double2 v;
      v.x = acc[i][ct][0];
      v.y = acc[i][ct][1];
      *reinterpret_cast<double2*>(XP + (row0 + i * 8 + (lane >> 2)) * LD + ct * 8 + 2 * (lane & 3)) = v;
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
#pragma unroll
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
__global__ void __launch_bounds__(FactorShape<NT>::NTHREADS) factor_level_kernel(FactorArgs args) {
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

  double acc_sl[S::MAXSL][SUB][SUB][2];
#pragma unroll
  for (int s = 0; s < S::MAXSL; ++s)
#pragma unroll
    for (int i = 0; i < SUB; ++i)
#pragma unroll
      for (int jj = 0; jj < SUB; ++jj) acc_sl[s][i][jj][0] = acc_sl[s][i][jj][1] = 0.0;

  for (int j = 0; j < J; ++j) {
    const bool last = (j == J - 1);
    const int piv = potrf_trtri<NT>(DL);  // begins with a barrier
    if (piv) {
      if (tid == 0 && piv <= n) report_npd(args.err, args.level, j, k, piv);
      return;
    }
    store_block<NT, LD, NTHREADS>(args.Linv + (start + j) * bs, DL, n, true);
    if (last && !coupled) break;

    cp_async_wait_all();
    __syncthreads();
    pt_gemm<NT>(XP, DL, coupled, warp, lane);
    __syncthreads();
    if (!last) {
      store_block<NT, LD, NTHREADS>(args.Lsub + (start + j) * bs, XP, n, false);  // L_{j+1,j}
      stage_block_async<NT, LD, NTHREADS>(DL, args.diag + (start + j + 1) * bs, n);
      cp_async_commit();
    }

    // ---- C = Pt Pt^T (lower): S_L tiles (persistent) and G tiles (held until XP is free) ----
    double held[S::MAXG][SUB][SUB][2];
    if (coupled) {
#pragma unroll
      for (int s = 0; s < S::MAXSL; ++s) {
        const int t = warp + s * NW;
        if (t < NSL) {
          int rr, cc;
          tri_decode(t, rr, cc);
          syrk_tile<NT>(XP, HALF + rr, HALF + cc, acc_sl[s], lane);
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
    cp_async_wait_all();
    __syncthreads();
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
    __syncthreads();  // every read of XP (Pt) is complete
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

  if (coupled) {
#pragma unroll
    for (int s = 0; s < S::MAXSL; ++s) {
      const int t = warp + s * NW;
      if (t >= NSL) continue;
      int rr, cc;
      tri_decode(t, rr, cc);
#pragma unroll
      for (int i = 0; i < SUB; ++i)
#pragma unroll
        for (int jj = 0; jj < SUB; ++jj) {
          if (rr == cc && jj > i) continue;
          const int r = rr * TS + i * 8 + (lane >> 2);
          const int c = cc * TS + jj * 8 + 2 * (lane & 3);
          if (r < n) {
            double* dst = args.Sl + (size_t)k * bs + (size_t)r * n;
            if (c < n) dst[c] = acc_sl[s][i][jj][0];
            if (c + 1 < n) dst[c + 1] = acc_sl[s][i][jj][1];
          }
        }
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
