// Level solve for n > 64 with few right-hand sides (d <= 4): one 256-thread CTA per segment and
// DC-column chunk, matrix blocks read straight from global memory (coalesced rows / columns),
// vectors in shared memory.  Same step algebra as btd_solve.cuh / btd_solve2.cuh:
//   down : forward z_j = Linv_j (b_j - L_{j,j-1} z_{j-1}); backward w_j = Linv_j^T (z_j - L_{j+1,j}^T
//          w_{j+1}); fold f_R = C_R w_last, f_L = C_L^T w_0           (bt/schur.py:230-260)
//   up   : b_0 -= C_L x_L, b_last -= C_R^T x_R, the same sweeps, x in the original order, separator
//          rows copied from the level below                            (bt/schur.py:214-227,263-286)
//   base : one uncoupled chain                                         (bt/block_cholesky.py:95-98)
// The tiled path (btd_big.cuh) stores Linv full (n x n, zero upper triangle).  With d <= 4 its tile
// GEMMs would fill 1-4 of 64 output columns; this kernel does matrix-vector work at the rate the
// blocks stream in.  z_j is parked in x (down: scratch; up/base: overwritten by w_j).
#pragma once

#include "btd_device.cuh"
#include "btd_solve.cuh"

namespace btd {

constexpr int kWideThreads = 256;

// y[r][c] (+)= sign * sum_{m} M[r][m] x[m][c]  (row form: warp per row, lanes over m, xor reduce);
// LOWER: M[r][m] == 0 for m > r (skipped)
template <int DC, bool LOWER>
__device__ __forceinline__ void wide_mv_rows(const double* __restrict__ M, int n, const double* x, double* y, double sign,
                                             bool accumulate) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = warp; r < n; r += kWideThreads / 32) {
    const double* row = M + (size_t)r * n;
    const int lim = LOWER ? r + 1 : n;
    double s[DC];
#pragma unroll
    for (int c = 0; c < DC; ++c) s[c] = 0.0;
    for (int m = lane; m < lim; m += 32) {
      const double v = __ldg(row + m);
#pragma unroll
      for (int c = 0; c < DC; ++c) s[c] = fma(v, x[m * DC + c], s[c]);
    }
#pragma unroll
    for (int c = 0; c < DC; ++c) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s[c] += __shfl_xor_sync(0xffffffffu, s[c], o);
      if (lane == 0) y[r * DC + c] = accumulate ? fma(sign, s[c], y[r * DC + c]) : sign * s[c];
    }
  }
}

// y[c][.] (+)= sign * sum_r M[r][c] x[r][.]  (column form: thread per column, coalesced rows);
// LOWER: M[r][c] == 0 for r < c (skipped)
template <int DC, bool LOWER>
__device__ __forceinline__ void wide_mv_cols(const double* __restrict__ M, int n, const double* x, double* y, double sign,
                                             bool accumulate) {
  for (int c = threadIdx.x; c < n; c += kWideThreads) {
    double s[4][DC];  // four interleaved partial sums: the row loop is a latency chain otherwise
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < DC; ++q) s[i][q] = 0.0;
    int r = LOWER ? c : 0;
    for (; r + 3 < n; r += 4) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double v = __ldg(M + (size_t)(r + i) * n + c);
#pragma unroll
        for (int q = 0; q < DC; ++q) s[i][q] = fma(v, x[(r + i) * DC + q], s[i][q]);
      }
    }
    for (; r < n; ++r) {
      const double v = __ldg(M + (size_t)r * n + c);
#pragma unroll
      for (int q = 0; q < DC; ++q) s[0][q] = fma(v, x[r * DC + q], s[0][q]);
    }
#pragma unroll
    for (int q = 0; q < DC; ++q) {
      const double t = (s[0][q] + s[1][q]) + (s[2][q] + s[3][q]);
      y[c * DC + q] = accumulate ? fma(sign, t, y[c * DC + q]) : sign * t;
    }
  }
}

template <int DC>
__global__ void __launch_bounds__(kWideThreads) solve_wide_kernel(SolveArgs a) {
  extern __shared__ __align__(16) double sw[];
  const int n = a.n, d = a.d, mode = a.mode;
  double* t = sw;              // n x DC
  double* u = t + n * DC;      // n x DC: z_{j-1} (forward) / w_{j+1} (backward)
  double* c0v = u + n * DC;    // up: C_L x_L
  double* c1v = c0v + n * DC;  // up: C_R^T x_R
  double* xs = c1v + n * DC;   // separator rhs / solution panel
  if (error_raised(a.err)) return;
  const bool base = mode == kSolveBase;
  const int k = base ? 0 : blockIdx.x;
  const int col0 = blockIdx.y * DC, dc = min(DC, d - col0);
  const long long start = base ? 0 : (long long)a.seps[k] + 1;
  const long long stop = base ? a.N : (long long)a.seps[k + 1];
  const int J = (int)(stop - start);
  const size_t bs = (size_t)n * n, ps = (size_t)n * d;
  const int tid = threadIdx.x;
  auto load_panel = [&](double* dst, const double* src) {  // n x dc rows of a (., n, d) panel
    for (int e = tid; e < n * DC; e += kWideThreads) {
      const int r = e / DC, c = e % DC;
      dst[e] = c < dc ? src[(size_t)r * d + col0 + c] : 0.0;
    }
  };
  auto store_panel = [&](double* dst, const double* src) {
    for (int e = tid; e < n * DC; e += kWideThreads) {
      const int r = e / DC, c = e % DC;
      if (c < dc) dst[(size_t)r * d + col0 + c] = src[e];
    }
  };
  if (mode == kSolveUp) {  // boundary corrections and the separator rows of the solution
    load_panel(xs, a.xsep + (size_t)k * ps);
    __syncthreads();
    wide_mv_rows<DC, false>(a.Lsub + (size_t)(start - 1) * bs, n, xs, c0v, 1.0, false);  // C_L x_L
    store_panel(a.x + (size_t)(start - 1) * ps, xs);
    __syncthreads();
    load_panel(xs, a.xsep + (size_t)(k + 1) * ps);
    __syncthreads();
    wide_mv_cols<DC, false>(a.Lsub + (size_t)(stop - 1) * bs, n, xs, c1v, 1.0, false);  // C_R^T x_R
    if (k == a.K - 1) store_panel(a.x + (size_t)stop * ps, xs);
    __syncthreads();
  }
  // ---- forward sweep ----
  for (int j = 0; j < J; ++j) {
    const long long row = start + j;
    load_panel(t, a.rhs + row * ps);
    if (mode == kSolveUp) {
      __syncthreads();
      for (int e = tid; e < n * DC; e += kWideThreads) {
        if (j == 0) t[e] -= c0v[e];
        if (j == J - 1) t[e] -= c1v[e];
      }
    }
    __syncthreads();
    if (j > 0) {
      wide_mv_rows<DC, false>(a.Lsub + (size_t)(row - 1) * bs, n, u, t, -1.0, true);
      __syncthreads();
    }
    wide_mv_rows<DC, true>(a.Linv + (size_t)row * bs, n, t, u, 1.0, false);  // z_j -> u
    __syncthreads();
    store_panel(a.x + row * ps, u);
  }
  // ---- backward sweep ----
  for (int j = J - 1; j >= 0; --j) {
    const long long row = start + j;
    if (j < J - 1) {  // t = z_j - L_{j+1,j}^T w_{j+1}
      load_panel(t, a.x + row * ps);
      __syncthreads();
      wide_mv_cols<DC, false>(a.Lsub + (size_t)row * bs, n, u, t, -1.0, true);
    } else {
      for (int e = tid; e < n * DC; e += kWideThreads) t[e] = u[e];  // z_{J-1} is still in u
    }
    __syncthreads();
    wide_mv_cols<DC, true>(a.Linv + (size_t)row * bs, n, t, u, 1.0, false);  // w_j -> u
    __syncthreads();
    if (mode != kSolveDown) store_panel(a.x + row * ps, u);
    if (mode == kSolveDown && j == J - 1) {  // f_R = C_R w_last
      wide_mv_rows<DC, false>(a.Lsub + (size_t)(stop - 1) * bs, n, u, xs, 1.0, false);
      __syncthreads();
      store_panel(a.fr + (size_t)k * ps, xs);
      __syncthreads();
    }
  }
  if (mode == kSolveDown) {  // f_L = C_L^T w_0
    wide_mv_cols<DC, false>(a.Lsub + (size_t)(start - 1) * bs, n, u, xs, 1.0, false);
    __syncthreads();
    store_panel(a.fl + (size_t)k * ps, xs);
  }
}


// ============================================================================================
// solve_dmma_kernel: the same level / base solve for n > 64 (multiples of 64) with 5 <= d <= 8
// (dispatch: use_wide_solve, btd_capi.cu), one 256-thread CTA per (segment, 8-column slice) --
// grid (ceil(d / 8), segments).  Each
// block product  y (n x 8) = M x  or  M^T x  runs on DMMA with M's fragments read straight from
// global memory (rows: M[r][k..k+3]; columns: M[k..k+3][r]), the 8-column panels in shared memory;
// a warp owns n / 64 row fragments and runs their k loops interleaved.  Replaces, for these
// shapes, the per-step tile-GEMM launch sequence of big_solve_level (btd_capi.cu), whose serial
// base issued ~5 launches of 4 CTAs per block row.
// ============================================================================================
constexpr int kDmmaDS = 8;  // right-hand-side columns per CTA

// y (n x 8 panel) (+)= sign * op(M) x; op(M) = M (TRANS = false) or M^T.  ZERO_ABOVE: op(M)[r][k]
// == 0 for k > r (op(M) = Linv); ZERO_BELOW: == 0 for k < r (op(M) = Linv^T): whole k steps
// outside the triangle are skipped.
template <bool TRANS, bool ZERO_ABOVE, bool ZERO_BELOW>
__device__ __forceinline__ void dmma_panel(const double* __restrict__ M, int n, const double* x, double* y,
                                           double sign, bool accumulate) {
  constexpr int DS = kDmmaDS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = lane >> 2, lk = lane & 3;
  const int nf = n / 8;  // row fragments
  for (int f0 = warp; f0 < nf; f0 += 32) {  // up to 4 fragments per warp: f0, f0+8, f0+16, f0+24
    double acc[4][2];
    int fr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      fr[i] = f0 + 8 * i < nf ? f0 + 8 * i : -1;
      acc[i][0] = acc[i][1] = 0.0;
    }
    // k range: ZERO_ABOVE (op(M) lower): k <= row, i.e. k0 <= 8 fr + 7; ZERO_BELOW: k >= row
    const int kmax = ZERO_ABOVE ? 8 * (fr[3] >= 0 ? fr[3] : fr[2] >= 0 ? fr[2] : fr[1] >= 0 ? fr[1] : fr[0]) + 8 : n;
    const int kmin = ZERO_BELOW ? 8 * fr[0] : 0;
#pragma unroll 2
    for (int k0 = kmin; k0 < kmax; k0 += 4) {
      const double b = x[(k0 + lk) * DS + lr];
      double av[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = 8 * fr[i] + lr, k = k0 + lk;
        const bool live = fr[i] >= 0 && (!ZERO_ABOVE || k0 <= 8 * fr[i] + 7) && (!ZERO_BELOW || k0 + 3 >= 8 * fr[i]);
        av[i] = live ? __ldg(TRANS ? M + (size_t)k * n + r : M + (size_t)r * n + k) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (fr[i] >= 0) dmma(acc[i], av[i], b);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (fr[i] < 0) continue;
      double* o = y + (8 * fr[i] + lr) * DS + 2 * lk;
      const double2 v = accumulate ? *reinterpret_cast<const double2*>(o) : make_double2(0.0, 0.0);
      *reinterpret_cast<double2*>(o) = make_double2(fma(sign, acc[i][0], v.x), fma(sign, acc[i][1], v.y));
    }
  }
}

__global__ void __launch_bounds__(kWideThreads) solve_dmma_kernel(SolveArgs a) {
  constexpr int DS = kDmmaDS;
  extern __shared__ __align__(16) double sd[];
  const int n = a.n, d = a.d, mode = a.mode;
  double* t = sd;              // n x DS
  double* u = t + n * DS;      // z_{j-1} (forward) / w_{j+1} (backward)
  double* c0v = u + n * DS;    // up: C_L x_L
  double* c1v = c0v + n * DS;  // up: C_R^T x_R
  double* xs = c1v + n * DS;   // separator panel
  if (error_raised(a.err)) return;
  const bool base = mode == kSolveBase;
  const int k = base ? 0 : blockIdx.y;
  const int col0 = blockIdx.x * DS, dc = min(DS, d - col0);
  const long long start = base ? 0 : (long long)a.seps[k] + 1;
  const long long stop = base ? a.N : (long long)a.seps[k + 1];
  const int J = (int)(stop - start);
  const size_t bs = (size_t)n * n, ps = (size_t)n * d;
  const int tid = threadIdx.x;
  auto load_panel = [&](double* dst, const double* src) {
    for (int e = tid; e < n * DS; e += kWideThreads) {
      const int r = e / DS, c = e % DS;
      dst[e] = c < dc ? src[(size_t)r * d + col0 + c] : 0.0;
    }
  };
  auto store_panel = [&](double* dst, const double* src) {
    for (int e = tid; e < n * DS; e += kWideThreads) {
      const int r = e / DS, c = e % DS;
      if (c < dc) dst[(size_t)r * d + col0 + c] = src[e];
    }
  };
  if (mode == kSolveUp) {
    load_panel(xs, a.xsep + (size_t)k * ps);
    __syncthreads();
    dmma_panel<false, false, false>(a.Lsub + (size_t)(start - 1) * bs, n, xs, c0v, 1.0, false);  // C_L x_L
    store_panel(a.x + (size_t)(start - 1) * ps, xs);
    __syncthreads();
    load_panel(xs, a.xsep + (size_t)(k + 1) * ps);
    __syncthreads();
    dmma_panel<true, false, false>(a.Lsub + (size_t)(stop - 1) * bs, n, xs, c1v, 1.0, false);  // C_R^T x_R
    if (k == a.K - 1) store_panel(a.x + (size_t)stop * ps, xs);
    __syncthreads();
  }
  for (int j = 0; j < J; ++j) {  // forward: z_j = Linv_j (b_j - L_{j,j-1} z_{j-1})
    const long long row = start + j;
    load_panel(t, a.rhs + row * ps);
    if (mode == kSolveUp) {
      __syncthreads();
      for (int e = tid; e < n * DS; e += kWideThreads) {
        if (j == 0) t[e] -= c0v[e];
        if (j == J - 1) t[e] -= c1v[e];
      }
    }
    __syncthreads();
    if (j > 0) {
      dmma_panel<false, false, false>(a.Lsub + (size_t)(row - 1) * bs, n, u, t, -1.0, true);
      __syncthreads();
    }
    dmma_panel<false, true, false>(a.Linv + (size_t)row * bs, n, t, u, 1.0, false);  // Linv lower
    __syncthreads();
    store_panel(a.x + row * ps, u);
  }
  for (int j = J - 1; j >= 0; --j) {  // backward: w_j = Linv_j^T (z_j - L_{j+1,j}^T w_{j+1})
    const long long row = start + j;
    if (j < J - 1) {
      load_panel(t, a.x + row * ps);
      __syncthreads();
      dmma_panel<true, false, false>(a.Lsub + (size_t)row * bs, n, u, t, -1.0, true);
    } else {
      for (int e = tid; e < n * DS; e += kWideThreads) t[e] = u[e];
    }
    __syncthreads();
    dmma_panel<true, false, true>(a.Linv + (size_t)row * bs, n, t, u, 1.0, false);  // Linv^T upper
    __syncthreads();
    if (mode != kSolveDown) store_panel(a.x + row * ps, u);
    if (mode == kSolveDown && j == J - 1) {  // f_R = C_R w_last
      dmma_panel<false, false, false>(a.Lsub + (size_t)(stop - 1) * bs, n, u, xs, 1.0, false);
      __syncthreads();
      store_panel(a.fr + (size_t)k * ps, xs);
      __syncthreads();
    }
  }
  if (mode == kSolveDown) {  // f_L = C_L^T w_0
    dmma_panel<true, false, false>(a.Lsub + (size_t)(start - 1) * bs, n, u, xs, 1.0, false);
    __syncthreads();
    store_panel(a.fl + (size_t)k * ps, xs);
  }
}

}  // namespace btd
