// Per-level solve kernels (one CTA per (segment, column chunk)).
//
// Down pass (replaces split_rhs + compute_separator_rhs, bt/schur.py:196-211,230-260):
//   w = A_uu^{-1} b_u  by forward z_j = Linv_j (b_j - L_{j,j-1} z_{j-1}) and backward
//   w_j = Linv_j^T (z_j - L_{j+1,j}^T w_{j+1});  fold  f_L = C_L^T w_0,  f_R = C_R w_last.
//   The separator RHS is then  b_s[p] - f_L[p] - f_R[p-1]  (assemble_separator_rhs_kernel),
//   identical to A_ll-side of Alg. 5 because  A_lu^T A_uu^{-1} b_u = A_lu^T w.
// Up pass (replaces update_boundary + solve_btd_batch + assemble_solution, bt/schur.py:214-227,263-286,373):
//   b_0 -= C_L x_{s_k}, b_last -= C_R^T x_{s_{k+1}}, then the same forward/backward sweep writes
//   X in the original block order; separator rows are copied from the level below.
// Base (serial_solve, bt/block_cholesky.py:95-98): one uncoupled sweep over the whole chain.
//
// The factor stores Linv (not L), so every block step is a mat-vec: no sequential trsv inside a block.
#pragma once

#include "btd_device.cuh"

namespace btd {

enum SolveMode : int { kSolveDown = 0, kSolveUp = 1, kSolveBase = 2 };

struct SolveArgs {
  const double* rhs;    // level rhs (N, n, d)
  const double* Linv;   // (N, n, n)
  const double* Lsub;   // (N-1, n, n)
  const int* seps;      // (K+1)
  const double* xsep;   // up: solution of the next level (K+1, n, d)
  double* x;            // (N, n, d): solution (up/base) or scratch (down)
  double* fl;           // down: (K, n, d) f_L per segment (into the next level's rhs slots)
  double* fr;           // down: (K, n, d) f_R per segment
  long long N;
  int n, d, K, mode;
  const DevErr* err;
};

template <int NT>
struct SolveShape {
  static constexpr int NTHREADS = NT == 64 ? 128 : NT == 32 ? 64 : 32;
  static constexpr int TPR = NTHREADS / NT;  // threads per row (non-transposed mat-vec)
  static constexpr int CPT = NT / TPR;       // columns per thread
};

// y[r][c] (+)= sign * sum_m op(M)[r][m] * x[m][c]    (M: n x n row-major in global memory)
// x, y: shared NT x DC panels. Ends with a barrier.
template <int NT, int DC, bool TRANS, bool PACKED = false>
__device__ __forceinline__ void block_mv(const double* __restrict__ M, int n, const double* x, double* y,
                                         double sign, bool accumulate, double* red) {
  using S = SolveShape<NT>;
  constexpr int TPR = S::TPR, CPT = S::CPT;
  const int tid = threadIdx.x;
  double part[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) part[c] = 0.0;
  if (!TRANS) {
    const int r = tid / TPR, q = tid % TPR;
    if (r < n) {
      const double* row = M + (size_t)r * n;
#pragma unroll 8
      for (int mm = 0; mm < CPT; ++mm) {
        const int m = q * CPT + mm;
        if (m < n && (!PACKED || m <= r)) {
          const double v = PACKED ? __ldg(M + packed_offset_(r) + m) : __ldg(row + m);
#pragma unroll
          for (int c = 0; c < DC; ++c) part[c] += v * x[m * DC + c];
        }
      }
    }
#pragma unroll
    for (int off = 1; off < TPR; off <<= 1)
#pragma unroll
      for (int c = 0; c < DC; ++c) part[c] += __shfl_xor_sync(0xffffffffu, part[c], off);
    if (q == 0 && r < NT) {
#pragma unroll
      for (int c = 0; c < DC; ++c) {
        const double v = (r < n) ? sign * part[c] : 0.0;
        y[r * DC + c] = accumulate ? y[r * DC + c] + v : v;
      }
    }
    __syncthreads();
  } else {
    const int r = tid % NT, g = tid / NT;  // column r of M, row group g
    constexpr int RPG = NT / TPR;
    if (r < n) {
#pragma unroll 8
      for (int mm = 0; mm < RPG; ++mm) {
        const int m = g * RPG + mm;
        if (m < n && (!PACKED || m >= r)) {
          const double v = PACKED ? __ldg(M + packed_offset_(m) + r) : __ldg(M + (size_t)m * n + r);
#pragma unroll
          for (int c = 0; c < DC; ++c) part[c] += v * x[m * DC + c];
        }
      }
    }
    if (TPR > 1) {
#pragma unroll
      for (int c = 0; c < DC; ++c) red[(g * NT + r) * DC + c] = part[c];
      __syncthreads();
      if (g == 0) {
#pragma unroll
        for (int c = 0; c < DC; ++c) {
          double s = 0.0;
#pragma unroll
          for (int gg = 0; gg < TPR; ++gg) s += red[(gg * NT + r) * DC + c];
          const double v = (r < n) ? sign * s : 0.0;
          y[r * DC + c] = accumulate ? y[r * DC + c] + v : v;
        }
      }
    } else {
#pragma unroll
      for (int c = 0; c < DC; ++c) {
        const double v = (r < n) ? sign * part[c] : 0.0;
        y[r * DC + c] = accumulate ? y[r * DC + c] + v : v;
      }
    }
    __syncthreads();
  }
}

template <int NT, int DC>
__device__ __forceinline__ void load_panel(double* v, const double* g, int n, int d, int c0, int dc) {
  for (int e = threadIdx.x; e < NT * DC; e += SolveShape<NT>::NTHREADS) {
    const int r = e / DC, c = e % DC;
    v[e] = (r < n && c < dc) ? g[(size_t)r * d + c0 + c] : 0.0;
  }
}

template <int NT, int DC>
__device__ __forceinline__ void store_panel(double* g, const double* v, int n, int d, int c0, int dc) {
  for (int e = threadIdx.x; e < n * DC; e += SolveShape<NT>::NTHREADS) {
    const int r = e / DC, c = e % DC;
    if (c < dc) g[(size_t)r * d + c0 + c] = v[e];
  }
}

template <int NT, int DC>
__global__ void __launch_bounds__(SolveShape<NT>::NTHREADS) solve_level_kernel(SolveArgs a) {
  if (error_raised(a.err)) return;
  __shared__ double t[NT * DC], u[NT * DC], w[NT * DC], xl[NT * DC], red[SolveShape<NT>::TPR * NT * DC];
  const int k = blockIdx.x;
  const int c0 = blockIdx.y * DC;
  const int dc = min(DC, a.d - c0);
  const int n = a.n, d = a.d;
  const bool coupled = a.mode != kSolveBase;
  const long long start = coupled ? (long long)a.seps[k] + 1 : 0;
  const long long stop = coupled ? (long long)a.seps[k + 1] : a.N;
  const int J = (int)(stop - start);
  const size_t bs = (size_t)n * n, ps = (size_t)n * d, pk = (size_t)packed_offset_(n);

  // forward sweep: z_j = Linv_j (b_j - L_{j,j-1} z_{j-1});  z kept in u, spilled to x[row]
  for (int j = 0; j < J; ++j) {
    const long long row = start + j;
    load_panel<NT, DC>(t, a.rhs + row * ps, n, d, c0, dc);
    if (a.mode == kSolveUp) {
      if (j == 0) {  // b_0 -= C_L x_{s_k}
        load_panel<NT, DC>(xl, a.xsep + (size_t)k * ps, n, d, c0, dc);
        __syncthreads();
        block_mv<NT, DC, false>(a.Lsub + (start - 1) * bs, n, xl, t, -1.0, true, red);
      }
      if (j == J - 1) {  // b_last -= C_R^T x_{s_{k+1}}
        __syncthreads();
        load_panel<NT, DC>(xl, a.xsep + (size_t)(k + 1) * ps, n, d, c0, dc);
        __syncthreads();
        block_mv<NT, DC, true>(a.Lsub + (stop - 1) * bs, n, xl, t, -1.0, true, red);
      }
    }
    __syncthreads();
    if (j > 0) block_mv<NT, DC, false>(a.Lsub + (row - 1) * bs, n, u, t, -1.0, true, red);
    block_mv<NT, DC, false, true>(a.Linv + row * pk, n, t, u, 1.0, false, red);
    if (j < J - 1) store_panel<NT, DC>(a.x + row * ps, u, n, d, c0, dc);
  }
  // backward sweep: x_j = Linv_j^T (z_j - L_{j+1,j}^T x_{j+1});  x_{j+1} kept in w
  for (int j = J - 1; j >= 0; --j) {
    const long long row = start + j;
    if (j == J - 1) {
      for (int e = threadIdx.x; e < NT * DC; e += SolveShape<NT>::NTHREADS) t[e] = u[e];
    } else {
      load_panel<NT, DC>(t, a.x + row * ps, n, d, c0, dc);
    }
    __syncthreads();
    if (j < J - 1) block_mv<NT, DC, true>(a.Lsub + row * bs, n, w, t, -1.0, true, red);
    block_mv<NT, DC, true, true>(a.Linv + row * pk, n, t, w, 1.0, false, red);
    if (a.mode == kSolveDown && j == J - 1) {  // f_R = C_R w_last
      block_mv<NT, DC, false>(a.Lsub + (stop - 1) * bs, n, w, xl, 1.0, false, red);
      store_panel<NT, DC>(a.fr + (size_t)k * ps, xl, n, d, c0, dc);
    }
    if (a.mode != kSolveDown) store_panel<NT, DC>(a.x + row * ps, w, n, d, c0, dc);
  }
  if (a.mode == kSolveDown) {  // f_L = C_L^T w_0
    block_mv<NT, DC, true>(a.Lsub + (start - 1) * bs, n, w, xl, 1.0, false, red);
    store_panel<NT, DC>(a.fl + (size_t)k * ps, xl, n, d, c0, dc);
  } else if (a.mode == kSolveUp) {  // separator rows come from the level below
    for (int e = threadIdx.x; e < n * DC; e += SolveShape<NT>::NTHREADS) {
      const int r = e / DC, c = e % DC;
      if (c >= dc) continue;
      a.x[(size_t)(start - 1) * ps + (size_t)r * d + c0 + c] = a.xsep[(size_t)k * ps + (size_t)r * d + c0 + c];
      if (k == a.K - 1)
        a.x[(size_t)stop * ps + (size_t)r * d + c0 + c] = a.xsep[(size_t)(k + 1) * ps + (size_t)r * d + c0 + c];
    }
  }
}

// Separator RHS of the next level: (b[s_p] - f_L[p]) - f_R[p-1]  (bt/schur.py:256-259 order).
// f_L[p] already sits in next_rhs[p].
__global__ void assemble_separator_rhs_kernel(const double* rhs, const int* seps, double* next_rhs,
                                              const double* fr, int K, int n, int d, const DevErr* err) {
  if (error_raised(err)) return;
  const size_t ps = (size_t)n * d;
  const size_t total = (size_t)(K + 1) * ps;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int p = (int)(e / ps);
    double v = rhs[(size_t)seps[p] * ps + e % ps];
    if (p < K) v -= next_rhs[e];
    if (p > 0) v -= fr[e - ps];
    next_rhs[e] = v;
  }
}

}  // namespace btd
