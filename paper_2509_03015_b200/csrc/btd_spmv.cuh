// Block-tridiagonal SpMV and fused residual norms.
//
// Replaces btd_matmul (bt/core.py:280-288) and the norm part of residual_report
// (bt/report.py:20-38):
//   y_i = D_i x_i + A_{i,i-1} x_{i-1} + A_{i+1,i}^T x_{i+1},   A_{i+1,i} = sub[i]
//   r   = b - A x ;  per column c:  ||r_c||_2^2 , ||b_c||_2^2
// HBM-bound: every block of A comes from HBM once (a CTA owns a contiguous run of block rows, so the
// second use of sub[i] -- row i+1 right after row i -- hits L2); x and y/b panels are small.  The norms are
// reduced deterministically: per-CTA partials in a fixed order, then one CTA sums the partials in
// CTA order (no floating-point atomics).
#pragma once

#include "btd_device.cuh"

namespace btd {

constexpr int kSpmvThreads = 256;
constexpr int kSpmvMaxD = 8;  // columns per pass (the grid's y dimension covers wider rhs)

struct SpmvArgs {
  const double* diag;
  const double* sub;
  const double* x;
  const double* b;  // residual mode: rhs (may be null for plain y = A x)
  double* y;        // y = A x (may be null in residual mode)
  double* partial;  // residual mode: (gridDim.x, 2 * d) per-CTA sums (r^2, b^2)
  long long N;
  int n, d;
  long long rows_per_cta;
};

// acc[c] += sum_m M(r, m) v(m, c)  (trans: M(m, r)); one thread = one (row, slice) pair, the 4
// slices of a row are reduced with shuffles.  M is a global n x n block, v a global n x d panel.
__device__ __forceinline__ void block_mv(const double* M, const double* v, bool trans, int n, int d, int c0, int dc,
                                         int r, int part, double (&acc)[kSpmvMaxD]) {
  if (r >= n) return;
#pragma unroll 4
  for (int m = part; m < n; m += 4) {
    const double a = trans ? M[(size_t)m * n + r] : M[(size_t)r * n + m];
    const double* vm = v + (size_t)m * d + c0;
#pragma unroll
    for (int c = 0; c < kSpmvMaxD; ++c)
      if (c < dc) acc[c] = fma(a, vm[c], acc[c]);
  }
}

__global__ void __launch_bounds__(kSpmvThreads) btd_spmv_kernel(SpmvArgs a) {
  __shared__ double red[kSpmvThreads / 32][2 * kSpmvMaxD];
  const int n = a.n, d = a.d;
  const int c0 = blockIdx.y * kSpmvMaxD, dc = min(kSpmvMaxD, d - c0);
  const long long r0 = (long long)blockIdx.x * a.rows_per_cta;
  const long long r1 = min(a.N, r0 + a.rows_per_cta);
  const size_t bs = (size_t)n * n, ps = (size_t)n * d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double rr[kSpmvMaxD], bb[kSpmvMaxD];
#pragma unroll
  for (int c = 0; c < kSpmvMaxD; ++c) rr[c] = bb[c] = 0.0;
  // rows are handled 64 at a time by the 256 threads (4 slices per row)
  for (long long i = r0; i < r1; ++i) {
    for (int rbase = 0; rbase < n; rbase += kSpmvThreads / 4) {
      const int r = rbase + tid / 4, part = tid & 3;
      double acc[kSpmvMaxD];
#pragma unroll
      for (int c = 0; c < kSpmvMaxD; ++c) acc[c] = 0.0;
      block_mv(a.diag + (size_t)i * bs, a.x + (size_t)i * ps, false, n, d, c0, dc, r, part, acc);
      if (i > 0) block_mv(a.sub + (size_t)(i - 1) * bs, a.x + (size_t)(i - 1) * ps, false, n, d, c0, dc, r, part, acc);
      if (i + 1 < a.N) block_mv(a.sub + (size_t)i * bs, a.x + (size_t)(i + 1) * ps, true, n, d, c0, dc, r, part, acc);
#pragma unroll
      for (int c = 0; c < kSpmvMaxD; ++c) {
        acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 1);
        acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 2);
      }
      if (part == 0 && r < n) {
#pragma unroll
        for (int c = 0; c < kSpmvMaxD; ++c) {
          if (c >= dc) break;
          const size_t off = (size_t)i * ps + (size_t)r * d + c0 + c;
          if (a.y) a.y[off] = acc[c];
          if (a.b) {
            const double bv = a.b[off], rv = bv - acc[c];
            rr[c] = fma(rv, rv, rr[c]);
            bb[c] = fma(bv, bv, bb[c]);
          }
        }
      }
    }
  }
  if (!a.b) return;
  // deterministic CTA reduction: warp shuffles, then warps in order
#pragma unroll
  for (int c = 0; c < kSpmvMaxD; ++c) {
    for (int o = 16; o > 0; o >>= 1) {
      rr[c] += __shfl_xor_sync(0xffffffffu, rr[c], o);
      bb[c] += __shfl_xor_sync(0xffffffffu, bb[c], o);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < kSpmvMaxD; ++c) {
      red[warp][c] = rr[c];
      red[warp][kSpmvMaxD + c] = bb[c];
    }
  }
  __syncthreads();
  if (tid < 2 * kSpmvMaxD) {
    double s = 0.0;
    for (int w = 0; w < kSpmvThreads / 32; ++w) s += red[w][tid];
    const int c = tid % kSpmvMaxD, which = tid / kSpmvMaxD;
    if (c < dc) a.partial[(size_t)blockIdx.x * 2 * d + which * d + c0 + c] = s;
  }
}

// Sum the per-CTA partials in CTA order: out[0..d) = ||r||^2, out[d..2d) = ||b||^2.
__global__ void btd_norm_finish_kernel(const double* partial, int ctas, int d, double* out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 2 * d) return;
  double s = 0.0;
  for (int i = 0; i < ctas; ++i) s += partial[(size_t)i * 2 * d + e];
  out[e] = s;
}

}  // namespace btd
