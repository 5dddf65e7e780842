// The reference's accelerator seam on the GPU (bt/kernels.py:164-338): batched in-place Cholesky,
// triangular solve and multiply-accumulate over K same-shaped members of ANY strides (the
// reference passes transposed views, e.g. block_cholesky.py:32 solves through
// `coupling.transpose(0, 2, 1)`).  These back the drop-in `kernels` / `block_cholesky` modules
// (serial_factorize, factorize_btd_batch, ...); the recursive hot path does not use them -- it
// runs the fused level kernels (btd_factor*.cuh), which store inverse factors instead of L.
//
// Errors go to a SeamErr word in device memory, chosen by atomicMin exactly like the reference's
// chunked `_run_members` + `_first_bad_pivot` (kernels.py:72-101, 136-161): NotPositiveDefinite
// keeps the earliest block step, then the lowest member, with the 1-based pivot; SingularDiagonal
// the lowest (member, row).  Launches never synchronize; the host reads the word once.
#pragma once

#include "btd_device.cuh"

namespace btd {

struct SeamErr {
  unsigned long long npd;   // (block << 43) | (member << 16) | pivot   (DevErr key layout)
  unsigned long long sing;  // (member << 24) | row (0-based)
};

struct Strides {
  long long k, r, c;  // element strides of member, row, column
};

constexpr int kSeamThreads = 256;
constexpr int kSeamSmemMaxN = 128;  // members up to 128 x 128 are factored in shared memory

__global__ void seam_err_init_kernel(SeamErr* e) {
  e->npd = kNoErr;
  e->sing = kNoErr;
}

// In-place lower Cholesky of every member (strict upper zeroed), chol_factor_batch
// (kernels.py:164-181).  One CTA per member; right-looking column elimination (the column scaled by
// 1/L_jj like LAPACK's potf2), in shared memory for n <= kSeamSmemMaxN, else in place.
// Fails like LAPACK: a pivot that is not > 0 (NaN included).
__global__ void __launch_bounds__(kSeamThreads) seam_chol_kernel(double* a, Strides s, int n, long long block,
                                                                 SeamErr* err) {
  extern __shared__ double sw[];
  // a zero diagonal found by an earlier triangular solve of the same sequence, or a failure at an
  // earlier block step, ends the sequence there (the reference raises at the first failure)
  if (*((volatile const unsigned long long*)&err->sing) != kNoErr) return;
  const unsigned long long prev = *((volatile const unsigned long long*)&err->npd);
  if (prev != kNoErr && (long long)(prev >> 43) < block) return;
  const long long m = blockIdx.x;
  double* A = a + m * s.k;
  const bool in_smem = n <= kSeamSmemMaxN;
  const int tid = threadIdx.x;
  auto W = [&](int r, int c) -> double& { return in_smem ? sw[r * n + c] : A[r * s.r + c * s.c]; };
  if (in_smem)
    for (int e = tid; e < n * n; e += kSeamThreads) {
      const int r = e / n, c = e % n;
      if (c <= r) sw[e] = A[r * s.r + c * s.c];
    }
  __shared__ int fail;
  __shared__ double root;
  if (tid == 0) fail = 0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (tid == 0) {
      const double d = W(j, j);
      if (!(d > 0.0)) {
        fail = j + 1;
      } else {
        root = sqrt(d);
        W(j, j) = root;
      }
    }
    __syncthreads();
    if (fail) break;
    const double rinv = 1.0 / root;
    for (int i = j + 1 + tid; i < n; i += kSeamThreads) W(i, j) *= rinv;
    __syncthreads();
    // trailing lower triangle: W(i, k) -= W(i, j) W(k, j), j < k <= i
    const int t = n - j - 1;
    for (int e = tid; e < t * t; e += kSeamThreads) {
      const int i = j + 1 + e / t, k = j + 1 + e % t;
      if (k <= i) W(i, k) -= W(i, j) * W(k, j);
    }
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) {
      const unsigned long long key = ((unsigned long long)block << 43) | ((unsigned long long)m << 16) |
                                     (unsigned long long)(fail & 0xffff);
      atomicMin(&err->npd, key);
    }
    return;
  }
  for (int e = tid; e < n * n; e += kSeamThreads) {
    const int r = e / n, c = e % n;
    A[r * s.r + c * s.c] = c > r ? 0.0 : (in_smem ? sw[e] : A[r * s.r + c * s.c]);
  }
}

// SingularDiagonal pre-check of trsm_lower_batch (kernels.py:227-233): lowest (member, row) with an
// exactly zero diagonal entry.
__global__ void seam_diag_check_kernel(const double* f, Strides s, int n, long long count, SeamErr* err) {
  if (*((volatile const unsigned long long*)&err->npd) != kNoErr) return;  // an earlier Cholesky failed
  const long long m = blockIdx.x;
  for (int r = threadIdx.x; r < n; r += blockDim.x)
    if (f[m * s.k + r * (s.r + s.c)] == 0.0) atomicMin(&err->sing, ((unsigned long long)m << 24) | (unsigned)r);
}

// In-place triangular solve of every member's panel (trsm_lower_batch, kernels.py:215-259):
// trans = 0: P <- L^{-1} P (forward sweep), trans = 1: P <- L^{-T} P (backward sweep); L is the lower
// triangle of the factor member.  grid = (count, column chunks); a thread owns one panel column.
// Skips everything when the pre-check found a zero diagonal (the reference raises before solving).
__global__ void __launch_bounds__(kSeamThreads) seam_trsm_kernel(const double* f, Strides fs, double* p, Strides ps,
                                                                 int n, int cols, int trans, const SeamErr* err) {
  if (*((volatile const unsigned long long*)&err->sing) != kNoErr ||
      *((volatile const unsigned long long*)&err->npd) != kNoErr)
    return;
  extern __shared__ double sl[];
  const long long m = blockIdx.x;
  const double* F = f + m * fs.k;
  double* P = p + m * ps.k;
  const bool in_smem = n <= kSeamSmemMaxN;
  if (in_smem)
    for (int e = threadIdx.x; e < n * n; e += kSeamThreads) {
      const int r = e / n, c = e % n;
      sl[e] = c <= r ? F[r * fs.r + c * fs.c] : 0.0;
    }
  __syncthreads();
  auto L = [&](int r, int c) -> double { return in_smem ? sl[r * n + c] : F[r * fs.r + c * fs.c]; };
  const int col = blockIdx.y * kSeamThreads + threadIdx.x;
  if (col >= cols) return;
  double* x = P + col * ps.c;
  if (!trans) {
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int k = 0; k < i; ++k) acc = fma(L(i, k), x[k * ps.r], acc);
      x[i * ps.r] = (x[i * ps.r] - acc) / L(i, i);
    }
  } else {
    for (int i = n - 1; i >= 0; --i) {
      double acc = 0.0;
      for (int k = i + 1; k < n; ++k) acc = fma(L(k, i), x[k * ps.r], acc);
      x[i * ps.r] = (x[i * ps.r] - acc) / L(i, i);
    }
  }
}

// out <- alpha op(a) op(b) + beta out per member (gemm_acc_batch, kernels.py:270-310).  The operand
// transposes are folded into the strides by the host.  alpha == 0 skips the product (out scaled by
// beta; beta == 0 writes exact zeros, so NaNs in out do not propagate, as in the reference).
// grid = (32 x 32 output tiles, count); k staged through shared memory in chunks of 32.
constexpr int kSeamTile = 32;
__global__ void __launch_bounds__(kSeamThreads) seam_gemm_kernel(double* out, Strides os, const double* a, Strides as,
                                                                 const double* b, Strides bs, int M, int Q, int Pc,
                                                                 int tiles_p, double alpha, double beta) {
  __shared__ double At[kSeamTile][kSeamTile + 1], Bt[kSeamTile][kSeamTile + 1];
  const long long m = blockIdx.y;
  const int tm = blockIdx.x / tiles_p, tp = blockIdx.x % tiles_p;
  const int r0 = tm * kSeamTile, c0 = tp * kSeamTile;
  const int tid = threadIdx.x, tr = tid / 8, tc = (tid % 8) * 4;  // 32 rows x (8 x 4 cols)
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const double* A = a + m * as.k;
  const double* B = b + m * bs.k;
  if (alpha != 0.0) {
    for (int k0 = 0; k0 < Q; k0 += kSeamTile) {
      for (int e = tid; e < kSeamTile * kSeamTile; e += kSeamThreads) {
        const int i = e / kSeamTile, kk = e % kSeamTile;
        At[i][kk] = (r0 + i < M && k0 + kk < Q) ? A[(r0 + i) * as.r + (k0 + kk) * as.c] : 0.0;
        Bt[kk][i] = (k0 + kk < Q && c0 + i < Pc) ? B[(k0 + kk) * bs.r + (c0 + i) * bs.c] : 0.0;
      }
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < kSeamTile; ++kk) {
        const double av = At[tr][kk];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = fma(av, Bt[kk][tc + q], acc[q]);
      }
      __syncthreads();
    }
  }
  double* O = out + m * os.k;
  const int r = r0 + tr;
  if (r >= M) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = c0 + tc + q;
    if (c >= Pc) continue;
    double& o = O[r * os.r + c * os.c];
    if (alpha == 0.0) {
      if (beta == 0.0) o = 0.0;
      else if (beta != 1.0) o *= beta;
    } else {
      const double prod = alpha == 1.0 ? acc[q] : acc[q] * alpha;
      o = beta == 0.0 ? prod : (beta == 1.0 ? o : o * beta) + prod;
    }
  }
}

}  // namespace btd
