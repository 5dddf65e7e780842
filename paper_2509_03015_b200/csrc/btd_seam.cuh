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

// Visit every (r, c) of an R x C window with lanes along the unit-stride axis (cfast: columns) and
// warps plus an 8-deep unroll along the other, so a lone CTA keeps 8 loads per thread in flight
// instead of one L2 round trip per element; no integer division in the index math.
template <class Src, class Dst>
__device__ __forceinline__ void seam_stage(int R, int C, bool cfast, Src src, Dst dst) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kSeamThreads / 32;
  const int outer = cfast ? R : C, inner = cfast ? C : R;
  for (int b = lane; b < inner; b += 32)
    for (int a0 = warp; a0 < outer; a0 += nw * 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int a = a0 + q * nw;
        v[q] = a < outer ? (cfast ? src(a, b) : src(b, a)) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int a = a0 + q * nw;
        if (a < outer) {
          if (cfast) dst(a, b, v[q]);
          else dst(b, a, v[q]);
        }
      }
    }
}

__host__ __device__ constexpr int seam_np(int n) { return (n + 7) & ~7; }  // padded to whole 8-row blocks
__host__ __device__ constexpr size_t seam_chol_smem(int n) {
  return (size_t)seam_np(n) * (seam_np(n) + 4) * sizeof(double);
}

// In-place lower Cholesky of every member (strict upper zeroed), chol_factor_batch
// (kernels.py:164-181), for n <= kSeamSmemMaxN.  One CTA per member, the member in shared memory
// padded with an identity tail to a multiple of 8; right-looking over 8-column panels: the panel
// factored one column per barrier with a thread per row (rows held in registers, the panel's own
// 8 rows exchanged through a double-buffered shared tile, every thread deriving the pivot itself,
// so a failure is seen by all threads at once), then the trailing lower triangle updated by DMMA.
// Column scaling by 1/L_jj like LAPACK's potf2; fails like LAPACK: the first pivot that is not > 0
// (NaN included), 1-based.
__global__ void __launch_bounds__(kSeamThreads) seam_chol_smem_kernel(double* a, Strides s, int n, long long block,
                                                                      SeamErr* err) {
  extern __shared__ double sw[];
  __shared__ double pbuf[2][8][9];
  // a zero diagonal found by an earlier triangular solve of the same sequence, or a failure at an
  // earlier block step, ends the sequence there (the reference raises at the first failure); both
  // words are stable during the launch (same-launch reports carry this launch's block)
  if (*((volatile const unsigned long long*)&err->sing) != kNoErr) return;
  const unsigned long long prev = *((volatile const unsigned long long*)&err->npd);
  if (prev != kNoErr && (long long)(prev >> 43) < block) return;
  const long long m = blockIdx.x;
  double* A = a + m * s.k;
  const int NP = seam_np(n), LL = NP + 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool cfast = llabs(s.c) <= llabs(s.r);
  seam_stage(
      NP, NP, cfast,
      [&](int r, int c) {
        return (r < n && c <= r) ? A[(long long)r * s.r + (long long)c * s.c] : (r == c ? 1.0 : 0.0);
      },
      [&](int r, int c, double v) { sw[r * LL + c] = v; });
  __syncthreads();
  int fail = 0;
  for (int j0 = 0; j0 < NP; j0 += 8) {
    const int r = j0 + tid;
    const bool own = r < NP;
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = own ? sw[r * LL + j0 + q] : 0.0;
    if (tid < 8)
#pragma unroll
      for (int q = 0; q < 8; ++q) pbuf[0][tid][q] = v[q];
    __syncthreads();
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const double(*pb)[9] = pbuf[jj & 1];
      const double d = pb[jj][jj];
      if (!(d > 0.0)) {
        fail = j0 + jj + 1;
        break;
      }
      const double root = sqrt(d), rinv = 1.0 / root;
      if (own && r >= j0 + jj) {
        if (r == j0 + jj) {
          v[jj] = root;
        } else {
          const double l = v[jj] * rinv;
          v[jj] = l;
#pragma unroll
          for (int kk = jj + 1; kk < 8; ++kk) v[kk] = fma(-l, pb[kk][jj] * rinv, v[kk]);
        }
      }
      if (tid < 8)
#pragma unroll
        for (int q = 0; q < 8; ++q) pbuf[(jj + 1) & 1][tid][q] = v[q];
      __syncthreads();
    }
    if (fail) break;
    if (own)
#pragma unroll
      for (int q = 0; q < 8; ++q) sw[r * LL + j0 + q] = v[q];
    __syncthreads();
    // trailing lower triangle: W(i, c) -= sum_k L(i, j0 + k) L(c, j0 + k), 8 x 8 tiles on DMMA
    const int R = (NP - j0 - 8) / 8;
    for (int t = warp; t < R * R; t += kSeamThreads / 32) {
      const int ti = t / R, tj = t % R;
      if (tj > ti) continue;
      const int i0 = j0 + 8 + ti * 8, c0 = j0 + 8 + tj * 8;
      const int rr = i0 + (lane >> 2), cc = c0 + 2 * (lane & 3);
      double dd[2] = {sw[rr * LL + cc], sw[rr * LL + cc + 1]};
#pragma unroll
      for (int ks = 0; ks < 8; ks += 4) {
        const double av = sw[(i0 + (lane >> 2)) * LL + j0 + ks + (lane & 3)];
        const double bv = sw[(c0 + (lane >> 2)) * LL + j0 + ks + (lane & 3)];
        dmma(dd, -av, bv);
      }
      sw[rr * LL + cc] = dd[0];
      sw[rr * LL + cc + 1] = dd[1];
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
  seam_stage(
      n, n, cfast, [&](int r, int c) { return c > r ? 0.0 : sw[r * LL + c]; },
      [&](int r, int c, double v) { A[(long long)r * s.r + (long long)c * s.c] = v; });
}

// The same for members larger than kSeamSmemMaxN: one CTA per member, right-looking column
// elimination in place in global memory.
__global__ void __launch_bounds__(kSeamThreads) seam_chol_kernel(double* a, Strides s, int n, long long block,
                                                                 SeamErr* err) {
  if (*((volatile const unsigned long long*)&err->sing) != kNoErr) return;
  const unsigned long long prev = *((volatile const unsigned long long*)&err->npd);
  if (prev != kNoErr && (long long)(prev >> 43) < block) return;
  const long long m = blockIdx.x;
  double* A = a + m * s.k;
  const int tid = threadIdx.x;
  auto W = [&](int r, int c) -> double& { return A[(long long)r * s.r + (long long)c * s.c]; };
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
    if (c > r) W(r, c) = 0.0;
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

// In-place triangular solve of every member's panel (trsm_lower_batch, kernels.py:215-259) for
// factors larger than kSeamSmemMaxN (smaller ones: seam_trsm_dmma_kernel below): trans = 0:
// P <- L^{-1} P (forward sweep), trans = 1: P <- L^{-T} P (backward sweep); L is the lower triangle
// of the factor member, read from global memory.  grid = (count, column chunks); a thread owns one
// panel column.  Skips everything when the pre-check found a zero diagonal (the reference raises
// before solving).
__global__ void __launch_bounds__(kSeamThreads) seam_trsm_kernel(const double* f, Strides fs, double* p, Strides ps,
                                                                 int n, int cols, int trans, const SeamErr* err) {
  if (*((volatile const unsigned long long*)&err->sing) != kNoErr ||
      *((volatile const unsigned long long*)&err->npd) != kNoErr)
    return;
  const long long m = blockIdx.x;
  const double* F = f + m * fs.k;
  double* P = p + m * ps.k;
  auto L = [&](int r, int c) -> double { return F[r * fs.r + c * fs.c]; };
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

// trsm_lower_batch for n <= kSeamSmemMaxN on the fp64 tensor core: the member's factor (lower
// triangle, padded to a multiple of 8 with an identity tail) and a 64-column chunk of its panel are
// staged in shared memory; rows are eliminated in blocks of 8 -- the 8 x 8 diagonal solve one
// thread per column, then the remaining rows updated by DMMA (X_rest -= L_rest,blk X_blk), the
// backward sweep the same bottom-up with L^T.  grid = (count, column chunks), 8 warps.
constexpr int kStCols = 64, kStLX = kStCols + 8;
__host__ __device__ constexpr size_t seam_trsm_smem(int n) {
  return ((size_t)seam_np(n) * (seam_np(n) + 4) + (size_t)seam_np(n) * kStLX) * sizeof(double);
}
__global__ void __launch_bounds__(kSeamThreads) seam_trsm_dmma_kernel(const double* f, Strides fs, double* p,
                                                                      Strides ps, int n, int cols, int trans,
                                                                      const SeamErr* err) {
  if (*((volatile const unsigned long long*)&err->sing) != kNoErr ||
      *((volatile const unsigned long long*)&err->npd) != kNoErr)
    return;
  extern __shared__ double sw[];
  const int NP = seam_np(n), LL = NP + 4;
  double* Ls = sw;            // Ls[r * LL + c]
  double* Xs = sw + NP * LL;  // Xs[r * kStLX + c]
  const long long m = blockIdx.x;
  const double* F = f + m * fs.k;
  double* P = p + m * ps.k;
  const int col0 = blockIdx.y * kStCols, w = min(kStCols, cols - col0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool f_cfast = llabs(fs.c) <= llabs(fs.r), p_cfast = llabs(ps.c) <= llabs(ps.r);
  seam_stage(
      NP, NP, f_cfast,
      [&](int r, int c) {
        return (r < n && c <= r) ? F[(long long)r * fs.r + (long long)c * fs.c] : (r == c ? 1.0 : 0.0);
      },
      [&](int r, int c, double v) { Ls[r * LL + c] = v; });
  seam_stage(
      NP, kStCols, p_cfast,
      [&](int r, int c) {
        return (r < n && c < w) ? P[(long long)r * ps.r + (long long)(col0 + c) * ps.c] : 0.0;
      },
      [&](int r, int c, double v) { Xs[r * kStLX + c] = v; });
  __syncthreads();
  // the diagonal is only ever divided by: keep its reciprocals in place (one multiply per row on
  // the serial path of the 8 x 8 solves instead of a division)
  for (int r = tid; r < NP; r += kSeamThreads) Ls[r * LL + r] = 1.0 / Ls[r * LL + r];
  __syncthreads();
  const int nb = NP / 8;
  for (int s = 0; s < nb; ++s) {
    const int rb = trans ? (nb - 1 - s) * 8 : s * 8;
    if (tid < kStCols) {  // the diagonal 8 x 8 block, one thread per column
      double x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = Xs[(rb + q) * kStLX + tid];
      if (!trans) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < q; ++k) acc = fma(Ls[(rb + q) * LL + rb + k], x[k], acc);
          x[q] = (x[q] - acc) * Ls[(rb + q) * LL + rb + q];
        }
      } else {
#pragma unroll
        for (int q = 7; q >= 0; --q) {
          double acc = 0.0;
#pragma unroll
          for (int k = q + 1; k < 8; ++k) acc = fma(Ls[(rb + k) * LL + rb + q], x[k], acc);
          x[q] = (x[q] - acc) * Ls[(rb + q) * LL + rb + q];
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) Xs[(rb + q) * kStLX + tid] = x[q];
    }
    __syncthreads();
    // the rest: forward rows below the block, backward rows above it; 8 x 16 output tiles over
    // warps (two DMMA chains sharing the L fragment)
    const int rlo = trans ? 0 : rb + 8, rows = trans ? rb : NP - rb - 8;
    const int tiles = (rows / 8) * (kStCols / 16);
    for (int t = warp; t < tiles; t += kSeamThreads / 32) {
      const int i0 = rlo + (t >> 2) * 8, c0 = (t & 3) * 16;
      const int rr = i0 + (lane >> 2), cc = c0 + 2 * (lane & 3);
      double d0[2] = {Xs[rr * kStLX + cc], Xs[rr * kStLX + cc + 1]};
      double d1[2] = {Xs[rr * kStLX + cc + 8], Xs[rr * kStLX + cc + 9]};
#pragma unroll
      for (int ks = 0; ks < 8; ks += 4) {
        const double av = trans ? Ls[(rb + ks + (lane & 3)) * LL + i0 + (lane >> 2)]
                                : Ls[(i0 + (lane >> 2)) * LL + rb + ks + (lane & 3)];
        const double* xb = Xs + (rb + ks + (lane & 3)) * kStLX + c0 + (lane >> 2);
        dmma(d0, -av, xb[0]);
        dmma(d1, -av, xb[8]);
      }
      Xs[rr * kStLX + cc] = d0[0];
      Xs[rr * kStLX + cc + 1] = d0[1];
      Xs[rr * kStLX + cc + 8] = d1[0];
      Xs[rr * kStLX + cc + 9] = d1[1];
    }
    __syncthreads();
  }
  seam_stage(
      n, w, p_cfast, [&](int r, int c) { return Xs[r * kStLX + c]; },
      [&](int r, int c, double v) { P[(long long)r * ps.r + (long long)(col0 + c) * ps.c] = v; });
}

// out <- alpha op(a) op(b) + beta out per member (gemm_acc_batch, kernels.py:270-310).  The operand
// transposes are folded into the strides by the host.  alpha == 0 skips the product (out scaled by
// beta; beta == 0 writes exact zeros, so NaNs in out do not propagate, as in the reference).
// grid = (64 x 64 output tiles, count), 8 warps; k staged through shared memory in chunks of 16
// (the next chunk's loads in flight during the current chunk's products), products on the fp64
// tensor core (DMMA m8n8k4), each warp a 32 x 16 sub-tile.  Staging loads run along whichever of
// the two operand strides is the smaller, so transposed views are read as coalesced as plain ones.
constexpr int kSgT = 64, kSgK = 16, kSgLA = kSgK + 4, kSgLB = kSgT + 8;  // pads: conflict-free fragments
__global__ void __launch_bounds__(kSeamThreads) seam_gemm_kernel(double* out, Strides os, const double* a, Strides as,
                                                                 const double* b, Strides bs, int M, int Q, int Pc,
                                                                 int tiles_p, double alpha, double beta) {
  __shared__ double At[kSgT * kSgLA];  // At[i][kk]
  __shared__ double Bt[kSgK * kSgLB];  // Bt[kk][c]
  const long long m = blockIdx.y;
  const int tm = blockIdx.x / tiles_p, tp = blockIdx.x % tiles_p;
  const int r0 = tm * kSgT, c0 = tp * kSgT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = (warp >> 2) * 32, wc = (warp & 3) * 16;
  double acc[4][2][2] = {};
  const double* A = a + m * as.k;
  const double* B = b + m * bs.k;
  const bool a_kfast = llabs(as.c) <= llabs(as.r), b_cfast = llabs(bs.c) <= llabs(bs.r);
  if (alpha != 0.0) {
    double ra[4], rb[4];
    auto load = [&](int k0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = tid + q * kSeamThreads;
        const int i = a_kfast ? e >> 4 : e & 63, kk = a_kfast ? e & 15 : e >> 6;
        ra[q] = (r0 + i < M && k0 + kk < Q) ? A[(long long)(r0 + i) * as.r + (long long)(k0 + kk) * as.c] : 0.0;
        const int c = b_cfast ? e & 63 : e >> 4, kb = b_cfast ? e >> 6 : e & 15;
        rb[q] = (k0 + kb < Q && c0 + c < Pc) ? B[(long long)(k0 + kb) * bs.r + (long long)(c0 + c) * bs.c] : 0.0;
      }
    };
    load(0);
    for (int k0 = 0; k0 < Q; k0 += kSgK) {
      __syncthreads();  // the previous chunk's fragments are consumed
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = tid + q * kSeamThreads;
        const int i = a_kfast ? e >> 4 : e & 63, kk = a_kfast ? e & 15 : e >> 6;
        At[i * kSgLA + kk] = ra[q];
        const int c = b_cfast ? e & 63 : e >> 4, kb = b_cfast ? e >> 6 : e & 15;
        Bt[kb * kSgLB + c] = rb[q];
      }
      __syncthreads();
      if (k0 + kSgK < Q) load(k0 + kSgK);
#pragma unroll
      for (int ks = 0; ks < kSgK; ks += 4) {
        double af[4], bf[2];
#pragma unroll
        for (int ti = 0; ti < 4; ++ti) af[ti] = At[(wr + ti * 8 + (lane >> 2)) * kSgLA + ks + (lane & 3)];
#pragma unroll
        for (int tj = 0; tj < 2; ++tj) bf[tj] = Bt[(ks + (lane & 3)) * kSgLB + wc + tj * 8 + (lane >> 2)];
#pragma unroll
        for (int ti = 0; ti < 4; ++ti)
#pragma unroll
          for (int tj = 0; tj < 2; ++tj) dmma(acc[ti][tj], af[ti], bf[tj]);
      }
    }
  }
  double* O = out + m * os.k;
#pragma unroll
  for (int ti = 0; ti < 4; ++ti) {
    const int r = r0 + wr + ti * 8 + (lane >> 2);
    if (r >= M) continue;
#pragma unroll
    for (int tj = 0; tj < 2; ++tj)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = c0 + wc + tj * 8 + 2 * (lane & 3) + h;
        if (c >= Pc) continue;
        double& o = O[(long long)r * os.r + (long long)c * os.c];
        if (alpha == 0.0) {
          if (beta == 0.0) o = 0.0;
          else if (beta != 1.0) o *= beta;
        } else {
          const double prod = alpha == 1.0 ? acc[ti][tj][h] : acc[ti][tj][h] * alpha;
          o = beta == 0.0 ? prod : (beta == 1.0 ? o : o * beta) + prod;
        }
      }
  }
}

}  // namespace btd
