// Kalman MAP-smoothing normal equations on the device: replaces
// build_normal_equations (bt/kalman.py:130-162) and _observation_terms (bt/kalman.py:105-127).
//
//   A[k,k]   = Q_k^-1 + H_k^T R_k^-1 H_k + G_{k+1}^T Q_{k+1}^-1 G_{k+1}
//   A[k+1,k] = -Q_{k+1}^-1 G_{k+1}
//   b[k]     = H_k^T R_k^-1 z_k + G_k^T Q_k^-1 zeta_k
// with every inverse realised through a Cholesky factor (never an explicit inverse of Q or R
// outside the CTA).  One CTA per time step k (n <= 64; dense R: m <= 64, diagonal R: any m):
//   kernel 1: chol(Q_k) -> Linv_Q (shared memory), Q^-1 = Linv^T Linv, Q^-1 G_k, Q^-1 zeta_k, the
//             observation terms (diagonal R: weights 1/r; dense R: chol(R_k), whitened H and z),
//             diag[k] = Q^-1 + H^T R^-1 H, cross[k] = G_k^T Q^-1 G_k, sub[k-1] = -Q^-1 G_k, rhs[k]
//   kernel 2: diag[k] += cross[k+1], then (D + D^T)/2 (new_btd symmetrisation, bt/core.py:211) --
//             the same summation order as the reference's loop.
// Failures: the first time step k whose process covariance (then measurement covariance) is not
// positive definite, with the 1-based pivot (NotPositiveDefinite(pivot, block=k, context=...)).
#pragma once

#include "btd_device.cuh"

namespace btd {

constexpr int kKalmanThreads = 256;
constexpr int kKalmanMaxN = 64;
constexpr int kKalmanMaxDenseM = 64;

struct KalmanArgs {
  const double* transition;   // (N, n, n)
  const double* observation;  // (N, m, n), or one (m, n) block if shared_h
  const double* process_cov;  // (N, n, n), or one block if shared_q
  const double* meas_cov;     // (N, m, m) dense / (N, m) diagonal, or one if shared_r
  const double* observations; // (N, m)
  const double* prior;        // (N, n)
  long long N;
  int n, m;
  int diag_r, shared_h, shared_q, shared_r;
  double* diag;   // (N, n, n) out
  double* sub;    // (N-1, n, n) out
  double* rhs;    // (N, n) out
  double* cross;  // (N, n, n) scratch: G_k^T Q_k^-1 G_k
  unsigned long long* err;  // min over failures of (k << 20) | (kind << 16) | pivot ; ~0 = none
};

// In-place lower Cholesky of an n x n shared tile (row stride ld) by the whole CTA, one column at a
// time (n <= 64: latency is fine, the per-step work is tiny).  Returns the 1-based failing pivot or 0
// (test `d <= 0` as LAPACK: NaN passes silently).  Also leaves 1/L_ii in rinv[i].
__device__ int chol_cta(double* A, int n, int ld, double* rinv, int* s_fail) {
  const int tid = threadIdx.x;
  if (tid == 0) *s_fail = 0;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const double d = A[k * ld + k];
    if (d <= 0.0) {
      if (tid == 0 && *s_fail == 0) *s_fail = k + 1;
    }
    const double ri = rsqrt(d);
    __syncthreads();
    if (*s_fail) return *s_fail;
    // column k below the diagonal
    for (int i = k + 1 + tid; i < n; i += blockDim.x) A[i * ld + k] *= ri;
    if (tid == 0) {
      A[k * ld + k] = d * ri;
      rinv[k] = ri;
    }
    __syncthreads();
    // trailing update of the lower triangle
    const int m = n - k - 1;
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int i = k + 1 + e / m, j = k + 1 + e % m;
      if (j <= i) A[i * ld + j] -= A[i * ld + k] * A[j * ld + k];
    }
    __syncthreads();
  }
  return 0;
}

// Linv = L^{-1} (lower), one thread per column, forward substitution; written to Li (stride ld).
__device__ void trinv_cta(const double* L, const double* rinv, double* Li, int n, int ld) {
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    for (int i = 0; i < n; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int q = c; q < i; ++q) s -= L[i * ld + q] * Li[q * ld + c];
      Li[i * ld + c] = (i >= c) ? s * rinv[i] : 0.0;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void report_kalman(unsigned long long* err, long long k, int kind, int pivot) {
  const unsigned long long key = ((unsigned long long)k << 20) | ((unsigned long long)kind << 16) |
                                 (unsigned long long)(pivot & 0xffff);
  atomicMin(err, key);
}

// dynamic shared memory (doubles) of kalman_terms_kernel for (n, m, dense R)
__host__ __device__ __forceinline__ size_t kalman_smem_doubles(int n, int m, int dense_r) {
  const size_t ld = (size_t)n + 1;
  size_t d = 4 * (size_t)n * ld + 4 * kKalmanMaxN;
  if (dense_r) d += (size_t)m * (m + 1) + (size_t)m * ld;
  return d;
}

__global__ void __launch_bounds__(kKalmanThreads) kalman_terms_kernel(KalmanArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_fail;
  const long long k = blockIdx.x;
  const int n = a.n, m = a.m, tid = threadIdx.x, T = blockDim.x;
  const int ld = n + 1, ldr = m + 1;
  double* Q = sm;             // n x ld : Q -> L_Q
  double* Li = Q + n * ld;    // n x ld : L_Q^{-1}
  double* Qi = Li + n * ld;   // n x ld : Q^{-1}
  double* QG = Qi + n * ld;   // n x ld : Q^{-1} G_k
  double* vec = QG + n * ld;  // 4 x 64 : zeta | Q^-1 zeta | 1/L_ii | H^T R^-1 z
  double* Rf = vec + 4 * kKalmanMaxN;  // dense R: m x ldr (R -> L_R)
  double* WH = Rf + m * ldr;           // dense R: m x ld  (L_R^{-1} [H | z])
  const size_t nn = (size_t)n * n;
  const double* G = a.transition + k * nn;
  const double* Qg = a.process_cov + (a.shared_q ? 0 : k * nn);
  const double* H = a.observation + (a.shared_h ? 0 : k * (size_t)m * n);

  // ---- process covariance ----
  for (int e = tid; e < n * n; e += T) Q[(e / n) * ld + e % n] = Qg[e];
  if (tid < n) vec[tid] = a.prior[k * n + tid];
  __syncthreads();
  double* rinv = vec + 2 * kKalmanMaxN;
  const int fq = chol_cta(Q, n, ld, rinv, &s_fail);
  if (fq) {
    if (tid == 0) report_kalman(a.err, k, 0, fq);
    return;
  }
  trinv_cta(Q, rinv, Li, n, ld);
  // Q^{-1} = Li^T Li
  for (int e = tid; e < n * n; e += T) {
    const int i = e / n, j = e % n;
    double s = 0.0;
    for (int q = max(i, j); q < n; ++q) s += Li[q * ld + i] * Li[q * ld + j];
    Qi[i * ld + j] = s;
  }
  __syncthreads();
  // Q^{-1} G, Q^{-1} zeta
  for (int e = tid; e < n * n; e += T) {
    const int i = e / n, j = e % n;
    double s = 0.0;
    for (int q = 0; q < n; ++q) s += Qi[i * ld + q] * G[q * n + j];
    QG[i * ld + j] = s;
  }
  if (tid < n) {
    double s = 0.0;
    for (int q = 0; q < n; ++q) s += Qi[tid * ld + q] * vec[q];
    vec[kKalmanMaxN + tid] = s;
  }
  __syncthreads();

  // ---- observation terms: H^T R^-1 H (into the diag output) and H^T R^-1 z ----
  double* out = a.diag + k * nn;
  const double* z = a.observations + k * (size_t)m;
  double* htriz = vec + 3 * kKalmanMaxN;
  if (a.diag_r) {
    const double* r = a.meas_cov + (a.shared_r ? 0 : k * (size_t)m);
    // failure: first non-positive variance (bt/kalman.py:111-114)
    if (tid == 0) {
      int bad = 0;
      for (int i = 0; i < m; ++i)
        if (r[i] <= 0.0) {
          bad = i + 1;
          break;
        }
      s_fail = bad;
    }
    __syncthreads();
    if (s_fail) {
      if (tid == 0) report_kalman(a.err, k, 1, s_fail);
      return;
    }
    for (int e = tid; e < n * n; e += T) {
      const int i = e / n, j = e % n;
      double s = 0.0;
      for (int q = 0; q < m; ++q) s += H[q * n + i] * (H[q * n + j] / r[q]);
      out[e] = Qi[i * ld + j] + s;
    }
    if (tid < n) {
      double s = 0.0;
      for (int q = 0; q < m; ++q) s += H[q * n + tid] * (z[q] / r[q]);
      htriz[tid] = s;
    }
  } else {
    const double* R = a.meas_cov + (a.shared_r ? 0 : k * (size_t)m * m);
    for (int e = tid; e < m * m; e += T) Rf[(e / m) * ldr + e % m] = R[e];
    __syncthreads();
    double* rinv_r = vec + 2 * kKalmanMaxN;  // Q's 1/L_ii are no longer needed
    const int fr = chol_cta(Rf, m, ldr, rinv_r, &s_fail);
    if (fr) {
      if (tid == 0) report_kalman(a.err, k, 1, fr);
      return;
    }
    // whitened H (forward substitution per column) and whitened z (thread n)
    for (int c = tid; c <= n; c += T) {
      for (int i = 0; i < m; ++i) {
        double s = (c < n) ? H[i * n + c] : z[i];
        for (int q = 0; q < i; ++q) s -= Rf[i * ldr + q] * WH[q * ld + c];
        WH[i * ld + c] = s * rinv_r[i];
      }
    }
    __syncthreads();
    for (int e = tid; e < n * n; e += T) {
      const int i = e / n, j = e % n;
      double s = 0.0;
      for (int q = 0; q < m; ++q) s += WH[q * ld + i] * WH[q * ld + j];
      out[e] = Qi[i * ld + j] + s;
    }
    __syncthreads();
    if (tid < n) {
      double s = 0.0;
      for (int q = 0; q < m; ++q) s += WH[q * ld + tid] * WH[q * ld + n];
      htriz[tid] = s;
    }
  }
  __syncthreads();
  // rhs[k] = H^T R^-1 z + G_k^T Q^-1 zeta ;  sub[k-1] = -Q^-1 G ;  cross[k] = G^T Q^-1 G
  if (tid < n) {
    double s = 0.0;
    for (int q = 0; q < n; ++q) s += G[q * n + tid] * vec[kKalmanMaxN + q];
    a.rhs[k * n + tid] = htriz[tid] + s;
  }
  for (int e = tid; e < n * n; e += T) {
    const int i = e / n, j = e % n;
    if (k > 0) a.sub[(k - 1) * nn + e] = -QG[i * ld + j];
    double s = 0.0;
    for (int q = 0; q < n; ++q) s += G[q * n + i] * QG[q * ld + j];
    a.cross[k * nn + e] = s;
  }
}

// diag[k] += cross[k+1] (k < N-1), then symmetrise (D + D^T)/2.
__global__ void kalman_finish_kernel(double* diag, const double* cross, long long N, int n,
                                     const unsigned long long* err) {
  if (*((volatile const unsigned long long*)err) != kNoErr) return;
  const size_t nn = (size_t)n * n;
  const size_t total = (size_t)N * nn;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const long long k = (long long)(e / nn);
    const int i = (int)((e % nn) / n), j = (int)(e % n);
    if (j < i) continue;  // each (i, j) / (j, i) pair once
    const size_t t = (size_t)k * nn + (size_t)j * n + i;
    double a = diag[e], b = diag[t];
    if (k + 1 < N) {
      a += cross[e + nn];
      b += cross[t + nn];
    }
    const double s = (a + b) / 2.0;
    diag[e] = s;
    diag[t] = s;
  }
}

}  // namespace btd
