// Streaming per-level solve (one CTA "team" per segment, persistent over segments).
//
// Same algebra as btd_solve.cuh (down: w = A_uu^{-1} b_u, fold f_L = C_L^T w_0, f_R = C_R w_last;
// up: b_0 -= C_L x_L, b_last -= C_R^T x_R, then forward/backward sweep), but built for HBM
// bandwidth: every block the sweep needs is streamed global->shared by a TMA producer warp through
// an mbarrier ring that runs ahead of the arithmetic across segment boundaries, and the inverse diagonal
// factors are read in packed lower-triangular form (n(n+1)/2 instead of n^2 doubles).  The
// backward sweep re-reads a segment's blocks right after the forward sweep, so they come from L2.
//
// Step streams (one step = at most one full n x n block + one packed block + one n x d panel):
//   down : F_0 .. F_{J-1}, B_{J-1}, CR, B_{J-2} .. B_0, CL
//   up   : CL, F_0 .. F_{J-2}, CR, F_{J-1}, B_{J-1} .. B_0
// F_j: t = b_j - L_{j,j-1} z_{j-1} (- boundary terms), z_j = Linv_j t
// B_j: t = z_j - L_{j+1,j}^T w_{j+1}, w_j = Linv_j^T t
#pragma once

#include "btd_device.cuh"
#include "btd_solve.cuh"

namespace btd {

template <int NT>
struct Solve2Shape {
  static constexpr int NTHREADS = 4 * NT;   // 4 threads per output row / column
  static constexpr int PARTS = 4;
  static constexpr int SPAN = NT / PARTS;  // inner-product slice per thread
  static constexpr int FULL = NT * NT;
  static constexpr int PACK = (NT & 1) ? 2 * (NT / 2 + 1) * (NT / 2 + 1) : 2 * (NT / 2) * (NT / 2 + 1);
  static constexpr int STAGES = NT == 64 ? 3 : NT == 32 ? 4 : 6;
  static constexpr int ZMAX = 16;  // longest segment served from the z cache in shared memory
};

// Packed lower-triangular storage of the inverse Cholesky factors.  Row r holds columns 0..r,
// padded with zeros to an even length so every row starts 16-byte aligned (vector loads):
//   row length L_r = 2 ceil((r+1)/2),  offset O_r = sum_{i<r} L_i  (= 2k(k+1) for r = 2k,
//   2(k+1)^2 for r = 2k+1);  block stride O_n (n = 64: 2112 doubles instead of 4096).
__host__ __device__ __forceinline__ int packed_row_offset(int r) {
  const int k = r >> 1;
  return (r & 1) ? 2 * (k + 1) * (k + 1) : 2 * k * (k + 1);
}
__host__ __device__ __forceinline__ int packed_stride(int n) { return packed_row_offset(n); }

enum StepKind : int { kStepF = 0, kStepB = 1, kStepCL = 2, kStepCR = 3, kStepNone = 4 };

// ============================================================================================
// Producer/consumer version (n == NT, n even): warp NCW (the last warp) streams the step blocks
// with TMA 1D bulk copies (cp.async.bulk, SASS UBLKCP) into a ring of STAGES slots guarded by
// full/empty mbarriers, running ahead across segment boundaries; warps [0, NCW) compute with
// vectorised, bank-rotated shared-memory mat-vecs.  Consumer barriers are named barrier 1.
// ============================================================================================
template <int NT>
__device__ __forceinline__ void csync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(4 * NT) : "memory");
}

__device__ __forceinline__ int nsteps(int mode, int J) { return mode == kSolveBase ? 2 * J : 2 * J + 2; }

__device__ __forceinline__ void step_kind(int mode, int J, int idx, int& kind, int& j) {
  if (mode == kSolveBase) {
    if (idx < J) kind = kStepF, j = idx;
    else kind = kStepB, j = 2 * J - 1 - idx;
  } else if (mode == kSolveDown) {
    if (idx < J) kind = kStepF, j = idx;
    else if (idx == J) kind = kStepB, j = J - 1;
    else if (idx == J + 1) kind = kStepCR, j = J - 1;
    else if (idx < 2 * J + 1) kind = kStepB, j = 2 * J - idx;
    else kind = kStepCL, j = 0;
  } else {
    if (idx == 0) kind = kStepCL, j = 0;
    else if (idx < J) kind = kStepF, j = idx - 1;
    else if (idx == J) kind = kStepCR, j = J - 1;
    else if (idx == J + 1) kind = kStepF, j = J - 1;
    else kind = kStepB, j = 2 * J + 1 - idx;
  }
}

// y (+)= sign * M x, M dense NT x NT (row-major, shared), x NT x DC
template <int NT, int DC>
__device__ __forceinline__ void fmv_full(const double* __restrict__ M, const double* __restrict__ x, double* y,
                                         double sign, bool acc_into) {
  constexpr int SPAN = NT / 4, NP = SPAN / 2, PM = NP - 1;
  const int tid = threadIdx.x, r = tid >> 2, part = tid & 3;
  const double* Mr = M + r * NT + part * SPAN;
  const double* xp = x + part * SPAN * DC;
  double a0[DC], a1[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) a0[c] = a1[c] = 0.0;
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const int qq = (q + r + 2 * part) & PM;
    const double2 v = *reinterpret_cast<const double2*>(Mr + 2 * qq);
    if (DC == 1) {
      const double2 xv = *reinterpret_cast<const double2*>(xp + 2 * qq);
      a0[0] = fma(v.x, xv.x, a0[0]);
      a1[0] = fma(v.y, xv.y, a1[0]);
    } else {
#pragma unroll
      for (int c = 0; c < DC; ++c) {
        a0[c] = fma(v.x, xp[(2 * qq) * DC + c], a0[c]);
        a1[c] = fma(v.y, xp[(2 * qq + 1) * DC + c], a1[c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < DC; ++c) {
    double t = a0[c] + a1[c];
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    t += __shfl_xor_sync(0xffffffffu, t, 2);
    if (part == 0) y[r * DC + c] = acc_into ? fma(sign, t, y[r * DC + c]) : sign * t;
  }
}

// y = Lp x (packed lower, zero padded rows)
template <int NT, int DC>
__device__ __forceinline__ void fmv_pack(const double* __restrict__ P, const double* __restrict__ x, double* y) {
  constexpr int SPAN = NT / 4, NP = SPAN / 2, PM = NP - 1;
  const int tid = threadIdx.x, r = tid >> 2, part = tid & 3;
  const double* row = P + packed_row_offset(r);
  const int npr = (r + 2) >> 1;  // pairs in row r
  const double* xp = x;
  double a0[DC], a1[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) a0[c] = a1[c] = 0.0;
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const int pq = part * NP + ((q + r + 2 * part) & PM);
    if (pq < npr) {
      const double2 v = *reinterpret_cast<const double2*>(row + 2 * pq);
      if (DC == 1) {
        const double2 xv = *reinterpret_cast<const double2*>(xp + 2 * pq);
        a0[0] = fma(v.x, xv.x, a0[0]);
        a1[0] = fma(v.y, xv.y, a1[0]);
      } else {
#pragma unroll
        for (int c = 0; c < DC; ++c) {
          a0[c] = fma(v.x, xp[(2 * pq) * DC + c], a0[c]);
          a1[c] = fma(v.y, xp[(2 * pq + 1) * DC + c], a1[c]);
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < DC; ++c) {
    double t = a0[c] + a1[c];
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    t += __shfl_xor_sync(0xffffffffu, t, 2);
    if (part == 0) y[r * DC + c] = t;
  }
}

// y (+)= sign * M^T x (dense) ; 4 row slices reduced through `red`
template <int NT, int DC>
__device__ __forceinline__ void fmv_full_t(const double* __restrict__ M, const double* __restrict__ x, double* y,
                                           double sign, bool acc_into, double* red) {
  constexpr int SPAN = NT / 4;
  const int tid = threadIdx.x, col = tid % NT, part = tid / NT;
  double a0[DC], a1[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) a0[c] = a1[c] = 0.0;
#pragma unroll
  for (int i = 0; i < SPAN; i += 2) {
    const int m = part * SPAN + i;
    const double v0 = M[m * NT + col], v1 = M[(m + 1) * NT + col];
#pragma unroll
    for (int c = 0; c < DC; ++c) {
      a0[c] = fma(v0, x[m * DC + c], a0[c]);
      a1[c] = fma(v1, x[(m + 1) * DC + c], a1[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < DC; ++c) red[(part * NT + col) * DC + c] = a0[c] + a1[c];
  csync<NT>();
  if (part == 0) {
#pragma unroll
    for (int c = 0; c < DC; ++c) {
      const double s4 = (red[col * DC + c] + red[(NT + col) * DC + c]) +
                        (red[(2 * NT + col) * DC + c] + red[(3 * NT + col) * DC + c]);
      y[col * DC + c] = acc_into ? fma(sign, s4, y[col * DC + c]) : sign * s4;
    }
  }
}

// y = Lp^T x
template <int NT, int DC>
__device__ __forceinline__ void fmv_pack_t(const double* __restrict__ P, const double* __restrict__ x, double* y,
                                           double* red) {
  constexpr int SPAN = NT / 4;
  const int tid = threadIdx.x, col = tid % NT, part = tid / NT;
  double a0[DC], a1[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) a0[c] = a1[c] = 0.0;
#pragma unroll
  for (int i = 0; i < SPAN; i += 2) {
    const int m = part * SPAN + i;
    if (m + 1 >= col) {  // rows m, m+1 (row m contributes only if m >= col; its pad is zero)
      const double v0 = (m >= col) ? P[packed_row_offset(m) + col] : 0.0;
      const double v1 = P[packed_row_offset(m + 1) + col];
#pragma unroll
      for (int c = 0; c < DC; ++c) {
        a0[c] = fma(v0, x[m * DC + c], a0[c]);
        a1[c] = fma(v1, x[(m + 1) * DC + c], a1[c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < DC; ++c) red[(part * NT + col) * DC + c] = a0[c] + a1[c];
  csync<NT>();
  if (part == 0) {
#pragma unroll
    for (int c = 0; c < DC; ++c)
      y[col * DC + c] = (red[col * DC + c] + red[(NT + col) * DC + c]) +
                        (red[(2 * NT + col) * DC + c] + red[(3 * NT + col) * DC + c]);
  }
}

template <int NT, int DC>
struct TmaShape {
  using S = Solve2Shape<NT>;
  static constexpr int NCW = S::NTHREADS / 32;  // consumer warps
  static constexpr int NTHREADS = S::NTHREADS + 32;
#ifndef BTD_TMA_STAGES64
#define BTD_TMA_STAGES64 4
#endif
  static constexpr int STAGES = NT == 64 ? (DC > 1 ? 3 : BTD_TMA_STAGES64) : 8;
  static constexpr int STAGE = S::FULL + S::PACK + NT * DC;  // doubles per slot
  static constexpr size_t SMEM = sizeof(double) * ((size_t)STAGES * STAGE + (size_t)(4 + S::ZMAX + S::PARTS) * NT * DC) +
                                 2 * STAGES * sizeof(unsigned long long);
};

template <int NT, int DC>
__global__ void __launch_bounds__(TmaShape<NT, DC>::NTHREADS) solve_tma_kernel(SolveArgs a) {
  using S = Solve2Shape<NT>;
  using T = TmaShape<NT, DC>;
  constexpr int STAGES = T::STAGES, STAGE = T::STAGE, NTH = S::NTHREADS;
  extern __shared__ __align__(16) double smem[];
  double* ring = smem;
  double* t = ring + STAGES * STAGE;
  double* u = t + NT * DC;
  double* corr = u + NT * DC;
  double* zc = corr + 2 * NT * DC;
  double* red = zc + S::ZMAX * NT * DC;
  unsigned long long* full_bar = reinterpret_cast<unsigned long long*>(red + S::PARTS * NT * DC);
  unsigned long long* empty_bar = full_bar + STAGES;
  if (error_raised(a.err)) return;
  const int n = NT, d = a.d, mode = a.mode;
  const int c0 = blockIdx.y * DC, dc = min(DC, d - c0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t ps = (size_t)n * d, bs = (size_t)n * n, pk = (size_t)S::PACK;
  // the rhs panel of one block row is contiguous when the CTA covers all d columns
  const bool vec_bulk = (c0 == 0 && dc == d && ((n * d) & 1) == 0);
  const int K = mode == kSolveBase ? 1 : a.K;

  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], T::NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == T::NCW) {
    // ===================== producer warp (one elected lane) =====================
    if (lane == 0) {
      int slot = 0;
      unsigned phase = 0;
      constexpr unsigned fb = NT * NT * sizeof(double), pb = S::PACK * sizeof(double);
      const unsigned vb = (unsigned)(n * d * sizeof(double));
      for (int k = blockIdx.x; k < K; k += gridDim.x) {
        const long long start = mode == kSolveBase ? 0 : (long long)a.seps[k] + 1;
        const long long stop = mode == kSolveBase ? a.N : (long long)a.seps[k + 1];
        const int J = (int)(stop - start);
        const int ns = nsteps(mode, J);
        for (int idx = 0; idx < ns; ++idx) {
          int kind, j;
          step_kind(mode, J, idx, kind, j);
          const long long row = start + j;
          const double *full = nullptr, *pack = nullptr, *vec = nullptr;
          if (kind == kStepF) {
            pack = a.Linv + row * pk;
            if (j > 0) full = a.Lsub + (row - 1) * bs;
            vec = a.rhs + row * ps;
          } else if (kind == kStepB) {
            pack = a.Linv + row * pk;
            if (j < J - 1) full = a.Lsub + row * bs;
          } else if (kind == kStepCL) {
            full = a.Lsub + (start - 1) * bs;
            if (mode == kSolveUp) vec = a.xsep + (size_t)k * ps;
          } else {
            full = a.Lsub + (stop - 1) * bs;
            if (mode == kSolveUp) vec = a.xsep + (size_t)(k + 1) * ps;
          }
          if (!vec_bulk) vec = nullptr;
          mbar_wait(&empty_bar[slot], phase ^ 1);
          double* st = ring + slot * STAGE;
          mbar_arrive_expect_tx(&full_bar[slot], (full ? fb : 0) + (pack ? pb : 0) + (vec ? vb : 0));
          if (full) tma_load_1d(st, full, fb, &full_bar[slot]);
          if (pack) tma_load_1d(st + S::FULL, pack, pb, &full_bar[slot]);
          if (vec) tma_load_1d(st + S::FULL + S::PACK, vec, vb, &full_bar[slot]);
          if (++slot == STAGES) {
            slot = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  // ===================== consumer warps =====================
  int slot = 0;
  unsigned phase = 0;
  for (int k = blockIdx.x; k < K; k += gridDim.x) {
    const long long start = mode == kSolveBase ? 0 : (long long)a.seps[k] + 1;
    const long long stop = mode == kSolveBase ? a.N : (long long)a.seps[k + 1];
    const int J = (int)(stop - start);
    const int ns = nsteps(mode, J);
    for (int idx = 0; idx < ns; ++idx) {
      int kind, j;
      step_kind(mode, J, idx, kind, j);
      const long long row = start + j;
      mbar_wait(&full_bar[slot], phase);
      const double* sf = ring + slot * STAGE;
      const double* sp = sf + S::FULL;
      const double* sv = sp + S::PACK;
      if (kind == kStepF) {
        for (int e = tid; e < NT * DC; e += NTH) {
          const int r = e / DC, c = e % DC;
          double v = 0.0;
          if (c < dc) v = vec_bulk ? sv[r * d + c] : a.rhs[row * ps + (size_t)r * d + c0 + c];
          if (mode == kSolveUp) {
            if (j == 0) v -= corr[e];
            if (j == J - 1) v -= corr[NT * DC + e];
          }
          t[e] = v;
        }
        csync<NT>();
        if (j > 0) {
          fmv_full<NT, DC>(sf, u, t, -1.0, true);
          csync<NT>();
        }
        fmv_pack<NT, DC>(sp, t, u);  // z_j -> u
        csync<NT>();
        double* zdst = j < S::ZMAX ? zc + j * NT * DC : nullptr;
        for (int e = tid; e < NT * DC; e += NTH) {
          if (zdst) zdst[e] = u[e];
          else if ((e % DC) < dc) a.x[row * ps + (size_t)(e / DC) * d + c0 + e % DC] = u[e];
        }
      } else if (kind == kStepB) {
        const double* zsrc = j < S::ZMAX ? zc + j * NT * DC : nullptr;
        for (int e = tid; e < NT * DC; e += NTH) {
          const int r = e / DC, c = e % DC;
          t[e] = zsrc ? zsrc[e] : (c < dc ? a.x[row * ps + (size_t)r * d + c0 + c] : 0.0);
        }
        csync<NT>();
        if (j < J - 1) {
          fmv_full_t<NT, DC>(sf, u, t, -1.0, true, red);
          csync<NT>();
        }
        fmv_pack_t<NT, DC>(sp, t, u, red);  // w_j -> u
        csync<NT>();
        if (mode != kSolveDown) {
          for (int e = tid; e < NT * DC; e += NTH)
            if ((e % DC) < dc) a.x[row * ps + (size_t)(e / DC) * d + c0 + e % DC] = u[e];
        }
      } else if (mode == kSolveDown) {  // fold: f_R = C_R w_last ; f_L = C_L^T w_0
        if (kind == kStepCR)
          fmv_full<NT, DC>(sf, u, t, 1.0, false);
        else
          fmv_full_t<NT, DC>(sf, u, t, 1.0, false, red);
        csync<NT>();
        double* dst = (kind == kStepCR ? a.fr : a.fl) + (size_t)k * ps;
        for (int e = tid; e < NT * DC; e += NTH)
          if ((e % DC) < dc) dst[(size_t)(e / DC) * d + c0 + e % DC] = t[e];
      } else {  // up: boundary corrections C_L x_L -> corr[0], C_R^T x_R -> corr[1]
        const double* xs = a.xsep + (size_t)(kind == kStepCL ? k : k + 1) * ps;
        for (int e = tid; e < NT * DC; e += NTH) {
          const int r = e / DC, c = e % DC;
          t[e] = c < dc ? (vec_bulk ? sv[r * d + c] : xs[(size_t)r * d + c0 + c]) : 0.0;
        }
        csync<NT>();
        if (kind == kStepCL)
          fmv_full<NT, DC>(sf, t, corr, 1.0, false);
        else
          fmv_full_t<NT, DC>(sf, t, corr + NT * DC, 1.0, false, red);
        for (int e = tid; e < NT * DC; e += NTH) {
          if ((e % DC) >= dc) continue;
          const size_t off = (size_t)(e / DC) * d + c0 + e % DC;
          if (kind == kStepCL) a.x[(size_t)(start - 1) * ps + off] = t[e];
          if (kind == kStepCR && k == K - 1) a.x[(size_t)stop * ps + off] = t[e];
        }
      }
      csync<NT>();  // slot and work panels fully consumed
      if (lane == 0) mbar_arrive(&empty_bar[slot]);
      if (++slot == STAGES) {
        slot = 0;
        phase ^= 1;
      }
    }
  }
}

}  // namespace btd
