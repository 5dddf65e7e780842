// Streaming per-level solve (one CTA "team" per segment, persistent over segments).
//
// Same algebra as btd_solve.cuh (down: w = A_uu^{-1} b_u, fold f_L = C_L^T w_0, f_R = C_R w_last;
// up: b_0 -= C_L x_L, b_last -= C_R^T x_R, then forward/backward sweep), but built for HBM
// bandwidth: every block the sweep needs is streamed global->shared through a STAGES-deep cp.async
// ring that runs ahead of the arithmetic across segment boundaries, and the inverse diagonal
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
  static constexpr int PACK = (NT * (NT + 1) / 2 + 1) / 2 * 2;
  static constexpr int STAGES = NT == 64 ? 3 : NT == 32 ? 4 : 6;
  static constexpr int ZMAX = 16;  // longest segment served from the z cache in shared memory
};

// packed lower-triangular stride (doubles) of a block of order n: n(n+1)/2 rounded up to even
__host__ __device__ __forceinline__ int packed_stride(int n) { return (n * (n + 1) / 2 + 1) / 2 * 2; }

enum StepKind : int { kStepF = 0, kStepB = 1, kStepCL = 2, kStepCR = 3, kStepNone = 4 };

struct StepDesc {
  const double* full;  // n x n (Lsub or coupling block), or nullptr
  const double* pack;  // packed Linv, or nullptr
  const double* vec;   // n x d panel (rhs row or separator solution), or nullptr
  int kind, j;
};

// Step `idx` of segment k.  Returns false past the end of the segment's stream.
__device__ __forceinline__ bool make_step(const SolveArgs& a, int k, int idx, StepDesc& s, int& J_out) {
  const long long start = (long long)a.seps[k] + 1, stop = (long long)a.seps[k + 1];
  const int J = (int)(stop - start);
  J_out = J;
  const size_t bs = (size_t)a.n * a.n, ps = (size_t)a.n * a.d, pk = (size_t)packed_stride(a.n);
  if (idx >= 2 * J + 2) return false;
  s.full = s.pack = s.vec = nullptr;
  int kind, j;
  if (a.mode == kSolveDown) {
    if (idx < J) {
      kind = kStepF, j = idx;
    } else if (idx == J) {
      kind = kStepB, j = J - 1;
    } else if (idx == J + 1) {
      kind = kStepCR, j = J - 1;
    } else if (idx < 2 * J + 1) {
      kind = kStepB, j = J - 2 - (idx - J - 2);
    } else {
      kind = kStepCL, j = 0;
    }
  } else {  // up
    if (idx == 0) {
      kind = kStepCL, j = 0;
    } else if (idx < J) {
      kind = kStepF, j = idx - 1;  // F_0 .. F_{J-2}
    } else if (idx == J) {
      kind = kStepCR, j = J - 1;
    } else if (idx == J + 1) {
      kind = kStepF, j = J - 1;
    } else {
      kind = kStepB, j = J - 1 - (idx - J - 2);
    }
  }
  const long long row = start + j;
  if (kind == kStepF) {
    s.pack = a.Linv + row * pk;
    if (j > 0) s.full = a.Lsub + (row - 1) * bs;
    s.vec = a.rhs + row * ps;
  } else if (kind == kStepB) {
    s.pack = a.Linv + row * pk;
    if (j < J - 1) s.full = a.Lsub + row * bs;
  } else if (kind == kStepCL) {
    s.full = a.Lsub + (start - 1) * bs;
    if (a.mode == kSolveUp) s.vec = a.xsep + (size_t)k * ps;
  } else {
    s.full = a.Lsub + (stop - 1) * bs;
    if (a.mode == kSolveUp) s.vec = a.xsep + (size_t)(k + 1) * ps;
  }
  s.kind = kind;
  s.j = j;
  return true;
}

template <int NT, int DC>
__device__ __forceinline__ void issue_stage(double* st, const StepDesc& s, int n, int d, int c0, int dc) {
  using S = Solve2Shape<NT>;
  const int tid = threadIdx.x;
  double* sf = st;
  double* sp = st + S::FULL;
  double* sv = st + S::FULL + S::PACK;
  const bool even = (n & 1) == 0;
  if (s.full) {
    if (even) {
      for (int i = tid; i < n * n / 2; i += S::NTHREADS) cp_async16(sf + 2 * i, s.full + 2 * i, 16);
    } else {
      for (int i = tid; i < n * n; i += S::NTHREADS) cp_async8(sf + i, s.full + i, 8);
    }
  }
  if (s.pack) {
    const int np = packed_stride(n);
    for (int i = tid; i < np / 2; i += S::NTHREADS) cp_async16(sp + 2 * i, s.pack + 2 * i, 16);
  }
  if (s.vec) {
    for (int e = tid; e < n * DC; e += S::NTHREADS) {
      const int r = e / DC, c = e % DC;
      if (c < dc) cp_async8(sv + e, s.vec + (size_t)r * d + c0 + c, 8);
    }
  }
}

// y (+)= sign * M x   (M dense n x n, row stride n, in shared memory)
template <int NT, int DC>
__device__ __forceinline__ void mv_full(const double* M, const double* x, double* y, int n, double sign,
                                        bool accumulate) {
  using S = Solve2Shape<NT>;
  const int tid = threadIdx.x, r = tid / S::PARTS, part = tid % S::PARTS;
  double acc[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) acc[c] = 0.0;
  if (r < n) {
#pragma unroll 4
    for (int i = 0; i < S::SPAN; ++i) {
      const int m = part * S::SPAN + (i + r) % S::SPAN;  // rotated: conflict-free rows
      if (m < n) {
        const double v = M[r * n + m];
#pragma unroll
        for (int c = 0; c < DC; ++c) acc[c] = fma(v, x[m * DC + c], acc[c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < DC; ++c) {
    acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 1);
    acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 2);
  }
  if (part == 0 && r < NT) {
#pragma unroll
    for (int c = 0; c < DC; ++c) {
      const double v = r < n ? sign * acc[c] : 0.0;
      y[r * DC + c] = accumulate ? y[r * DC + c] + v : v;
    }
  }
}

// y (+)= sign * M^T x   (dense), reduction over the 4 row slices through `red`
template <int NT, int DC>
__device__ __forceinline__ void mv_full_t(const double* M, const double* x, double* y, int n, double sign,
                                          bool accumulate, double* red) {
  using S = Solve2Shape<NT>;
  const int tid = threadIdx.x, col = tid % NT, part = tid / NT;
  double acc[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) acc[c] = 0.0;
  if (col < n) {
#pragma unroll 4
    for (int i = 0; i < S::SPAN; ++i) {
      const int m = part * S::SPAN + i;
      if (m < n) {
        const double v = M[m * n + col];
#pragma unroll
        for (int c = 0; c < DC; ++c) acc[c] = fma(v, x[m * DC + c], acc[c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < DC; ++c) red[(part * NT + col) * DC + c] = acc[c];
  __syncthreads();
  if (part == 0) {
#pragma unroll
    for (int c = 0; c < DC; ++c) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < S::PARTS; ++q) s += red[(q * NT + col) * DC + c];
      const double v = col < n ? sign * s : 0.0;
      y[col * DC + c] = accumulate ? y[col * DC + c] + v : v;
    }
  }
}

// y = Lp x   (packed lower triangular: row r at r(r+1)/2)
template <int NT, int DC>
__device__ __forceinline__ void mv_pack(const double* P, const double* x, double* y, int n) {
  using S = Solve2Shape<NT>;
  const int tid = threadIdx.x, r = tid / S::PARTS, part = tid % S::PARTS;
  double acc[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) acc[c] = 0.0;
  if (r < n) {
    const double* row = P + r * (r + 1) / 2;
#pragma unroll 4
    for (int i = 0; i < S::SPAN; ++i) {
      const int m = part * S::SPAN + (i + r) % S::SPAN;
      if (m <= r) {
        const double v = row[m];
#pragma unroll
        for (int c = 0; c < DC; ++c) acc[c] = fma(v, x[m * DC + c], acc[c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < DC; ++c) {
    acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 1);
    acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 2);
  }
  if (part == 0 && r < NT) {
#pragma unroll
    for (int c = 0; c < DC; ++c) y[r * DC + c] = r < n ? acc[c] : 0.0;
  }
}

// y = Lp^T x
template <int NT, int DC>
__device__ __forceinline__ void mv_pack_t(const double* P, const double* x, double* y, int n, double* red) {
  using S = Solve2Shape<NT>;
  const int tid = threadIdx.x, col = tid % NT, part = tid / NT;
  double acc[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) acc[c] = 0.0;
  if (col < n) {
#pragma unroll 4
    for (int i = 0; i < S::SPAN; ++i) {
      const int m = part * S::SPAN + i;
      if (m < n && m >= col) {
        const double v = P[m * (m + 1) / 2 + col];
#pragma unroll
        for (int c = 0; c < DC; ++c) acc[c] = fma(v, x[m * DC + c], acc[c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < DC; ++c) red[(part * NT + col) * DC + c] = acc[c];
  __syncthreads();
  if (part == 0) {
#pragma unroll
    for (int c = 0; c < DC; ++c) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < S::PARTS; ++q) s += red[(q * NT + col) * DC + c];
      y[col * DC + c] = col < n ? s : 0.0;
    }
  }
}

template <int NT, int DC>
__global__ void __launch_bounds__(Solve2Shape<NT>::NTHREADS) solve_stream_kernel(SolveArgs a) {
  using S = Solve2Shape<NT>;
  constexpr int STAGE = S::FULL + S::PACK + NT * DC;
  extern __shared__ __align__(16) double smem[];
  double* ring = smem;                                  // STAGES x STAGE
  double* t = ring + S::STAGES * STAGE;                 // NT x DC work panel
  double* u = t + NT * DC;                              // z_{j-1} / w_{j+1}
  double* corr = u + NT * DC;                           // up: boundary corrections (2 panels)
  double* zc = corr + 2 * NT * DC;                      // z cache: ZMAX panels
  double* red = zc + S::ZMAX * NT * DC;                 // PARTS x NT x DC
  if (error_raised(a.err)) return;
  const int n = a.n, d = a.d;
  const int c0 = blockIdx.y * DC, dc = min(DC, d - c0);
  const int tid = threadIdx.x;
  const size_t ps = (size_t)n * d;

  // producer cursor (segment kp, step ip) runs STAGES-1 steps ahead of the consumer
  int kp = blockIdx.x, ip = 0;
  auto produce = [&](int slot) {
    StepDesc s;
    int J;
    while (kp < a.K && !make_step(a, kp, ip, s, J)) {
      kp += gridDim.x;
      ip = 0;
    }
    if (kp < a.K) {
      issue_stage<NT, DC>(ring + slot * STAGE, s, n, d, c0, dc);
      ++ip;
    }
    cp_async_commit();  // (possibly empty) group per slot keeps the wait_group arithmetic uniform
  };
  for (int sidx = 0; sidx < S::STAGES - 1; ++sidx) produce(sidx);

  int slot = 0;
  for (int k = blockIdx.x; k < a.K; k += gridDim.x) {
    const long long start = (long long)a.seps[k] + 1, stop = (long long)a.seps[k + 1];
    const int J = (int)(stop - start);
    for (int idx = 0; idx < 2 * J + 2; ++idx) {
      StepDesc s;
      int Jd;
      make_step(a, k, idx, s, Jd);
      cp_async_wait_group<S::STAGES - 2>();
      __syncthreads();
      const double* sf = ring + slot * STAGE;
      const double* sp = sf + S::FULL;
      const double* sv = sp + S::PACK;
      const long long row = start + s.j;
      if (s.kind == kStepF) {
        // t = b_j - L_{j,j-1} z_{j-1} - (up) boundary corrections
        for (int e = tid; e < NT * DC; e += S::NTHREADS) {
          const int r = e / DC;
          double v = (r < n && (e % DC) < dc) ? sv[e] : 0.0;
          if (a.mode == kSolveUp) {
            if (s.j == 0) v -= corr[e];
            if (s.j == J - 1) v -= corr[NT * DC + e];
          }
          t[e] = v;
        }
        __syncthreads();
        if (s.j > 0) {
          mv_full<NT, DC>(sf, u, t, n, -1.0, true);
          __syncthreads();
        }
        mv_pack<NT, DC>(sp, t, u, n);  // z_j -> u
        __syncthreads();
        double* zdst = s.j < S::ZMAX ? zc + s.j * NT * DC : nullptr;
        for (int e = tid; e < NT * DC; e += S::NTHREADS) {
          if (zdst) zdst[e] = u[e];
          else if ((e / DC) < n && (e % DC) < dc) a.x[row * ps + (size_t)(e / DC) * d + c0 + e % DC] = u[e];
        }
      } else if (s.kind == kStepB) {
        const double* zsrc = s.j < S::ZMAX ? zc + s.j * NT * DC : nullptr;
        for (int e = tid; e < NT * DC; e += S::NTHREADS) {
          const int r = e / DC, c = e % DC;
          t[e] = zsrc ? zsrc[e] : ((r < n && c < dc) ? a.x[row * ps + (size_t)r * d + c0 + c] : 0.0);
        }
        __syncthreads();
        if (s.j < J - 1) {
          mv_full_t<NT, DC>(sf, u, t, n, -1.0, true, red);
          __syncthreads();
        }
        mv_pack_t<NT, DC>(sp, t, u, n, red);  // w_j -> u
        __syncthreads();
        if (a.mode == kSolveUp) {
          for (int e = tid; e < n * DC; e += S::NTHREADS)
            if ((e % DC) < dc) a.x[row * ps + (size_t)(e / DC) * d + c0 + e % DC] = u[e];
        }
      } else if (a.mode == kSolveDown) {  // fold: f_R = C_R w_last ; f_L = C_L^T w_0
        if (s.kind == kStepCR)
          mv_full<NT, DC>(sf, u, t, n, 1.0, false);
        else
          mv_full_t<NT, DC>(sf, u, t, n, 1.0, false, red);
        __syncthreads();
        double* dst = (s.kind == kStepCR ? a.fr : a.fl) + (size_t)k * ps;
        for (int e = tid; e < n * DC; e += S::NTHREADS)
          if ((e % DC) < dc) dst[(size_t)(e / DC) * d + c0 + e % DC] = t[e];
      } else {  // up: boundary corrections C_L x_L -> corr[0], C_R^T x_R -> corr[1]
        for (int e = tid; e < NT * DC; e += S::NTHREADS) t[e] = ((e / DC) < n && (e % DC) < dc) ? sv[e] : 0.0;
        __syncthreads();
        if (s.kind == kStepCL)
          mv_full<NT, DC>(sf, t, corr, n, 1.0, false);
        else
          mv_full_t<NT, DC>(sf, t, corr + NT * DC, n, 1.0, false, red);
        // separator rows of the solution come from the level below
        for (int e = tid; e < n * DC; e += S::NTHREADS) {
          if ((e % DC) >= dc) continue;
          const size_t off = (size_t)(e / DC) * d + c0 + e % DC;
          if (s.kind == kStepCL) a.x[(size_t)(start - 1) * ps + off] = t[e];
          if (s.kind == kStepCR && k == a.K - 1) a.x[(size_t)stop * ps + off] = t[e];
        }
      }
      __syncthreads();  // slot fully consumed
      produce(slot == 0 ? S::STAGES - 1 : slot - 1);
      slot = slot + 1 == S::STAGES ? 0 : slot + 1;
    }
  }
  cp_async_wait_group<0>();
}

}  // namespace btd
