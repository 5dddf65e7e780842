// Streaming per-level solve (one CTA "team" per segment, persistent over segments).
//
// Same algebra as btd_solve.cuh (down: w = A_uu^{-1} b_u, fold f_L = C_L^T w_0, f_R = C_R w_last;
// up: b_0 -= C_L x_L, b_last -= C_R^T x_R, then forward/backward sweep), but built for HBM
// bandwidth: every block the sweep needs is streamed global->shared by a TMA producer warp through
// an mbarrier ring that runs ahead of the arithmetic across segment boundaries, and the inverse diagonal
// factors are read in packed lower-triangular form (n(n+1)/2 instead of n^2 doubles).  The
// backward sweep re-reads a segment's blocks right after the forward sweep, so they come from L2
// (forward loads carry an L2 evict_last hint, last uses evict_first: with two segments in flight
// per SM on wide levels the re-read window is ~120 MB, close to the L2 size).
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

#ifdef BTD_PHASE_PROF
#define BTD_SPH(i)                                                          \
  do {                                                                      \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                              \
      long long _now = clock64();                                           \
      atomicAdd(&g_phase_cycles[i], (unsigned long long)(_now - _sp_last)); \
      _sp_last = _now;                                                      \
    }                                                                       \
  } while (0)
#else
#define BTD_SPH(i)
#endif

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
// vectorised, conflict-free shared-memory mat-vecs (two per step, one named barrier after each;
// each warp releases a slot on its own).  Consumer barriers are named barrier 1.
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

// Row form: s[c] = sum_m M[r][m] x[m][c] for the thread's row r = tid / 4 (valid on the 4 lanes
// of the row quad); rotated double2 reads keep the quad's rows conflict-free.
template <int NT, int DC>
__device__ __forceinline__ void mv_rows(const double* __restrict__ M, const double* __restrict__ x, double (&s)[DC]) {
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
#pragma unroll
    for (int c = 0; c < DC; ++c) {
      a0[c] = fma(v.x, xp[(2 * qq) * DC + c], a0[c]);
      a1[c] = fma(v.y, xp[(2 * qq + 1) * DC + c], a1[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < DC; ++c) {
    double v = a0[c] + a1[c];
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    s[c] = v;
  }
}

// Row form of the packed lower-triangular Linv: s[c] = sum_{m <= r} Lp[r][m] x[m][c].
template <int NT, int DC>
__device__ __forceinline__ void mv_pack_rows(const double* __restrict__ P, const double* __restrict__ x, double (&s)[DC]) {
  constexpr int SPAN = NT / 4, NP = SPAN / 2, PM = NP - 1;
  const int tid = threadIdx.x, r = tid >> 2, part = tid & 3;
  const double* row = P + packed_row_offset(r);
  const int npr = (r + 2) >> 1;  // pairs in row r
  double a0[DC], a1[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) a0[c] = a1[c] = 0.0;
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const int pq = part * NP + ((q + r + 2 * part) & PM);
    if (pq < npr) {
      const double2 v = *reinterpret_cast<const double2*>(row + 2 * pq);
#pragma unroll
      for (int c = 0; c < DC; ++c) {
        a0[c] = fma(v.x, x[(2 * pq) * DC + c], a0[c]);
        a1[c] = fma(v.y, x[(2 * pq + 1) * DC + c], a1[c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < DC; ++c) {
    double v = a0[c] + a1[c];
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    s[c] = v;
  }
}

// Transposed form on warps [0, NT/16): v[h][c] = sum_m M[m][col + h] x[m][c] for the column pair
// col = 16 warp + 2 (lane % 8).  A warp owns 16 columns: lane = pair + 8 part, part sweeping rows
// part, part + 4, ...; each row's 16 columns are one contiguous 128-byte run (conflict-free
// double2 reads), and the 4 parts are reduced with xor shuffles (result on every lane).
// PACKED: M is the packed lower triangle (only m >= col contributes; pairs past the row are skipped).
template <int NT, int DC, bool PACKED>
__device__ __forceinline__ void mtv(const double* __restrict__ M, const double* __restrict__ x, double (&v)[2][DC]) {
  constexpr int CW = NT < 16 ? NT : 16, PR = CW / 2, PT = 32 / PR;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int part = lane / PR, col = CW * w + 2 * (lane % PR);
  double a[2][2][DC];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < DC; ++c) a[0][h][c] = a[1][h][c] = 0.0;
#pragma unroll
  for (int i = 0; i < NT / PT; ++i) {
    const int m = part + PT * i;
    double2 e = make_double2(0.0, 0.0);
    if (!PACKED) e = *reinterpret_cast<const double2*>(M + m * NT + col);
    else if (col <= m) e = *reinterpret_cast<const double2*>(M + packed_row_offset(m) + col);
#pragma unroll
    for (int c = 0; c < DC; ++c) {
      const double xv = x[m * DC + c];
      a[i & 1][0][c] = fma(e.x, xv, a[i & 1][0][c]);
      a[i & 1][1][c] = fma(e.y, xv, a[i & 1][1][c]);
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < DC; ++c) {
      double s = a[0][h][c] + a[1][h][c];
#pragma unroll
      for (int o = PR; o < 32; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      v[h][c] = s;
    }
}

// Column stride of the d = 4 shared-memory vectors (x[c][kXLD]): 72, not 64, so the transposed
// product's one-value-per-lane stores (8 columns x 4 rhs columns per warp) fall in 2 wavefronts.
constexpr int kXLD = 72;

// Row form at NT == 64, DC == 4: warp w owns rows 8w..8w+7, lane half h = lane / 16 the rows
// 8w + 4h + i (i < 4), and lane q = lane % 16 the column pairs (2q, 2q+1) and (32+2q, 33+2q), so
// each half-warp reads one contiguous 256-byte run per load and holds 16 partials (4 rows x 4 rhs
// columns), reduced over the 16 lanes of the half by a transposing butterfly (8+4+2+1 shuffles,
// against 36 for mv64 at d = 4).  Lane l ends with row 8w + l / 4 (= tid / 4), rhs column l % 4.
template <bool PACKED>
__device__ __forceinline__ double mv64x4(const double* __restrict__ M, const double* __restrict__ x) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ca = 2 * (lane & 15), cb = 32 + ca, r0 = 8 * w + 4 * (lane >> 4);
  double2 xa[4], xb[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    xa[c] = *reinterpret_cast<const double2*>(x + c * kXLD + ca);
    xb[c] = *reinterpret_cast<const double2*>(x + c * kXLD + cb);
  }
  double a[16];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + i;
    double2 ea = make_double2(0.0, 0.0), eb = make_double2(0.0, 0.0);
    if (!PACKED) {
      ea = *reinterpret_cast<const double2*>(M + r * 64 + ca);
      eb = *reinterpret_cast<const double2*>(M + r * 64 + cb);
    } else {
      if (ca <= r) ea = *reinterpret_cast<const double2*>(M + packed_row_offset(r) + ca);
      if (cb <= r) eb = *reinterpret_cast<const double2*>(M + packed_row_offset(r) + cb);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
      a[i * 4 + c] = fma(eb.y, xb[c].y, fma(eb.x, xb[c].x, fma(ea.y, xa[c].y, ea.x * xa[c].x)));
  }
#pragma unroll
  for (int o = 8, h = 8; o >= 1; o >>= 1, h >>= 1) {
    const bool hi = lane & o;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k < h) {
        const double snd = hi ? a[k] : a[k + h], kp = hi ? a[k + h] : a[k];
        a[k] = kp + __shfl_xor_sync(0xffffffffu, snd, o);
      }
    }
  }
  return a[0];
}

// Row form at NT == 64, DC == 1 with mv64x4's half-warp row groups: 4 partials per lane, a
// transposing butterfly over lane bits 3, 2 then two plain levels (5 shuffles instead of mv64's 9);
// the total of row 8w + l / 4 (= tid / 4) ends on the 4 lanes of that row's quad (mv64's mapping).
template <bool PACKED>
__device__ __forceinline__ double mv64x1(const double* __restrict__ M, const double* __restrict__ x) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ca = 2 * (lane & 15), cb = 32 + ca, r0 = 8 * w + 4 * (lane >> 4);
  const double2 xa = *reinterpret_cast<const double2*>(x + ca);
  const double2 xb = *reinterpret_cast<const double2*>(x + cb);
  double a[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + i;
    double2 ea = make_double2(0.0, 0.0), eb = make_double2(0.0, 0.0);
    if (!PACKED) {
      ea = *reinterpret_cast<const double2*>(M + r * 64 + ca);
      eb = *reinterpret_cast<const double2*>(M + r * 64 + cb);
    } else {
      if (ca <= r) ea = *reinterpret_cast<const double2*>(M + packed_row_offset(r) + ca);
      if (cb <= r) eb = *reinterpret_cast<const double2*>(M + packed_row_offset(r) + cb);
    }
    a[i] = fma(eb.y, xb.y, fma(eb.x, xb.x, fma(ea.y, xa.y, ea.x * xa.x)));
  }
  {
    const bool hi = lane & 8;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double snd = hi ? a[k] : a[k + 2], kp = hi ? a[k + 2] : a[k];
      a[k] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
    }
  }
  const bool hi = lane & 4;
  const double snd = hi ? a[0] : a[1], kp = hi ? a[1] : a[0];
  double v = kp + __shfl_xor_sync(0xffffffffu, snd, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;
}

// Transposed form at NT == 64, DC == 4 on all 8 consumer warps (the 4-warp mtv leaves half the
// consumers idle on the backward sweep, the longer half of the step at d = 4): warp w owns the 8
// columns 8w..8w+7, lane = column pair p (lane % 4) + 4 part, part sweeping rows part, part + 8, ...
// The 8 partials of a lane (2 columns x 4 rhs columns) are reduced over the 8 parts by a
// transposing butterfly (4 + 2 + 1 shuffles): lane (p, part) ends with the total of column
// 8w + 2p + (part >> 2), rhs column part & 3.  x is column-major (x[c][kXLD]).
template <bool PACKED>
__device__ __forceinline__ double mtv64x4(const double* __restrict__ M, const double* __restrict__ x, int& col,
                                          int& rc) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int part = lane >> 2, c2 = 8 * w + 2 * (lane & 3);
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = part + 8 * i;
    double2 e = make_double2(0.0, 0.0);
    if (!PACKED) e = *reinterpret_cast<const double2*>(M + m * 64 + c2);
    else if (c2 <= m) e = *reinterpret_cast<const double2*>(M + packed_row_offset(m) + c2);
    const double x0 = x[m], x1 = x[kXLD + m], x2 = x[2 * kXLD + m], x3 = x[3 * kXLD + m];  // x[c][kXLD]
    a[0] = fma(e.x, x0, a[0]);
    a[1] = fma(e.x, x1, a[1]);
    a[2] = fma(e.x, x2, a[2]);
    a[3] = fma(e.x, x3, a[3]);
    a[4] = fma(e.y, x0, a[4]);
    a[5] = fma(e.y, x1, a[5]);
    a[6] = fma(e.y, x2, a[6]);
    a[7] = fma(e.y, x3, a[7]);
  }
  const bool b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double snd = b4 ? a[i] : a[i + 4], kp = b4 ? a[i + 4] : a[i];
    a[i] = kp + __shfl_xor_sync(0xffffffffu, snd, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double snd = b3 ? a[i] : a[i + 2], kp = b3 ? a[i + 2] : a[i];
    a[i] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
  }
  const double snd = b2 ? a[0] : a[1], kp = b2 ? a[1] : a[0];
  const double v = kp + __shfl_xor_sync(0xffffffffu, snd, 4);
  // value index 4 b4 + 2 b3 + b2 = part: column half b4, rhs column 2 b3 + b2
  col = c2 + (part >> 2);
  rc = part & 3;
  return v;
}

// Transposed form at NT == 64, DC == 1 on all 8 consumer warps (mtv64x4's mapping): warp w owns
// columns 8w..8w+7, lane = column pair (lane % 4) + 4 part, part sweeping rows part + 8i; the two
// column partials are split over lane bit 4 and reduced over the parts (3 shuffles).  The total of
// column 8w + 2 (lane % 4) + lane / 16 ends on the 4 lanes with equal lane % 4 and lane / 16.
template <bool PACKED>
__device__ __forceinline__ double mtv64x1(const double* __restrict__ M, const double* __restrict__ x, int& col) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int part = lane >> 2, c2 = 8 * w + 2 * (lane & 3);
  double a[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = part + 8 * i;
    double2 e = make_double2(0.0, 0.0);
    if (!PACKED) e = *reinterpret_cast<const double2*>(M + m * 64 + c2);
    else if (c2 <= m) e = *reinterpret_cast<const double2*>(M + packed_row_offset(m) + c2);
    const double xv = x[m];
    a[i & 1][0] = fma(e.x, xv, a[i & 1][0]);
    a[i & 1][1] = fma(e.y, xv, a[i & 1][1]);
  }
  const double a0 = a[0][0] + a[1][0], a1 = a[0][1] + a[1][1];
  const bool hi = lane & 16;
  double v = (hi ? a1 : a0) + __shfl_xor_sync(0xffffffffu, hi ? a0 : a1, 16);
  v += __shfl_xor_sync(0xffffffffu, v, 8);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  col = c2 + (lane >> 4);
  return v;
}

// Row form at NT == 64 without the rotated reads: warp w owns rows 8w..8w+7 and lane l the column
// pair (2l, 2l+1), so each row read is one contiguous conflict-free 512-byte run and x[2l..2l+1]
// is loaded once into registers; the 8 row partials are reduced across the warp by a
// transposing butterfly (4 + 2 + 1 + 2 shuffles).  The total of row 8w + lane/4 (= tid/4, the
// mv_rows mapping) is returned on the 4 lanes of that row's quad.
// XT: x is stored column-major (x[c][64], see solve_tma_kernel's vidx), so lane l's pair of
// entries of each rhs column is one conflict-free 16-byte read (row-major at d = 4 put the 32 lanes'
// reads 64 bytes apart: 16 shared-memory wavefronts per load instead of 4).
template <int DC, bool PACKED, bool XT = false>
__device__ __forceinline__ void mv64(const double* __restrict__ M, const double* __restrict__ x, double (&s)[DC]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c2 = 2 * lane;
  double x0[DC], x1[DC], v[8][DC];
  if constexpr (XT) {
#pragma unroll
    for (int c = 0; c < DC; ++c) {
      const double2 xv = *reinterpret_cast<const double2*>(x + c * kXLD + c2);
      x0[c] = xv.x;
      x1[c] = xv.y;
    }
  } else if (DC == 1) {
    const double2 xv = *reinterpret_cast<const double2*>(x + c2);
    x0[0] = xv.x;
    x1[0] = xv.y;
  } else {
#pragma unroll
    for (int c = 0; c < DC; ++c) {
      x0[c] = x[c2 * DC + c];
      x1[c] = x[(c2 + 1) * DC + c];
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = 8 * w + i;
    double2 e = make_double2(0.0, 0.0);
    if (!PACKED) e = *reinterpret_cast<const double2*>(M + r * 64 + c2);
    else if (c2 <= r) e = *reinterpret_cast<const double2*>(M + packed_row_offset(r) + c2);
#pragma unroll
    for (int c = 0; c < DC; ++c) v[i][c] = fma(e.x, x0[c], e.y * x1[c]);
  }
  const bool b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1;
#pragma unroll
  for (int c = 0; c < DC; ++c) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double snd = b4 ? v[i][c] : v[i + 4][c], kp = b4 ? v[i + 4][c] : v[i][c];
      v[i][c] = kp + __shfl_xor_sync(0xffffffffu, snd, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const double snd = b3 ? v[i][c] : v[i + 2][c], kp = b3 ? v[i + 2][c] : v[i][c];
      v[i][c] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
    }
    {
      const double snd = b2 ? v[0][c] : v[1][c], kp = b2 ? v[1][c] : v[0][c];
      v[0][c] = kp + __shfl_xor_sync(0xffffffffu, snd, 4);
    }
    double t = v[0][c];
    t += __shfl_xor_sync(0xffffffffu, t, 2);
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    s[c] = t;
  }
}

template <int NT, int DC>
__device__ __forceinline__ void mv_full_rows(const double* M, const double* x, double (&s)[DC]) {
  if constexpr (NT == 64 && DC == 1) { s[0] = mv64x1<false>(M, x); return; }
  if constexpr (NT == 64) { mv64<DC, false, DC == 4>(M, x, s); return; }
  mv_rows<NT, DC>(M, x, s);
}
template <int NT, int DC>
__device__ __forceinline__ void mv_packed_rows(const double* M, const double* x, double (&s)[DC]) {
  if constexpr (NT == 64 && DC == 1) { s[0] = mv64x1<true>(M, x); return; }
  if constexpr (NT == 64) { mv64<DC, true, DC == 4>(M, x, s); return; }
  mv_pack_rows<NT, DC>(M, x, s);
}

// Segment bounds of the persistent loops, with the next segment's separators loaded one segment
// ahead (their global-load latency would otherwise stall every segment start).
struct SegBounds {
  long long start, stop;
  int nlo, nhi;
  __device__ SegBounds(const SolveArgs& a, int mode, int k, int K) {
    start = stop = 0;
    nlo = nhi = 0;
    if (mode == kSolveBase) {
      start = 0;
      stop = a.N;
    } else if (k < K) {
      start = (long long)a.seps[k] + 1;
      stop = a.seps[k + 1];
    }
  }
  __device__ __forceinline__ void advance(const SolveArgs& a, int mode, int kn, int K) {
    if (mode != kSolveBase && kn < K) {
      nlo = __ldg(a.seps + kn);
      nhi = __ldg(a.seps + kn + 1);
    }
  }
  __device__ __forceinline__ void next() {
    start = (long long)nlo + 1;
    stop = nhi;
  }
};

// WIDE (levels with at least as many segments as SMs, n = 64, d <= 4): two CTAs per SM (two
// segments in flight per SM) with 2-slot rings; otherwise one CTA per SM with a deeper ring.  With
// d > 1 two CTAs' rings leave no room for the forward sweep's z cache (ZMAX = 0): z_j goes through
// the solution buffer (L2) instead.
template <int NT, int DC, bool WIDE = false>
struct TmaShape {
  using S = Solve2Shape<NT>;
  static constexpr int NCW = S::NTHREADS / 32;  // consumer warps
  static constexpr int NTHREADS = S::NTHREADS + 32;
  static constexpr bool TWO = WIDE && NT == 64 && DC <= 4;
  static constexpr int STAGES = NT == 64 ? (TWO ? 2 : (DC > 1 ? 3 : 4)) : 8;
  static constexpr int STAGE = S::FULL + S::PACK + NT * DC;  // doubles per slot
  static constexpr int ZMAX = (TWO && DC > 1) ? 0 : S::ZMAX;
  static constexpr int VS = (NT == 64 && DC == 4) ? DC * kXLD : NT * DC;  // doubles per shared vector
  static constexpr int MINB = TWO ? 2 : 1;  // resident CTAs per SM (register cap 112 when 2)
  static constexpr size_t SMEM = sizeof(double) * ((size_t)STAGES * STAGE + (size_t)(4 + ZMAX) * VS) +
                                 2 * STAGES * sizeof(unsigned long long);
};

template <int NT, int DC, bool WIDE>
__global__ void __launch_bounds__(TmaShape<NT, DC, WIDE>::NTHREADS, TmaShape<NT, DC, WIDE>::MINB)
    solve_tma_kernel(SolveArgs a) {
  using S = Solve2Shape<NT>;
  using T = TmaShape<NT, DC, WIDE>;
  constexpr int STAGES = T::STAGES, STAGE = T::STAGE, NTH = S::NTHREADS;
  extern __shared__ __align__(16) double smem[];
  double* ring = smem;
  double* t = ring + STAGES * STAGE;
  constexpr int VS = T::VS;
  double* u = t + VS;
  double* corr = u + VS;
  double* zc = corr + 2 * VS;
  unsigned long long* full_bar = reinterpret_cast<unsigned long long*>(zc + T::ZMAX * VS);
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
      const unsigned long long pol_keep = l2_policy_evict_last(), pol_drop = l2_policy_evict_first();
      constexpr unsigned fb = NT * NT * sizeof(double), pb = S::PACK * sizeof(double);
      const unsigned vb = (unsigned)(n * d * sizeof(double));
      SegBounds sb(a, mode, blockIdx.x, K);
      for (int k = blockIdx.x; k < K; k += gridDim.x) {
        const long long start = sb.start, stop = sb.stop;
        sb.advance(a, mode, k + gridDim.x, K);  // the next segment's separators load behind this one
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
          // forward-sweep blocks are read again by the backward sweep: keep them in L2 (evict_last);
          // the backward sweep is their last use (evict_first)
          const unsigned long long pol = (kind == kStepF) ? pol_keep : pol_drop;
          if (full) tma_load_1d_hint(st, full, fb, &full_bar[slot], pol);
          if (pack) tma_load_1d_hint(st + S::FULL, pack, pb, &full_bar[slot], pol);
          if (vec) tma_load_1d(st + S::FULL + S::PACK, vec, vb, &full_bar[slot]);
          if (++slot == STAGES) {
            slot = 0;
            phase ^= 1;
          }
        }
        sb.next();
      }
    }
    return;
  }

  // ===================== consumer warps =====================
  // Two dependent mat-vecs per step and one barrier after each (the slot is released per warp):
  // row-form products (forward sweep, C_R fold) on all consumer warps, 4 threads per row;
  // transposed products (backward sweep, C_L fold) on the first TW warps with every part of a
  // column inside one warp (xor-shuffle reduction, no shared-memory partials).
  constexpr int TW = NT < 16 ? 1 : NT / 16;
  constexpr bool X4 = NT == 64 && DC == 4;  // transposed products on all consumer warps
  constexpr bool X1 = NT == 64 && DC == 1;  // backward-sweep transposed products on all warps
  const bool x1lead = ((lane >> 2) & 3) == 0;
  // shared-memory vectors (t, u, z cache, corrections): row-major [r][c], column-major at X4
  auto vi = [](int r, int c) { return X4 ? c * kXLD + r : r * DC + c; };
  constexpr int CW = NT < 16 ? NT : 16, PR = CW / 2;
  const int rr = tid >> 2;
  const bool rlead = (tid & 3) == 0;
  const int tc = CW * warp + 2 * (lane % PR);
  const bool tlead = warp < TW && lane < PR;
  int slot = 0;
  unsigned phase = 0;
#ifdef BTD_PHASE_PROF
  long long _sp_last = clock64();
#endif
  SegBounds sb(a, mode, blockIdx.x, K);
  for (int k = blockIdx.x; k < K; k += gridDim.x) {
    const long long start = sb.start, stop = sb.stop;
    sb.advance(a, mode, k + gridDim.x, K);  // the next segment's separators load behind this one
    const int J = (int)(stop - start);
    const int ns = nsteps(mode, J);
    for (int idx = 0; idx < ns; ++idx) {
      int kind, j;
      step_kind(mode, J, idx, kind, j);
      const long long row = start + j;
      BTD_SPH(0);
      // X4 backward steps without the z cache: this lane's z_j entry (the one it combines in the
      // transposed product, lane-fixed) is read from the solution buffer before the slot wait, so
      // its L2 latency is not on the step's critical path
      double zpre = 0.0;
      if constexpr (X4) {
        if (kind == kStepB && j >= T::ZMAX) {
          const int oc = 8 * warp + 2 * (lane & 3) + (lane >> 4), orc = (lane >> 2) & 3;
          if (orc < dc) zpre = a.x[row * ps + (size_t)oc * d + c0 + orc];
        }
      }
      mbar_wait(&full_bar[slot], phase);
      BTD_SPH(1);
      const double* sf = ring + slot * STAGE;
      const double* sp = sf + S::FULL;
      const double* sv = sp + S::PACK;
      // b_j[r][c] with the up-pass boundary corrections
      auto bval = [&](int r, int c) -> double {
        double v = 0.0;
        if (c < dc) v = vec_bulk ? sv[r * d + c] : a.rhs[row * ps + (size_t)r * d + c0 + c];
        if (mode == kSolveUp) {
          if (j == 0) v -= corr[vi(r, c)];
          if (j == J - 1) v -= corr[VS + vi(r, c)];
        }
        return v;
      };
      if (kind == kStepNone) {
      } else if (kind == kStepF) {
        // t = b_j - L_{j,j-1} z_{j-1}
        if (j > 0) {
          double sm[DC];
          if constexpr (X4) {
            const double sv4 = mv64x4<false>(sf, u);
            t[vi(rr, lane & 3)] = bval(rr, lane & 3) - sv4;
          } else {
            mv_full_rows<NT, DC>(sf, u, sm);
            if (rlead) {
#pragma unroll
              for (int c = 0; c < DC; ++c) t[vi(rr, c)] = bval(rr, c) - sm[c];
            }
          }
        } else {
          for (int e = tid; e < NT * DC; e += NTH) t[vi(e / DC, e % DC)] = bval(e / DC, e % DC);
        }
        BTD_SPH(2);
        csync<NT>();
        BTD_SPH(3);
        // z_j = Linv_j t
        double sm[DC];
        if constexpr (X4) {
          const double sv4 = mv64x4<true>(sp, t);
          const int c = lane & 3;
          u[vi(rr, c)] = sv4;
          if (j < T::ZMAX) zc[j * VS + vi(rr, c)] = sv4;
          else if (c < dc) a.x[row * ps + (size_t)rr * d + c0 + c] = sv4;
        } else {
        mv_packed_rows<NT, DC>(sp, t, sm);
        if (rlead) {
          double* zdst = j < T::ZMAX ? zc + j * VS : nullptr;
#pragma unroll
          for (int c = 0; c < DC; ++c) {
            u[vi(rr, c)] = sm[c];
            if (zdst) zdst[vi(rr, c)] = sm[c];
            else if (c < dc) a.x[row * ps + (size_t)rr * d + c0 + c] = sm[c];
          }
        }
        }
        BTD_SPH(4);
        csync<NT>();
        BTD_SPH(5);
      } else if (kind == kStepB) {
        const double* zsrc = j < T::ZMAX ? zc + j * VS : nullptr;
        auto zval = [&](int r, int c) -> double {
          return zsrc ? zsrc[vi(r, c)] : (c < dc ? a.x[row * ps + (size_t)r * d + c0 + c] : 0.0);
        };
        const double* src = zsrc;
        if (j < J - 1) {  // t = z_j - L_{j+1,j}^T w_{j+1}
          if constexpr (X4) {
            int oc, orc;
            const double ov = mtv64x4<false>(sf, u, oc, orc);
            t[vi(oc, orc)] = (zsrc ? zsrc[vi(oc, orc)] : zpre) - ov;
          } else if constexpr (X1) {
            int oc;
            const double ov = mtv64x1<false>(sf, u, oc);
            if (x1lead) t[oc] = zval(oc, 0) - ov;
          } else if (warp < TW) {
            double v[2][DC];
            mtv<NT, DC, false>(sf, u, v);
            if (tlead) {
#pragma unroll
              for (int c = 0; c < DC; ++c) {
                t[vi(tc, c)] = zval(tc, c) - v[0][c];
                t[vi(tc + 1, c)] = zval(tc + 1, c) - v[1][c];
              }
            }
          }
          BTD_SPH(6);
          csync<NT>();
          BTD_SPH(7);
          src = t;
        } else if (!zsrc) {
          if constexpr (X4) t[vi(8 * warp + 2 * (lane & 3) + (lane >> 4), (lane >> 2) & 3)] = zpre;
          else
            for (int e = tid; e < NT * DC; e += NTH) t[vi(e / DC, e % DC)] = zval(e / DC, e % DC);
          csync<NT>();
          src = t;
        }
        // w_j = Linv_j^T t
        if constexpr (X4) {
          int oc, orc;
          const double ov = mtv64x4<true>(sp, src, oc, orc);
          u[vi(oc, orc)] = ov;
          if (mode != kSolveDown && orc < dc) a.x[row * ps + (size_t)oc * d + c0 + orc] = ov;
        } else if constexpr (X1) {
          int oc;
          const double ov = mtv64x1<true>(sp, src, oc);
          if (x1lead) {
            u[oc] = ov;
            if (mode != kSolveDown) a.x[row * ps + (size_t)oc * d + c0] = ov;
          }
        } else if (warp < TW) {
          double v[2][DC];
          mtv<NT, DC, true>(sp, src, v);
          if (tlead) {
#pragma unroll
            for (int c = 0; c < DC; ++c)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                u[vi(tc + h, c)] = v[h][c];
                if (mode != kSolveDown && c < dc) a.x[row * ps + (size_t)(tc + h) * d + c0 + c] = v[h][c];
              }
          }
        }
        BTD_SPH(8);
        csync<NT>();
        BTD_SPH(9);
      } else if (mode == kSolveDown) {  // fold: f_R = C_R w_last ; f_L = C_L^T w_0 (no barrier needed)
        double* dst = (kind == kStepCR ? a.fr : a.fl) + (size_t)k * ps;
        if (kind == kStepCR) {
          double sm[DC];
          if constexpr (X4) {
            const double sv4 = mv64x4<false>(sf, u);
            if ((lane & 3) < dc) dst[(size_t)rr * d + c0 + (lane & 3)] = sv4;
          } else {
            mv_full_rows<NT, DC>(sf, u, sm);
            if (rlead) {
#pragma unroll
              for (int c = 0; c < DC; ++c)
                if (c < dc) dst[(size_t)rr * d + c0 + c] = sm[c];
            }
          }
        } else if constexpr (X4) {
          int oc, orc;
          const double ov = mtv64x4<false>(sf, u, oc, orc);
          if (orc < dc) dst[(size_t)oc * d + c0 + orc] = ov;
        } else if (warp < TW) {
          double v[2][DC];
          mtv<NT, DC, false>(sf, u, v);
          if (tlead) {
#pragma unroll
            for (int c = 0; c < DC; ++c)
#pragma unroll
              for (int h = 0; h < 2; ++h)
                if (c < dc) dst[(size_t)(tc + h) * d + c0 + c] = v[h][c];
          }
        }
      } else {  // up: boundary corrections C_L x_L -> corr[0], C_R^T x_R -> corr[1]
        const double* xs = a.xsep + (size_t)(kind == kStepCL ? k : k + 1) * ps;
        for (int e = tid; e < NT * DC; e += NTH) {
          const int r = e / DC, c = e % DC;
          const double v = c < dc ? (vec_bulk ? sv[r * d + c] : xs[(size_t)r * d + c0 + c]) : 0.0;
          t[vi(r, c)] = v;
          if (c < dc) {
            const size_t off = (size_t)r * d + c0 + c;
            if (kind == kStepCL) a.x[(size_t)(start - 1) * ps + off] = v;
            if (kind == kStepCR && k == K - 1) a.x[(size_t)stop * ps + off] = v;
          }
        }
        csync<NT>();
        if (kind == kStepCL) {
          double sm[DC];
          if constexpr (X4) {
            corr[vi(rr, lane & 3)] = mv64x4<false>(sf, t);
          } else {
            mv_full_rows<NT, DC>(sf, t, sm);
            if (rlead) {
#pragma unroll
              for (int c = 0; c < DC; ++c) corr[vi(rr, c)] = sm[c];
            }
          }
        } else if constexpr (X4) {
          int oc, orc;
          const double ov = mtv64x4<false>(sf, t, oc, orc);
          corr[VS + vi(oc, orc)] = ov;
        } else if (warp < TW) {
          double v[2][DC];
          mtv<NT, DC, false>(sf, t, v);
          if (tlead) {
#pragma unroll
            for (int c = 0; c < DC; ++c) {
              corr[VS + vi(tc, c)] = v[0][c];
              corr[VS + vi(tc + 1, c)] = v[1][c];
            }
          }
        }
        csync<NT>();
      }
      BTD_SPH(10);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[slot]);  // this warp is done with the slot
      BTD_SPH(11);
      if (++slot == STAGES) {
        slot = 0;
        phase ^= 1;
      }
    }
    sb.next();
  }
}

}  // namespace btd
