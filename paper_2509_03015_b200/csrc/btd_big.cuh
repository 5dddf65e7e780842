// Block sizes n > 64 (multiples of 64, e.g. BASELINE config 4 with n = 256): the same Y-form
// recursion as btd_factor.cuh, sequenced on the host as a handful of batched launches per
// elimination step.  Every launch is batched over the segments of a level (blockIdx.y = segment);
// operand addresses are derived on the device from the level plan (separators, step j), so no
// pointer arrays are built on the host.
//
//   big_potrf_kernel : one CTA per segment, blocked (64-tile) Cholesky + inverse of the n x n
//                      diagonal block D_j (potrf_trtri<64> on diagonal tiles, DMMA tile GEMMs
//                      for the panel solve, trailing update and the inverse)
//   bt_gemm_kernel   : C = alpha op(A) op(B) + beta C_in on 64 x 64 output tiles (DMMA m8n8k4),
//                      used for Pt = Xt Linv^T, the Schur/fill/diag updates and the solve panels
//   bt_copy_kernel   : block copies / transposed copies (staging, coupling copies)
#pragma once

#include "btd_factor.cuh"

namespace btd {

constexpr int BT = 64;        // tile edge
constexpr int BLD = BT + 4;   // shared tile leading dimension
constexpr int BTHREADS = 256;

// How a batch entry (segment k at step j) addresses an operand.
enum OperandIndex : int {
  kIdxSegRow = 0,   // block row seps[k] + 1 + j + delta of a level array (base: j + delta)
  kIdxSeg = 1,      // per-segment workspace slot k (+ delta)
  kIdxSegStop = 2,  // block row seps[k+1] + delta (the right separator side)
  kIdxSegStart = 3  // block row seps[k] + delta (the left separator side)
};

struct Operand {
  const double* base;
  long long stride;  // doubles between consecutive indexed blocks
  int ld;            // leading dimension (doubles) of the stored matrix
  int index, delta;
  int row0, col0;    // offset of the op()-matrix inside the stored block (before transposition)
  int trans;         // op(X) = X^T
};

__device__ __forceinline__ const double* operand_ptr(const Operand& o, const int* seps, int base_mode, int k, int j) {
  long long idx;
  switch (o.index) {
    case kIdxSegRow: idx = (base_mode ? 0ll : (long long)seps[k] + 1) + j + o.delta; break;
    case kIdxSeg: idx = (long long)k + o.delta; break;
    case kIdxSegStop: idx = (long long)seps[k + 1] + o.delta; break;
    default: idx = (long long)seps[k] + o.delta; break;
  }
  return o.base + idx * o.stride;
}

// activity of a segment at step j
enum Activity : int { kActAll = 0, kActNotLast = 1, kActLast = 2, kActBeforeSecondLast = 3, kActSecondLast = 4 };

__device__ __forceinline__ bool segment_active(const int* seps, int base_mode, long long N, int k, int j, int act,
                                               int& J) {
  J = base_mode ? (int)N : seps[k + 1] - seps[k] - 1;
  if (j >= J) return false;
  if (act == kActNotLast) return j < J - 1;
  if (act == kActLast) return j == J - 1;
  if (act == kActBeforeSecondLast) return j < J - 2;
  if (act == kActSecondLast) return j == J - 2;
  return true;
}

struct GemmArgs {
  Operand A, B, Cin, Cout;
  const int* seps;
  long long N;
  int base_mode, j, act;
  int level;             // factor level of the launch (INT_MAX: a solve launch, any error stops it)
  int m, n, k;           // op(A) m x k, op(B) k x n
  double alpha, beta;    // Cout = alpha op(A) op(B) + beta Cin   (beta == 0: Cin unused)
  int lower_only;        // skip tiles strictly above the diagonal (symmetric outputs)
  int tri;               // 1: op(B)[k][c] == 0 for k > c (B = L^T, L lower); 2: op(A)[r][k] == 0 for k > r;
                         // 3: op(A)[r][k] == 0 for k < r (A = L^T)
  int store_trans;       // write Cout^T
  int tiles_n;
  int k0;                // first segment of this launch (blockIdx.y = k - k0)
  int ksplit;            // > 1: split-k over ksplit CTAs per tile, raw partials into `part`
  double* part;          //      (tile, split, 64 x 64), summed in split order by bt_gemm_reduce_kernel
  const DevErr* err;
};

// ---------------------------------------------------------------------------------------------
// Pipelined 64 x 64 output-tile GEMM: k in chunks of BK = 32, two stages in flight (cp.async.cg
// 16-byte copies; the chunk k+1 loads while chunk k is multiplied).  Operand tiles stay in their
// storage orientation in shared memory (every global read is a contiguous 16-byte run, with no
// transposition on the fly); the DMMA fragment loads index them according to TA / TB.
//   A tile: !TA -> As[r][k] (64 x BK, ld BK+4)      TA -> As[k][r] (BK x 64, ld 64+4)
//   B tile (op(B) is k x n): !TB -> Bs[k][c] (BK x 64, ld 64+4)   TB -> Bs[c][k] (64 x BK, ld BK+4)
// ---------------------------------------------------------------------------------------------
constexpr int BK = 32;
constexpr int LDK = BK + 4;  // tiles whose rows run along k
constexpr int LDM = BT + 4;  // tiles whose rows run along m / n
constexpr int GSTAGE = (BT * LDK > BK * LDM) ? BT * LDK : BK * LDM;  // doubles per operand tile slot

// Stage the region rows [r0, r0+R) x cols [c0, c0+C) of a stored row-major matrix X (ld, logical
// bounds rows x cols) into S (ld LS), zero filling outside the bounds.
template <int R, int C, int LS>
__device__ __forceinline__ void stage_region(double* S, const double* X, int ld, int r0, int c0, int rows, int cols) {
  constexpr int CH = C / 2;  // 16-byte chunks per row
  for (int e = threadIdx.x; e < R * CH; e += BTHREADS) {
    const int r = e / CH, c = (e % CH) * 2;
    const int gr = r0 + r, gc = c0 + c;
    double* dst = S + r * LS + c;
    const double* src = X + (size_t)gr * ld + gc;
    if (gr < rows && gc + 1 < cols && (((size_t)src & 15) == 0)) {
      cp_async16(dst, src, 16);
    } else {
      cp_async8(dst, (gr < rows && gc < cols) ? (const void*)src : (const void*)X, (gr < rows && gc < cols) ? 8 : 0);
      cp_async8(dst + 1, (gr < rows && gc + 1 < cols) ? (const void*)(src + 1) : (const void*)X,
                (gr < rows && gc + 1 < cols) ? 8 : 0);
    }
  }
}

template <bool TA, bool TB>
__device__ __forceinline__ void stage_chunk(double* As, double* Bs, const double* A, int lda, const double* B, int ldb,
                                            int m, int n, int kdim, int m0, int n0, int kc) {
  // op(A) is m x kdim: stored A is m x kdim (!TA) or kdim x m (TA)
  if (!TA) stage_region<BT, BK, LDK>(As, A, lda, m0, kc, m, kdim);
  else stage_region<BK, BT, LDM>(As, A, lda, kc, m0, kdim, m);
  // op(B) is kdim x n: stored B is kdim x n (!TB) or n x kdim (TB)
  if (!TB) stage_region<BK, BT, LDM>(Bs, B, ldb, kc, n0, kdim, n);
  else stage_region<BT, BK, LDK>(Bs, B, ldb, n0, kc, n, kdim);
}

template <bool TA, bool TB>
__device__ __forceinline__ void chunk_mma(double (&acc)[2][4][2], const double* As, const double* Bs, int kn) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rw = (warp >> 1) * 16, cw = (warp & 1) * 32;
  const int lr = lane >> 2, lk = lane & 3;
#pragma unroll 2
  for (int kk = 0; kk < kn; kk += 4) {
    double a[2], b[4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
      a[i] = TA ? As[(kk + lk) * LDM + rw + i * 8 + lr] : As[(rw + i * 8 + lr) * LDK + kk + lk];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      b[q] = TB ? Bs[(cw + q * 8 + lr) * LDK + kk + lk] : Bs[(kk + lk) * LDM + cw + q * 8 + lr];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q) dmma(acc[i][q], a[i], b[q]);
  }
}

template <bool TA, bool TB>
__device__ __forceinline__ void gemm_tile_pipelined(double (&acc)[2][4][2], const double* A, int lda, const double* B,
                                                    int ldb, int m, int n, int kdim, int m0, int n0, int kbeg, int kend,
                                                    double* sm) {
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q][0] = acc[i][q][1] = 0.0;
  const int nch = (kend - kbeg + BK - 1) / BK;
  if (nch <= 0) return;
  stage_chunk<TA, TB>(sm, sm + GSTAGE, A, lda, B, ldb, m, n, kdim, m0, n0, kbeg);
  cp_async_commit();
  for (int c = 0; c < nch; ++c) {
    double* cur = sm + (c & 1) * 2 * GSTAGE;
    if (c + 1 < nch) {
      double* nxt = sm + ((c + 1) & 1) * 2 * GSTAGE;
      stage_chunk<TA, TB>(nxt, nxt + GSTAGE, A, lda, B, ldb, m, n, kdim, m0, n0, kbeg + (c + 1) * BK);
      cp_async_commit();
      cp_async_wait_group<1>();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    chunk_mma<TA, TB>(acc, cur, cur + GSTAGE, min(BK, kend - kbeg - c * BK));
    __syncthreads();
  }
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(BTHREADS) bt_gemm_kernel(GemmArgs g) {
  const int k = g.k0 + blockIdx.y;
  // skip only when a recorded failure can no longer be superseded by this (step, member): a lower
  // member failing at a later 64-column tile of the same step must still be found
  if (cta_superseded(g.err, g.level, g.j, k)) return;
  int J;
  if (!segment_active(g.seps, g.base_mode, g.N, k, g.j, g.act, J)) return;
  const int ks = g.ksplit > 1 ? g.ksplit : 1;
  const int tile = blockIdx.x / ks, sp = blockIdx.x % ks;
  const int tm = tile / g.tiles_n, tn = tile % g.tiles_n;
  const int m0 = tm * BT, n0 = tn * BT;
  if (g.lower_only && n0 > m0) return;
  extern __shared__ __align__(16) double gsm[];
  const double* A = operand_ptr(g.A, g.seps, g.base_mode, k, g.j) + (size_t)g.A.row0 * g.A.ld + g.A.col0;
  const double* B = operand_ptr(g.B, g.seps, g.base_mode, k, g.j) + (size_t)g.B.row0 * g.B.ld + g.B.col0;
  int kbeg = 0, kend = g.k;
  if (g.tri == 1) kend = min(kend, n0 + BT);
  if (g.tri == 2) kend = min(kend, m0 + BT);
  if (g.tri == 3) kbeg = m0 / BT * BT;
  if (g.tri == 4) kbeg = max(kbeg, n0 / BT * BT);  // op(B)[k][c] == 0 for k < c (B lower triangular)
  if (ks > 1) {  // this CTA's share of the k range, in whole BK chunks
    const int chunk = ((kend - kbeg + ks - 1) / ks + BK - 1) / BK * BK;
    const int b = kbeg + sp * chunk;
    kend = min(kend, b + chunk);
    kbeg = b;
  }
  double acc[2][4][2];
  gemm_tile_pipelined<TA, TB>(acc, A, g.A.ld, B, g.B.ld, g.m, g.n, g.k, m0, n0, kbeg, kend, gsm);
  if (ks > 1) {  // raw partial of (tile, sp)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rw = (warp >> 1) * 16, cw = (warp & 1) * 32;
    double* pt = g.part + ((size_t)tile * ks + sp) * BT * BT;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<double2*>(pt + (rw + i * 8 + (lane >> 2)) * BT + cw + q * 8 + 2 * (lane & 3)) =
            make_double2(acc[i][q][0], acc[i][q][1]);
    return;
  }
  const double* Cin = g.beta != 0.0 ? operand_ptr(g.Cin, g.seps, g.base_mode, k, g.j) : nullptr;
  if (Cin) Cin += (size_t)g.Cin.row0 * g.Cin.ld + g.Cin.col0;
  double* Cout = const_cast<double*>(operand_ptr(g.Cout, g.seps, g.base_mode, k, g.j)) +
                 (size_t)g.Cout.row0 * g.Cout.ld + g.Cout.col0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rw = (warp >> 1) * 16, cw = (warp & 1) * 32;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = m0 + rw + i * 8 + (lane >> 2);
        const int c = n0 + cw + q * 8 + 2 * (lane & 3) + h;
        if (r >= g.m || c >= g.n) continue;
        double v = g.alpha * acc[i][q][h];
        if (Cin) v += g.beta * Cin[(size_t)r * g.Cin.ld + c];
        if (g.store_trans)
          Cout[(size_t)c * g.Cout.ld + r] = v;
        else
          Cout[(size_t)r * g.Cout.ld + c] = v;
      }
}

// Split-k epilogue: C = alpha * (sum of the partials in split order) + beta * Cin, per 64 x 64 tile
// (deterministic: fixed summation order).  grid.x = tiles, blockIdx.y = segment (as the GEMM).
__global__ void __launch_bounds__(BTHREADS) bt_gemm_reduce_kernel(GemmArgs g) {
  const int k = g.k0 + blockIdx.y;
  if (npd_superseded(g.err, g.level, g.j, k)) return;
  int J;
  if (!segment_active(g.seps, g.base_mode, g.N, k, g.j, g.act, J)) return;
  const int tile = blockIdx.x, tm = tile / g.tiles_n, tn = tile % g.tiles_n;
  const int m0 = tm * BT, n0 = tn * BT;
  if (g.lower_only && n0 > m0) return;
  const double* Cin = g.beta != 0.0 ? operand_ptr(g.Cin, g.seps, g.base_mode, k, g.j) : nullptr;
  if (Cin) Cin += (size_t)g.Cin.row0 * g.Cin.ld + g.Cin.col0;
  double* Cout = const_cast<double*>(operand_ptr(g.Cout, g.seps, g.base_mode, k, g.j)) +
                 (size_t)g.Cout.row0 * g.Cout.ld + g.Cout.col0;
  const double* pt = g.part + (size_t)tile * g.ksplit * BT * BT;
  for (int e = threadIdx.x; e < BT * BT; e += BTHREADS) {
    const int r = m0 + e / BT, c = n0 + e % BT;
    if (r >= g.m || c >= g.n) continue;
    double s = 0.0;
    for (int q = 0; q < g.ksplit; ++q) s += pt[(size_t)q * BT * BT + e];
    double v = g.alpha * s;
    if (Cin) v += g.beta * Cin[(size_t)r * g.Cin.ld + c];
    if (g.store_trans)
      Cout[(size_t)c * g.Cout.ld + r] = v;
    else
      Cout[(size_t)r * g.Cout.ld + c] = v;
  }
}

// ---------------------------------------------------------------------------------------------
// Host-sequenced blocked Cholesky + inverse of the n x n blocks (big_potrf_seq, btd_capi.cu): the
// 64 x 64 diagonal tiles are factored and inverted here (one 128-thread CTA per segment,
// potrf_trtri<64>), the panel / trailing / inverse products run as batched tile GEMMs over every
// segment and tile -- the machine-wide parallelism the one-CTA-per-block kernel lacks.
// ---------------------------------------------------------------------------------------------
struct BigDiagArgs {
  Operand D, Linv;  // segment's working block (in: updated D; tile kb factored) and Linv output
  const int* seps;
  long long N;
  int base_mode, j, kb, n, level, k0;
  DevErr* err;
};

__global__ void __launch_bounds__(128) big_diag_potrf_kernel(BigDiagArgs g) {
  constexpr int LD = FactorShape<64>::LD;
  const int k = g.k0 + blockIdx.x;
  if (cta_superseded(g.err, g.level, g.j, k)) return;
  int J;
  if (!segment_active(g.seps, g.base_mode, g.N, k, g.j, kActAll, J)) return;
  __shared__ __align__(16) double DL[BT * LD];
  __shared__ int s_fail;
  const double* D = operand_ptr(g.D, g.seps, g.base_mode, k, g.j);
  double* Li = const_cast<double*>(operand_ptr(g.Linv, g.seps, g.base_mode, k, g.j));
  const int n = g.n, o = g.kb * BT;
  for (int e = threadIdx.x; e < BT * BT; e += 128) DL[(e / BT) * LD + e % BT] = D[(size_t)(o + e / BT) * n + o + e % BT];
  __syncthreads();
  const int fail = potrf_trtri<64>(DL, &s_fail);  // warps 0..3 = group A
  if (fail) {
    if (threadIdx.x == 0) report_npd(g.err, g.level, g.j, k, o + fail);
    return;
  }
  for (int e = threadIdx.x; e < BT * BT; e += 128) {
    const int r = e / BT, c = e % BT;
    Li[(size_t)(o + r) * n + o + c] = c <= r ? DL[r * LD + c] : 0.0;
  }
}

// zero the strict upper 64 x 64 tiles of every active segment's n x n Linv (grid.x = tile pairs)
__global__ void big_zero_upper_kernel(BigDiagArgs g) {
  const int k = g.k0 + blockIdx.y;
  if (npd_superseded(g.err, g.level, g.j, k)) return;
  int J;
  if (!segment_active(g.seps, g.base_mode, g.N, k, g.j, kActAll, J)) return;
  double* Li = const_cast<double*>(operand_ptr(g.Linv, g.seps, g.base_mode, k, g.j));
  int t = blockIdx.x, ib = 0;
  const int NB = g.n / BT;
  while (t >= NB - 1 - ib) {  // pair t -> (ib, jb > ib)
    t -= NB - 1 - ib;
    ++ib;
  }
  const int jb = ib + 1 + t;
  for (int e = threadIdx.x; e < BT * BT; e += blockDim.x)
    Li[(size_t)(ib * BT + e / BT) * g.n + jb * BT + e % BT] = 0.0;
}

struct CopyArgs {
  Operand src, dst;
  const int* seps;
  long long N;
  int base_mode, j, act;
  int level;       // as GemmArgs::level
  int rows, cols;  // of the destination
  int k0;          // first segment of this launch
  const DevErr* err;
};

// dst[r][c] = src[r][c] (or src[c][r] when src.trans); blockIdx.y = segment
__global__ void bt_copy_kernel(CopyArgs c) {
  const int k = c.k0 + blockIdx.y;
  if (npd_superseded(c.err, c.level, c.j, k)) return;
  int J;
  if (!segment_active(c.seps, c.base_mode, c.N, k, c.j, c.act, J)) return;
  const double* s = operand_ptr(c.src, c.seps, c.base_mode, k, c.j);
  double* d = const_cast<double*>(operand_ptr(c.dst, c.seps, c.base_mode, k, c.j));
  const long long tot = (long long)c.rows * c.cols;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / c.cols), col = (int)(e % c.cols);
    const double v = c.src.trans ? s[(size_t)(c.src.row0 + col) * c.src.ld + c.src.col0 + r]
                                 : s[(size_t)(c.src.row0 + r) * c.src.ld + c.src.col0 + col];
    d[(size_t)(c.dst.row0 + r) * c.dst.ld + c.dst.col0 + col] = v;
  }
}

struct BigPotrfArgs {
  Operand D;     // n x n working block (in: D_j lower; out: L lower)
  Operand Linv;  // n x n output (full, zero upper)
  const int* seps;
  long long N;
  int base_mode, j, n, level;
  int csize;     // CTAs per segment (a thread-block cluster when > 1)
  int k0;        // first segment of this launch
  DevErr* err;
};

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Blocked Cholesky + inverse of an n x n block (n = 64 NB).  One segment per thread-block
// cluster of `csize` CTAs (csize = 1: one CTA per segment): rank 0 factors the 64 x 64 diagonal
// tiles (potrf_trtri), the panel, trailing-update and inverse tile GEMMs of each phase are dealt
// round-robin to the cluster's CTAs, and the phases are separated by cluster barriers (the tiles
// live in global memory / L2; barrier.cluster release/acquire orders them).  Levels with few
// segments (the serial base, narrow levels) use clusters so one block's tile work spreads over
// several SMs instead of running serially in one CTA.
__global__ void __launch_bounds__(BTHREADS) big_potrf_kernel(BigPotrfArgs g) {
  using S = FactorShape<64>;
  constexpr int LD = S::LD;
  const int C = g.csize;
  const int k = g.k0 + blockIdx.x / C, rank = blockIdx.x % C;
  int J;
  // exits must be uniform over a cluster (cluster barriers follow): with csize > 1 a segment does
  // not skip on another segment's error (its own step-(j-1) failure was already reported, and a
  // later report can never supersede an earlier one)
  if (C == 1 && cta_superseded(g.err, g.level, g.j, k)) return;
  if (!segment_active(g.seps, g.base_mode, g.N, k, g.j, kActAll, J)) return;
  extern __shared__ __align__(16) double sm[];
  double* DL = sm;             // 64 x LD diagonal tile (rank 0)
  double* As = DL + BT * LD;   // two-stage staging of the tile GEMMs (4 * GSTAGE doubles)
  __shared__ int s_fail;
  double* D = const_cast<double*>(operand_ptr(g.D, g.seps, g.base_mode, k, g.j));
  double* Li = const_cast<double*>(operand_ptr(g.Linv, g.seps, g.base_mode, k, g.j));
  const int n = g.n, NB = n / BT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rw = (warp >> 1) * 16, cw = (warp & 1) * 32;
  auto store_acc = [&](double* dst, int ld, double (&acc)[2][4][2], double sign, const double* addsrc) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = rw + i * 8 + (lane >> 2), c = cw + q * 8 + 2 * (lane & 3) + h;
          const double v = sign * acc[i][q][h];
          dst[(size_t)r * ld + c] = addsrc ? addsrc[(size_t)r * ld + c] + v : v;
        }
  };
  auto csync = [&]() {
    if (C > 1) cluster_sync_all();
    else __syncthreads();
  };
  double acc[2][4][2];
  for (int kb = 0; kb < NB; ++kb) {
    // diagonal tile -> DL, factor + invert (rank 0, warps 0..3, named barrier 1)
    if (rank == 0) {
      __syncthreads();
      for (int e = tid; e < BT * BT; e += BTHREADS) DL[(e / BT) * LD + e % BT] = D[(size_t)(kb * BT + e / BT) * n + kb * BT + e % BT];
      __syncthreads();
      // the single-warp left-looking pivot chain, then the inverse by recursive doubling on
      // group A (the schedule of factor_level_kernel<64>)
      int fail = 0;
      if (warp < S::NWA) {
        if (warp == 0) {
          const int f = chain_potrf<LD, 64>(DL, lane);
          if (lane == 0) s_fail = f;
        }
        named_sync(kBarA, S::NWA * 32);
        fail = s_fail;
        if (!fail) trtri_doubling<64>(DL, warp, lane);
      }
      __syncthreads();
      if (tid == 0) s_fail = fail;
      __syncthreads();
      if (s_fail) {
        if (tid == 0) report_npd(g.err, g.level, g.j, k, kb * BT + s_fail);
      } else {
        // Linv_kk -> Li (full tile, zero upper); L_kk is not needed again
        for (int e = tid; e < BT * BT; e += BTHREADS) {
          const int r = e / BT, c = e % BT;
          Li[(size_t)(kb * BT + r) * n + kb * BT + c] = c <= r ? DL[r * LD + c] : 0.0;
        }
      }
    }
    csync();
    if (C > 1) {  // every other rank learns the outcome from rank 0's shared memory
      if (tid == 0 && rank != 0) {
        unsigned addr = (unsigned)__cvta_generic_to_shared(&s_fail), remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(addr));
        int f;
        asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(f) : "r"(remote) : "memory");
        s_fail = f;
      }
      __syncthreads();
      const int f = s_fail;
      csync();  // rank 0's flag is not reused before everyone has read it
      if (f) return;
    } else if (s_fail) {
      return;
    }
    // panel: L_ib = A_ib Linv_kk^T  (i > kb), in place in D
    for (int ib = kb + 1 + rank; ib < NB; ib += C) {
      gemm_tile_pipelined<false, true>(acc, D + (size_t)ib * BT * n + kb * BT, n, Li + (size_t)kb * BT * n + kb * BT, n, BT, BT, BT, 0, 0, 0, BT, As);
      __syncthreads();
      store_acc(D + (size_t)ib * BT * n + kb * BT, n, acc, 1.0, nullptr);
    }
    csync();
    // trailing: A_ij -= L_ib L_jb^T  (kb < jb <= ib), tiles dealt round-robin
    int t = 0;
    for (int ib = kb + 1; ib < NB; ++ib)
      for (int jb = kb + 1; jb <= ib; ++jb, ++t) {
        if (t % C != rank) continue;
        gemm_tile_pipelined<false, true>(acc, D + (size_t)ib * BT * n + kb * BT, n, D + (size_t)jb * BT * n + kb * BT, n, BT, BT, BT, 0, 0, 0, BT, As);
        __syncthreads();
        double* tt = D + (size_t)ib * BT * n + jb * BT;
        store_acc(tt, n, acc, -1.0, tt);
      }
    csync();
  }
  // inverse, block row by block row: Linv_ij = -Linv_ii sum_{m=j}^{i-1} L_im Linv_mj  (i > j)
  // T = sum_m L_im Linv_mj is formed in the (unused) strict upper tile D[j][i] as scratch.
  for (int ib = 1; ib < NB; ++ib) {
    for (int jb = rank; jb < ib; jb += C) {
      // T = L[ib][jb..ib-1] * Linv[jb..ib-1][jb]   (k range (ib - jb) tiles)
      gemm_tile_pipelined<false, false>(acc, D + (size_t)ib * BT * n + jb * BT, n, Li + (size_t)jb * BT * n + jb * BT, n, BT, BT, (ib - jb) * BT, 0, 0, 0, (ib - jb) * BT, As);
      __syncthreads();
      store_acc(D + (size_t)jb * BT * n + ib * BT, n, acc, 1.0, nullptr);
    }
    csync();
    for (int jb = rank; jb < ib; jb += C) {
      gemm_tile_pipelined<false, false>(acc, Li + (size_t)ib * BT * n + ib * BT, n, D + (size_t)jb * BT * n + ib * BT, n, BT, BT, BT, 0, 0, 0, BT, As);
      __syncthreads();
      store_acc(Li + (size_t)ib * BT * n + jb * BT, n, acc, -1.0, nullptr);
    }
    csync();
  }
  // zero the strict upper off-diagonal tiles of Linv
  int t = 0;
  for (int ib = 0; ib < NB; ++ib)
    for (int jb = ib + 1; jb < NB; ++jb, ++t) {
      if (t % C != rank) continue;
      for (int e = tid; e < BT * BT; e += BTHREADS) Li[(size_t)(ib * BT + e / BT) * n + jb * BT + e % BT] = 0.0;
    }
}

}  // namespace btd
