// Small-block (n <= 8) level elimination and level solve: one 8-lane group of a warp per segment
// (lane = one block row), 4 segments per warp, 16 per 128-thread CTA.
//
// At n = 8 (BASELINE config 3, N = 2^20) a 64-element block is far too small for a CTA-per-segment
// kernel (factor_level_kernel<8> would keep one warp per segment at ~16 CTAs/SM, latency bound).
// Here the per-step algebra is row-parallel inside the group and the blocks move through small
// per-group shared-memory tiles: coalesced cp.async streaming one step ahead, cross-lane exchange
// by broadcast shared-memory reads.  (Round 1 exchanged rows with width-8 warp shuffles: ~470 SHFL
// per warp-step, and SHFL issues at one warp-instruction per clock per SM -- the level-0 factor of
// config 3 took 1.04 ms; with the shared-memory exchange 0.66 ms.)
//
// Factor (same Y-form algebra as factor_level_kernel, reference chain permute_split /
// factorize_btd_batch / solve_btd_batch(F) / compute_schur, bt/schur.py:98-193,
// bt/block_cholesky.py:24-68), per step j with lane r holding row r:
//   L L^T = D_j (redundant in every lane of the group)  Linv = L^{-1} (row r by lane r) -> HBM
//   Pt1 = X1 Linv^T, Pt2 = Gt Linv^T                   -> L_{j+1,j} = Pt1 -> HBM
//   D_{j+1} = A_{j+1,j+1} - Pt1 Pt1^T, Gt_{j+1} = -Pt2 Pt1^T, S_L += Pt2 Pt2^T
//   last row: S_R = Pt1 Pt1^T, S_sub = -Pt1 Pt2^T.
#pragma once

#include "btd_factor.cuh"
#include "btd_solve.cuh"
#include "btd_solve2.cuh"

namespace btd {

constexpr int kSmallNT = 8;
constexpr int kSmallThreads = 128;  // 4 warps, 16 segments per CTA

// row r of an n x n row-major block (zero padded to 8; `eye` puts 1 on padded diagonal entries)
__device__ __forceinline__ void load_row8(double (&v)[8], const double* blk, int n, int r, bool ok, bool eye) {
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = (ok && r < n && c < n) ? blk[r * n + c] : ((eye && r == c && r >= n) ? 1.0 : 0.0);
}
// column r of an n x n block (= row r of its transpose)
__device__ __forceinline__ void load_col8(double (&v)[8], const double* blk, int n, int r, bool ok) {
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = (ok && r < n && c < n) ? blk[c * n + r] : 0.0;
}
__device__ __forceinline__ void store_row8(double* blk, const double (&v)[8], int n, int r, bool ok) {
  if (!ok || r >= n) return;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (c < n) blk[r * n + c] = v[c];
}

// ============================================================================================
// factor_small_kernel.  Per 8-lane group (segment), 8 x 8 tiles in shared memory
// (row stride 10 doubles: the 8 rows of a tile fall in 8 different 16-byte bank quads):
//   tA  A_{j+1,j+1}, tX  X1 = A_{j+1,j} (or C_R): streamed with cp.async one step ahead, lane r
//       copies and later reads only its own row r (no cross-lane hazard, no barrier);
//   tD  D_j for the Cholesky, then Pt1;   tL  rows of Linv_j, then Pt2;   tS  S_L (own row).
// Per step (lane r = block row r):
//   1. row r of D_j -> tD; every lane of the group factors the whole 8 x 8 lower triangle
//      redundantly in registers (20 broadcast LDS.128, no communication inside the pivot chain);
//   2. lane r forms row r of Linv_j = L_j^{-1} from its copy of L (backward substitution over
//      columns) -> tL and the packed hierarchy row;
//   3. Pt1 = X1 Linv^T, Pt2 = Gt Linv^T, row r by lane r (Linv rows read as broadcasts);
//      Pt1 row -> L_sub (HBM) and tD, Pt2 row -> tL;
//   4. D_{j+1} = A - Pt1 Pt1^T, Gt_{j+1} = -Pt2 Pt1^T, S_L += Pt2 Pt2^T (rows of Pt1 / Pt2 read as
//      broadcasts); last row: S_R = Pt1 Pt1^T, S_sub = -Pt1 Pt2^T.
// ~130 shared-memory instructions per warp-step instead of ~470 SHFL + ~60 scalar global accesses.
// ============================================================================================
constexpr int kS2LD = 10;                       // padded tile row stride (doubles)
constexpr int kS2Tile = 8 * kS2LD;              // one 8 x 8 tile
constexpr int kS2Group = 5 * kS2Tile + 2;       // +16 B: the 4 groups of a warp start in different bank quads
constexpr int kS2Warps = 4;                     // 128 threads, 16 segments per CTA
constexpr size_t kS2Smem = (size_t)kS2Warps * 4 * kS2Group * sizeof(double);

// An n x n block -> the group's padded tile, coalesced: lane l of the group moves the 16-byte chunks
// l, l+8, l+16, l+24 of the contiguous block (8 lanes cover 128 contiguous bytes per instruction).
// Only the n x n part is written (the tile's padding stays as initialised).  The rows are read by
// other lanes: cp.async wait + __syncwarp before use.
__device__ __forceinline__ void s2_block_async(double* tile, const double* blk, int n, int l, bool ok) {
  if (!ok) return;
  if (n == 8) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = l + 8 * i;
      cp_async16(tile + (c >> 2) * kS2LD + 2 * (c & 3), blk + 2 * c, 16);
    }
  } else if ((n & 1) == 0) {
    const int nc = n * n / 2;
    for (int c = l; c < nc; c += 8) {
      const int e = 2 * c;
      cp_async16(tile + (e / n) * kS2LD + e % n, blk + e, 16);
    }
  } else {
    const int ne = n * n;
    for (int e = l; e < ne; e += 8) cp_async8(tile + (e / n) * kS2LD + e % n, blk + e, 8);
  }
}
__device__ __forceinline__ void s2_ld_row(double (&v)[8], const double* trow) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double2 t = *reinterpret_cast<const double2*>(trow + 2 * q);
    v[2 * q] = t.x;
    v[2 * q + 1] = t.y;
  }
}
__device__ __forceinline__ void s2_st_row(double* trow, const double (&v)[8]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) *reinterpret_cast<double2*>(trow + 2 * q) = make_double2(v[2 * q], v[2 * q + 1]);
}
// row r of an n x n block in HBM (n even: 16-byte stores)
__device__ __forceinline__ void s2_st_global_row(double* blk, const double (&v)[8], int n, int r) {
  if (r >= n) return;
  double* row = blk + (size_t)r * n;
  if ((n & 1) == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (2 * q < n) *reinterpret_cast<double2*>(row + 2 * q) = make_double2(v[2 * q], v[2 * q + 1]);
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < n) row[c] = v[c];
  }
}

// three CTAs per SM: 168 registers, no spills (four CTAs at 128 registers spill the pivot block
// and measured slower: level 0 of cfg3 0.649 vs 0.598 ms)
__global__ void __launch_bounds__(kSmallThreads, 3) factor_small_kernel(FactorArgs a) {
  extern __shared__ __align__(16) double s2sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 3, r = lane & 7;
  const bool coupled = !a.base;
  const int kend = a.kend ? a.kend : a.K;
  const int k = coupled ? a.k0 + (blockIdx.x * 4 + warp) * 4 + g : 0;
  const bool valid = coupled ? (k < kend) : (blockIdx.x == 0 && warp == 0 && g == 0);
  const int n = a.n;
  const size_t bs = (size_t)n * n;
  const int pk = packed_offset_(n);
  // CTA-uniform early exit (the CTA's first segment has the lowest k)
  if (cta_superseded(a.err, a.level, 0, coupled ? a.k0 + blockIdx.x * 16 : 0)) return;
  const long long start = !valid ? 0 : (coupled ? (long long)a.seps[k] + 1 : 0);
  const long long stop = !valid ? 0 : (coupled ? (long long)a.seps[k + 1] : a.N);
  const int J = (int)(stop - start);
  int jw = J;  // the warp iterates to its longest segment (__syncwarp needs the whole warp)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) jw = max(jw, __shfl_xor_sync(0xffffffffu, jw, o));

  double* tA = s2sm + (warp * 4 + g) * kS2Group;
  double* tX = tA + kS2Tile;
  double* tD = tX + kS2Tile;
  double* tL = tD + kS2Tile;
  double* rS = tL + kS2Tile + r * kS2LD;  // this lane's row of the running S_L (own row only)
  double* rA = tA + r * kS2LD;
  double* rX = tX + r * kS2LD;
  const double* fb = a.diag;
  // X1 of step j: A_{j+1,j} inside the segment; C_R at the last row of a coupled segment
  auto x_src = [&](int j) -> const double* {
    return (j + 1 < J) ? a.sub + (start + j) * bs : a.sub + (stop - 1) * bs;
  };
  auto x_ok = [&](int j) { return valid && j < J && (coupled || j + 1 < J); };

  // ---- segment start: A_0 -> tA, X_0 -> tX, Gt_0 = C_L^T, the hierarchy's coupling copies ----
  {
    double z[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) z[c] = 0.0;
    s2_st_row(rA, z);
    s2_st_row(rX, z);
  }
  __syncwarp();
  s2_block_async(tA, valid ? a.diag + start * bs : fb, n, r, valid);
  cp_async_commit();
  s2_block_async(tX, x_ok(0) ? x_src(0) : fb, n, r, x_ok(0));
  cp_async_commit();
  double G[8], Dr[8];
  {
    double z[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) z[c] = 0.0;
    s2_st_row(rS, z);
  }
  if (valid && coupled) {
    load_col8(G, a.sub + (start - 1) * bs, n, r, true);
    // the hierarchy's copies of C_L and C_R (two contiguous blocks: 16-byte copies for even n)
    if ((n & 1) == 0) {
      const int nc = n * n / 2;
      const double2* cl = reinterpret_cast<const double2*>(a.sub + (start - 1) * bs);
      const double2* cr = reinterpret_cast<const double2*>(a.sub + (stop - 1) * bs);
      double2* dl = reinterpret_cast<double2*>(a.Lsub + (start - 1) * bs);
      double2* dr = reinterpret_cast<double2*>(a.Lsub + (stop - 1) * bs);
      for (int c = r; c < nc; c += 8) {
        dl[c] = cl[c];
        dr[c] = cr[c];
      }
    } else {
      double t[8];
      load_row8(t, a.sub + (start - 1) * bs, n, r, true, false);
      store_row8(a.Lsub + (start - 1) * bs, t, n, r, true);
      load_row8(t, a.sub + (stop - 1) * bs, n, r, true, false);
      store_row8(a.Lsub + (stop - 1) * bs, t, n, r, true);
    }
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) G[c] = 0.0;
  }
  cp_async_wait_group<1>();
  __syncwarp();
  s2_ld_row(Dr, rA);
  if (r >= n) {
#pragma unroll
    for (int c = 0; c < 8; ++c) Dr[c] = (c == r) ? 1.0 : 0.0;
  }
  __syncwarp();  // every lane has read its row of A_0
  s2_block_async(tA, a.diag + (start + 1) * bs, n, r, valid && J > 1);  // A_1
  cp_async_commit();

  int fail = 0, fail_j = 0;
  for (int j = 0; j < jw; ++j) {
    const bool act = valid && j < J && fail == 0;
    const bool last = (j == J - 1);
    // ---- 1. D_j -> tD; redundant Cholesky of the whole block in every lane of the group ----
    __syncwarp();  // the previous step's reads of Pt1 (tD) / Pt2 (tL) are done
    s2_st_row(tD + r * kS2LD, Dr);
    __syncwarp();
    double L[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c <= i; c += 2) {
        const double2 t = *reinterpret_cast<const double2*>(tD + i * kS2LD + c);
        L[i][c] = t.x;
        if (c + 1 <= i) L[i][c + 1] = t.y;
      }
    double ri[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const double d = L[kk][kk];
      if (act && fail == 0 && d <= 0.0) fail = kk + 1;
      ri[kk] = rsqrt(d);
      L[kk][kk] = d * ri[kk];
#pragma unroll
      for (int i = kk + 1; i < 8; ++i) L[i][kk] *= ri[kk];
#pragma unroll
      for (int i = kk + 1; i < 8; ++i)
#pragma unroll
        for (int c = kk + 1; c <= i; ++c) L[i][c] = fma(-L[i][kk], L[c][kk], L[i][c]);
    }
    if (fail && act) fail_j = j;
    // ---- 2. row r of Linv: x L = e_r, columns 7..0 ----
    double x[8];
#pragma unroll
    for (int c = 7; c >= 0; --c) {
      double s = (c == r) ? 1.0 : 0.0;
#pragma unroll
      for (int i = c + 1; i < 8; ++i) s = fma(-x[i], L[i][c], s);
      x[c] = (c <= r) ? s * ri[c] : 0.0;
    }
    s2_st_row(tL + r * kS2LD, x);
    if (act && r < n) {  // packed row r: columns 0..r, zero pad for even r
      double* row = a.Linv + (start + j) * (size_t)pk + packed_offset_(r);
      const int len = ((r + 2) >> 1) << 1;
      if ((pk & 1) == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (2 * q < len) *reinterpret_cast<double2*>(row + 2 * q) = make_double2(x[2 * q], x[2 * q + 1]);
      }
    }
    __syncwarp();
    // ---- 3. Pt1 = X1 Linv^T, Pt2 = Gt Linv^T (row r) ----
    cp_async_wait_group<1>();  // X_j (A_{j+1} may still be in flight)
    __syncwarp();
    double Xr[8];
    s2_ld_row(Xr, rX);
    double P1[8], P2[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double lc[8];
#pragma unroll
      for (int q = 0; q <= c; q += 2) {
        const double2 t = *reinterpret_cast<const double2*>(tL + c * kS2LD + q);
        lc[q] = t.x;
        lc[q + 1] = t.y;
      }
      double s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int q = 0; q <= c; ++q) {
        s1 = fma(Xr[q], lc[q], s1);
        s2 = fma(G[q], lc[q], s2);
      }
      P1[c] = s1;
      P2[c] = s2;
    }
    if (act && !last) s2_st_global_row(a.Lsub + (start + j) * bs, P1, n, r);  // L_{j+1,j}
    __syncwarp();  // every lane is done with X_j, the Linv rows (tL) and the Cholesky reads (tD)
    const bool xnext = x_ok(j + 1) && act;
    s2_block_async(tX, xnext ? x_src(j + 1) : fb, n, r, xnext);  // X_{j+1}
    cp_async_commit();
    s2_st_row(tD + r * kS2LD, P1);
    s2_st_row(tL + r * kS2LD, P2);
    __syncwarp();
    // ---- 4. products with the rows of Pt1 / Pt2 ----
    cp_async_wait_group<1>();  // A_{j+1}
    __syncwarp();
    s2_ld_row(Dr, rA);  // A_{j+1,j+1} row r (stale / zero past the segment: unused)
    const bool fin = act && last && coupled && r < n;
    double SL[8];
    s2_ld_row(SL, rS);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      double p1[8], p2[8];
      s2_ld_row(p1, tD + b * kS2LD);
      s2_ld_row(p2, tL + b * kS2LD);
      double s11 = 0.0, s21 = 0.0, s22 = 0.0, s12 = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        s11 = fma(P1[q], p1[q], s11);
        s21 = fma(P2[q], p1[q], s21);
        s22 = fma(P2[q], p2[q], s22);
        s12 = fma(P1[q], p2[q], s12);
      }
      Dr[b] = (r >= n) ? ((b == r) ? 1.0 : 0.0) : Dr[b] - s11;
      G[b] = -s21;
      if (coupled) SL[b] += s22;
      if (fin && b < n) {
        a.Sr[(size_t)k * bs + r * n + b] = s11;
        a.Ssub[(size_t)k * bs + r * n + b] = -s12;
      }
    }
    if (coupled) s2_st_row(rS, SL);
    if (fin) store_row8(a.Sl + (size_t)k * bs, SL, n, r, true);
    __syncwarp();  // every lane has read its row of A_{j+1}
    const bool anext = act && j + 2 < J;
    s2_block_async(tA, anext ? a.diag + (start + j + 2) * bs : fb, n, r, anext);  // A_{j+2}
    cp_async_commit();
  }
  cp_async_wait_all();
  if (fail && r == 0 && valid && fail <= n) report_npd(a.err, a.level, fail_j, k, fail);
}

// ============================================================================================
// solve_small_kernel<DC>: the level solve for n <= 8 (same algebra, outputs and argument contract
// as solve_level_kernel / solve_tma_kernel, btd_solve.cuh; Alg. 5-7 of the reference,
// bt/schur.py:196-286).  Per step, the group's Lsub block and packed Linv block are
// moved into shared memory with coalesced cp.async one step ahead (double-buffered; L2 hints:
// forward sweep evict_last, backward sweep -- their last use -- evict_first), lane r reads row r
// (forward) or column r (backward) from the tile, and the two per-step vectors (t, then z / w) are
// exchanged through shared memory: ~25-30 shared-memory instructions per warp-step instead of
// ~17 scalar uncoalesced loads + 32 SHFL (DC = 1).
// ============================================================================================
template <int DC>
struct SS2 {
  static constexpr int PK = 40;                                   // packed Linv block, n = 8
  static constexpr int GROUP = 2 * kS2Tile + 2 * PK + 16 * DC + 2;  // +16 B: groups in distinct bank quads
  static constexpr size_t SMEM = (size_t)16 * GROUP * sizeof(double);
};

__device__ __forceinline__ void cp_async16_hint(void* smem, const void* gmem, unsigned long long pol) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, 16, %2;\n" ::"r"(s), "l"(gmem), "l"(pol));
}
__device__ __forceinline__ void cp_async8_hint(void* smem, const void* gmem, unsigned long long pol) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, 8, %2;\n" ::"r"(s), "l"(gmem), "l"(pol));
}
// n x n block -> padded tile (coalesced, see s2_block_async), with an L2 policy
__device__ __forceinline__ void ss2_block(double* tile, const double* blk, int n, int l, unsigned long long pol) {
  if (n == 8) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = l + 8 * i;
      cp_async16_hint(tile + (c >> 2) * kS2LD + 2 * (c & 3), blk + 2 * c, pol);
    }
  } else if ((n & 1) == 0) {
    for (int c = l; c < n * n / 2; c += 8) cp_async16_hint(tile + (2 * c / n) * kS2LD + (2 * c) % n, blk + 2 * c, pol);
  } else {
    for (int e = l; e < n * n; e += 8) cp_async8_hint(tile + (e / n) * kS2LD + e % n, blk + e, pol);
  }
}
// packed Linv block (pk doubles, pk even, 16-byte aligned) -> tile
__device__ __forceinline__ void ss2_packed(double* tile, const double* blk, int pk, int l, unsigned long long pol) {
  for (int c = l; c < pk / 2; c += 8) cp_async16_hint(tile + 2 * c, blk + 2 * c, pol);
}

template <int DC>
__global__ void __launch_bounds__(kSmallThreads) solve_small_kernel(SolveArgs a) {
  extern __shared__ __align__(16) double ss2sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 3, r = lane & 7;
  const int n = a.n, d = a.d, mode = a.mode;
  const int c0 = blockIdx.y * DC;
  const bool base = mode == kSolveBase;
  const int k = base ? 0 : (blockIdx.x * 4 + warp) * 4 + g;
  const bool valid = base ? (blockIdx.x == 0 && warp == 0 && g == 0) : (k < a.K);
  if (error_raised(a.err)) return;
  const size_t bs = (size_t)n * n, ps = (size_t)n * d;
  const int pk = packed_offset_(n);
  const long long start = !valid ? 0 : (base ? 0 : (long long)a.seps[k] + 1);
  const long long stop = !valid ? 0 : (base ? a.N : (long long)a.seps[k + 1]);
  const int J = (int)(stop - start);
  int jw = J;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) jw = max(jw, __shfl_xor_sync(0xffffffffu, jw, o));
  const bool rv = valid && r < n;
  const unsigned long long pol_keep = l2_policy_evict_last(), pol_drop = l2_policy_evict_first();

  double* tM = ss2sm + (warp * 4 + g) * SS2<DC>::GROUP;  // 2 Lsub tiles
  double* tP = tM + 2 * kS2Tile;                          // 2 packed Linv blocks
  double* tt = tP + 2 * SS2<DC>::PK;                      // t (8 x DC)
  double* tz = tt + 8 * DC;                               // z / w (8 x DC)
  // zero the tiles once: the padding past n is never written by the copies
#pragma unroll
  for (int c = 0; c < 2 * kS2Tile + 2 * SS2<DC>::PK + 16 * DC; c += 8) tM[c + r] = 0.0;
  __syncwarp();

  auto ld_vec = [&](const double* p, double (&v)[DC]) {  // row r of an n x d panel, columns c0..
#pragma unroll
    for (int c = 0; c < DC; ++c) v[c] = (p && rv && c0 + c < d) ? p[(size_t)r * d + c0 + c] : 0.0;
  };
  auto st_vec = [&](double* p, const double (&v)[DC], bool ok) {
    if (!ok || !rv || !p) return;
#pragma unroll
    for (int c = 0; c < DC; ++c)
      if (c0 + c < d) p[(size_t)r * d + c0 + c] = v[c];
  };
  auto publish = [&](double* vec, const double (&v)[DC]) {
#pragma unroll
    for (int c = 0; c < DC; ++c) vec[r * DC + c] = v[c];
  };
  auto gather = [&](const double* vec, double (&all)[8][DC]) {
#pragma unroll
    for (int e = 0; e < 8 * DC; e += 2) {
      const double2 t = *reinterpret_cast<const double2*>(vec + e);
      all[e / DC][e % DC] = t.x;
      all[(e + 1) / DC][(e + 1) % DC] = t.y;
    }
  };
  // one-off mat-vecs of the coupling blocks (corrections / fold): y += op(M) v, v from the group
  auto mv_once = [&](const double* M, bool trans, const double (&v)[DC], double (&y)[DC], bool ok) {
    __syncwarp();
    publish(tt, v);
    __syncwarp();
    double all[8][DC];
    gather(tt, all);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double m = (ok && rv && q < n) ? (trans ? M[(size_t)q * n + r] : M[(size_t)r * n + q]) : 0.0;
#pragma unroll
      for (int c = 0; c < DC; ++c) y[c] = fma(m, all[q][c], y[c]);
    }
  };

  double corr0[DC], corr1[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) corr0[c] = corr1[c] = 0.0;
  if (mode == kSolveUp) {
    double xs0[DC], xs1[DC];
    ld_vec(valid ? a.xsep + (size_t)k * ps : nullptr, xs0);
    ld_vec(valid ? a.xsep + (size_t)(k + 1) * ps : nullptr, xs1);
    mv_once(valid ? a.Lsub + (start - 1) * bs : nullptr, false, xs0, corr0, valid);  // C_L x_L
    mv_once(valid ? a.Lsub + (stop - 1) * bs : nullptr, true, xs1, corr1, valid);    // C_R^T x_R
    st_vec(valid ? a.x + (start - 1) * ps : nullptr, xs0, valid);                    // separator rows
    st_vec(valid ? a.x + stop * ps : nullptr, xs1, valid && k == a.K - 1);
  }

  // ---- forward sweep: z_j = Linv_j (b_j - L_{j,j-1} z_{j-1}) ----
  auto issue_fwd = [&](int j) {
    const bool act = valid && j < J;
    double* M = tM + (j & 1) * kS2Tile;
    double* P = tP + (j & 1) * SS2<DC>::PK;
    if (act && j > 0) ss2_block(M, a.Lsub + (start + j - 1) * bs, n, r, pol_keep);
    if (act) ss2_packed(P, a.Linv + (start + j) * (size_t)pk, pk, r, pol_keep);
    cp_async_commit();
  };
  double z[DC], fb[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) z[c] = 0.0;
  __syncwarp();
  publish(tz, z);
  issue_fwd(0);
  ld_vec(valid && J > 0 ? a.rhs + start * ps : nullptr, fb);
  const int lenr = ((r + 2) >> 1) << 1;
  for (int j = 0; j < jw; ++j) {
    const bool act = valid && j < J;
    issue_fwd(j + 1);
    double nb[DC];
    ld_vec(valid && j + 1 < J ? a.rhs + (start + j + 1) * ps : nullptr, nb);
    cp_async_wait_group<1>();
    __syncwarp();
    const double* M = tM + (j & 1) * kS2Tile;
    const double* P = tP + (j & 1) * SS2<DC>::PK;
    double t[DC];
#pragma unroll
    for (int c = 0; c < DC; ++c) {
      t[c] = fb[c];
      if (act && j == 0) t[c] -= corr0[c];
      if (act && j == J - 1) t[c] -= corr1[c];
    }
    if (j > 0) {
      double m[8], zall[8][DC];
      s2_ld_row(m, M + r * kS2LD);
      gather(tz, zall);
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int c = 0; c < DC; ++c) t[c] = fma(-m[q], zall[q][c], t[c]);
    }
    publish(tt, t);
    __syncwarp();
    double tall[8][DC], zn[DC];
    gather(tt, tall);
#pragma unroll
    for (int c = 0; c < DC; ++c) zn[c] = 0.0;
#pragma unroll
    for (int q = 0; q < 8; q += 2) {
      if (q < lenr) {
        const double2 pv = *reinterpret_cast<const double2*>(P + packed_offset_(r) + q);
#pragma unroll
        for (int c = 0; c < DC; ++c) zn[c] = fma(pv.y, tall[q + 1][c], fma(pv.x, tall[q][c], zn[c]));
      }
    }
    if (act) {
#pragma unroll
      for (int c = 0; c < DC; ++c) z[c] = zn[c];
    }
    st_vec(act ? a.x + (start + j) * ps : nullptr, z, act);
    publish(tz, z);
    __syncwarp();
#pragma unroll
    for (int c = 0; c < DC; ++c) fb[c] = nb[c];
  }
  cp_async_wait_all();
  __syncwarp();

  // ---- backward sweep: w_j = Linv_j^T (z_j - L_{j+1,j}^T w_{j+1}) ----
  auto jof = [&](int jj) { return jj - (jw - J); };  // group-local row of warp iteration jj
  auto issue_bwd = [&](int jj) {
    const int j = jof(jj);
    const bool act = valid && j >= 0 && jj >= 0;
    double* M = tM + (jj & 1) * kS2Tile;
    double* P = tP + (jj & 1) * SS2<DC>::PK;
    if (act && j < J - 1) ss2_block(M, a.Lsub + (start + j) * bs, n, r, pol_drop);
    if (act) ss2_packed(P, a.Linv + (start + j) * (size_t)pk, pk, r, pol_drop);
    cp_async_commit();
  };
  double w[DC], w_last[DC], bz[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) w[c] = w_last[c] = 0.0;
  publish(tz, w);
  issue_bwd(jw - 1);
  {
    const int j = jof(jw - 1);
    ld_vec(valid && j >= 0 ? a.x + (start + j) * ps : nullptr, bz);
  }
  __syncwarp();
  for (int jj = jw - 1; jj >= 0; --jj) {
    const int j = jof(jj);
    const bool act = valid && j >= 0;
    issue_bwd(jj - 1);
    double nz[DC];
    {
      const int jn = jof(jj - 1);
      ld_vec(valid && jj >= 1 && jn >= 0 ? a.x + (start + jn) * ps : nullptr, nz);
    }
    cp_async_wait_group<1>();
    __syncwarp();
    const double* M = tM + (jj & 1) * kS2Tile;
    const double* P = tP + (jj & 1) * SS2<DC>::PK;
    double t[DC];
#pragma unroll
    for (int c = 0; c < DC; ++c) t[c] = bz[c];
    if (act && j < J - 1) {
      double wall[8][DC];
      gather(tz, wall);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double m = M[q * kS2LD + r];  // L_{j+1,j}[q][r]
#pragma unroll
        for (int c = 0; c < DC; ++c) t[c] = fma(-m, wall[q][c], t[c]);
      }
    }
    publish(tt, t);
    __syncwarp();
    double tall[8][DC], wn[DC];
    gather(tt, tall);
#pragma unroll
    for (int c = 0; c < DC; ++c) wn[c] = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double pv = (q >= r) ? P[packed_offset_(q) + r] : 0.0;  // Linv[q][r]
#pragma unroll
      for (int c = 0; c < DC; ++c) wn[c] = fma(pv, tall[q][c], wn[c]);
    }
    if (act) {
#pragma unroll
      for (int c = 0; c < DC; ++c) w[c] = wn[c];
    }
    if (mode != kSolveDown) st_vec(act ? a.x + (start + j) * ps : nullptr, w, act);
    if (act && j == J - 1) {
#pragma unroll
      for (int c = 0; c < DC; ++c) w_last[c] = w[c];
    }
    publish(tz, w);
    __syncwarp();
#pragma unroll
    for (int c = 0; c < DC; ++c) bz[c] = nz[c];
  }
  cp_async_wait_all();
  if (mode == kSolveDown) {  // fold: f_R = C_R w_last ; f_L = C_L^T w_0
    double fr[DC], fl[DC];
#pragma unroll
    for (int c = 0; c < DC; ++c) fr[c] = fl[c] = 0.0;
    mv_once(valid ? a.Lsub + (stop - 1) * bs : nullptr, false, w_last, fr, valid);
    mv_once(valid ? a.Lsub + (start - 1) * bs : nullptr, true, w, fl, valid);
    st_vec(valid ? a.fr + (size_t)k * ps : nullptr, fr, valid);
    st_vec(valid ? a.fl + (size_t)k * ps : nullptr, fl, valid);
  }
}

}  // namespace btd
