// Fused per-level segment elimination for n <= 64 (one CTA per interior segment).
//
// Replaces, for one recursion level, the reference chain
//   permute_split            bt/schur.py:98-138
//   factorize_btd_batch      bt/block_cholesky.py:24-42,60-68   (potrf / trsm / gemm sweeps)
//   _coupling_panels         bt/schur.py:141-153
//   solve_btd_batch(F)       bt/block_cholesky.py:45-57 via bt/schur.py:339-341
//   compute_schur            bt/schur.py:156-193
// with ONE launch.  Algorithm ("Y-form"): eliminate the segment rows in order,
// carrying the fill coupling G_j between the current row and the left separator:
//
//   Linv_j          = chol(D_j)^{-1}                       (stored; the solve only needs Linv, L_sub)
//   [P1 | P2]       = Linv_j [A_{j+1,j}^T | G_j]            (P1 = L_{j+1,j}^T, P2 = Y_L[j])
//   D_{j+1}         = A_{j+1,j+1} - P1^T P1
//   G_{j+1}         = -P1^T P2
//   S_L            += P2^T P2                              (Schur downdate of the left separator)
// and at the last row, with P1 := Linv C_R^T (= Y_R):
//   S_R = Y_R^T Y_R ,  S_sub = -Y_R^T Y_L[last]
// Everything lives in shared memory in transposed form Pt = [P1^T ; P2^T] so that every product is
// an "A row-major x B col-major" DMMA (mma.sync.m8n8k4.f64):  Pt = Xt Linv^T  and  C = Pt Pt^T.
// The lower triangle of C holds [D-update | G^T | S_L] at once.
#pragma once

#include "btd_device.cuh"

namespace btd {

#ifdef BTD_PHASE_PROF
__device__ unsigned long long g_phase_cycles[16];
#define BTD_PHASE_INIT() long long _ph_last = clock64();
#define BTD_PHASE(i)                                                        \
  do {                                                                      \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                              \
      long long _now = clock64();                                           \
      atomicAdd(&g_phase_cycles[i], (unsigned long long)(_now - _ph_last)); \
      _ph_last = _now;                                                      \
    }                                                                       \
  } while (0)
#else
#define BTD_PHASE_INIT()
#define BTD_PHASE(i)
#endif

struct FactorArgs {
  const double* diag;  // level matrix: (N, n, n)
  const double* sub;   // (N-1, n, n), sub[i] = A_{i+1,i}
  const int* seps;     // (K+1) separators of this level (unused for the base)
  long long N;
  int n;
  int K;        // segments (base: 1)
  int k0;       // first segment of this launch (blockIdx.x = k - k0): chunked level-0 launches
  int kend;     // one past the last segment of this launch (0: K)
  int base;     // 1: serial base case, the whole chain is one uncoupled segment
  int level;
  double* Linv;  // (N, packed) out: inverse Cholesky factor of every interior row, packed lower
                 // triangle (row r at r(r+1)/2), block stride n(n+1)/2 rounded up to even
  double* Lsub;  // (N-1, n, n) out: L_{i,i-1} inside segments; coupling copies at segment edges
  double* Sl;    // (K, n, n) out: S_L per segment (written into the next level's diag slots)
  double* Sr;    // (K, n, n) out: S_R per segment
  double* Ssub;  // (K, n, n) out: next level sub block k = -Y_R^T Y_L[last]
  DevErr* err;
};

template <int NT>
struct FactorShape {
  static constexpr int LD = NT + 4;  // +4 doubles: conflict-free DMMA fragment loads
  static constexpr int NTHREADS = NT == 64 ? 256 : NT == 32 ? 128 : NT == 16 ? 64 : 32;
  static constexpr int NW = NTHREADS / 32;
  // warp specialisation: group A (warps [0, NWA)) factors the diagonal block, group B
  // (warps [NWA, NW)) finishes the previous step's Schur/fill updates concurrently.
  static constexpr int NWA = NW >= 2 ? NW / 2 : 1;
  static constexpr int NWB = NW - NWA;
  static constexpr int TS = NT == 8 ? 8 : 16;  // syrk warp tile
  static constexpr int SUB = TS / 8;
  static constexpr int TSR = 2 * NT / TS;
  static constexpr int HALF = TSR / 2;
  static constexpr int NSL = HALF * (HALF + 1) / 2;
  static constexpr int ND = NSL;
  static constexpr int MAXD = (ND + NW - 1) / NW;
  static constexpr int MAXV = (NT * NT / 256 + NWA - 1) / NWA > 0 ? (NT * NT / 256 + NWA - 1) / NWA : 1;
  static constexpr size_t SMEM = (size_t)3 * NT * LD * sizeof(double);
  static constexpr int MINB = NT == 64 ? 2 : NT == 32 ? 4 : NT == 16 ? 8 : 16;  // CTAs per SM (NT = 8: 124 regs, no spills)
  static_assert(NT / 8 == NW, "one trtri leaf per warp");
  static_assert(NWB == 0 || 16 * NWB == NT, "group B owns 16 rows of the fill block per warp");
};

constexpr int kBarA = 1;  // named barrier of group A
constexpr int kBarB = 2;  // named barrier of group B

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void tri_decode(int s, int& r, int& c) {
  r = 0;
  while ((r + 1) * (r + 2) / 2 <= s) ++r;
  c = s - r * (r + 1) / 2;
}

// Inverse of one 8x8 lower-triangular diagonal tile, in place (lanes 0..7: one column each).
// 1/L_ii was stored at DL[i][NT] by the panel factorization.
template <int NT>
__device__ __forceinline__ void leaf_inverse(double* DL, int d0, int lane) {
  constexpr int LD = FactorShape<NT>::LD;
  double x[8];
  if (lane < 8) {
    const int c = lane;
    double ri[8], row[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) ri[i] = DL[(d0 + i) * LD + NT];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = (i == c) ? ri[i] : 0.0;
#pragma unroll
    for (int i = 1; i < 8; ++i) {
#pragma unroll
      for (int mm = 0; mm < i; ++mm) row[mm] = DL[(d0 + i) * LD + d0 + mm];
      double s0 = 0.0, s1 = 0.0;  // x[mm] == 0 for mm < c, so no predicate is needed
#pragma unroll
      for (int mm = 0; mm < i; ++mm) {
        if (mm & 1)
          s1 = fma(row[mm], x[mm], s1);
        else
          s0 = fma(row[mm], x[mm], s0);
      }
      if (i > c) x[i] = -(s0 + s1) * ri[i];
    }
  }
  __syncwarp();
  if (lane < 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i) DL[(d0 + i) * LD + d0 + lane] = x[i];
  }
}

// fp64 reciprocal / reciprocal square root for the pivot chain: the MUFU seed (rcp.approx: 27
// cycles, rsqrt.approx: 74 cycles measured, tools/fp64_mix.cu) refined by two Newton steps, instead
// of the libdevice sequences (rsqrt(double) ~75 + special-case handling, 1.0/x ~80 cycles).
// Inputs are positive normal pivots (a non-positive pivot is reported, its values discarded).
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const double h = x * r;
    const double e = fma(-h, r, 1.0);  // 1 - x r^2
    r = fma(0.5 * r, e, r);
  }
  return r;
}

// One 8-column panel of the Cholesky factorization, factored by a single warp in registers
// (lane l owns panel rows p0+l and, when HASB, p0+l+32).  The pivot chain is latency bound
// (shfl -> rsqrt -> fma per column); it is software-pipelined so that the next column's pivot and
// multipliers are shuffled right after that column's own update, ahead of the other updates.
// Branch-free: a data-dependent `break` costs ~40% of the chain (tools/panel_bench.cu); a failed
// pivot only poisons values that are discarded.  Returns the 1-based failing pivot or 0.
template <int NT, bool HASB, bool RCP = false>
__device__ __forceinline__ int panel_chain(double* DL, int p0, int lane) {
  constexpr int LD = FactorShape<NT>::LD;
  const int ra = p0 + lane, rb = p0 + lane + 32;
  const bool ha = ra < NT, hb = HASB && rb < NT;
  double va[8], vb[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    va[c] = ha ? DL[ra * LD + p0 + c] : 0.0;
    vb[c] = hb ? DL[rb * LD + p0 + c] : 0.0;
  }
  int fail = 0;
  double d = __shfl_sync(0xffffffffu, va[0], 0);
  double lck[8];
#pragma unroll
  for (int c = 1; c < 8; ++c) lck[c] = __shfl_sync(0xffffffffu, va[0], c);
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    double t[8], u[8];
#pragma unroll
    for (int c = kk + 1; c < 8; ++c) {  // multipliers, ready before the pivot root
      t[c] = va[kk] * lck[c];
      if (HASB) u[c] = vb[kk] * lck[c];
    }
    fail = (fail == 0 && d <= 0.0) ? p0 + kk + 1 : fail;
    double rinv, dinv;
    if (RCP) {  // 1/d on the chain (rcp seed + Newton), the root off it
      dinv = rcp_nr(d);
      rinv = rsqrt_nr(d);
    } else {
      rinv = rsqrt(d);
      dinv = rinv * rinv;
    }
    double nd = 0.0, nl[8];
    if (kk + 1 < 8) {
      va[kk + 1] = fma(-t[kk + 1], dinv, va[kk + 1]);
      if (HASB) vb[kk + 1] = fma(-u[kk + 1], dinv, vb[kk + 1]);
      nd = __shfl_sync(0xffffffffu, va[kk + 1], kk + 1);
#pragma unroll
      for (int c = kk + 2; c < 8; ++c) nl[c] = __shfl_sync(0xffffffffu, va[kk + 1], c);
    }
#pragma unroll
    for (int c = kk + 2; c < 8; ++c) {
      va[c] = fma(-t[c], dinv, va[c]);
      if (HASB) vb[c] = fma(-u[c], dinv, vb[c]);
    }
    va[kk] *= rinv;  // row p0+kk: d * rinv = sqrt(d)
    if (HASB) vb[kk] *= rinv;
    if (lane == kk) DL[(p0 + kk) * LD + NT] = rinv;  // 1 / L_kk for the inverse
    d = nd;
#pragma unroll
    for (int c = kk + 2; c < 8; ++c) lck[c] = nl[c];
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (ha) DL[ra * LD + p0 + c] = va[c];
    if (hb) DL[rb * LD + p0 + c] = vb[c];
  }
  return fail;
}

// C fragment read-modify-write (tile (tr, tc) -= acc) as one 16-byte access per lane: half the
// shared-memory wavefronts of two 8-byte accesses on the LD = NT + 4 layout.
template <int LD>
__device__ __forceinline__ void sub_frag(double* DL, int tr, int tc, int lane, const double (&acc)[2]) {
  double2* dst = reinterpret_cast<double2*>(DL + (tr * 8 + (lane >> 2)) * LD + tc * 8 + 2 * (lane & 3));
  double2 v = *dst;
  v.x -= acc[0];
  v.y -= acc[1];
  *dst = v;
}

// rank-8 update of one 8x8 tile (tr, tc) by panel p: A[tr][tc] -= L[tr][p] L[tc][p]^T
template <int NT>
__device__ __forceinline__ void tile_update(double* DL, int tr, int tc, int p0, int lane) {
  constexpr int LD = FactorShape<NT>::LD;
  const double* pa = DL + (tr * 8 + (lane >> 2)) * LD + p0 + (lane & 3);
  const double* pb = DL + (tc * 8 + (lane >> 2)) * LD + p0 + (lane & 3);
  double acc[2] = {0.0, 0.0};
  dmma(acc, pa[0], pb[0]);
  dmma(acc, pa[4], pb[4]);
  sub_frag<LD>(DL, tr, tc, lane, acc);
}

}  // namespace btd
#include "btd_chain.cuh"
namespace btd {

// Rank-8 updates by the panel at column p0 of the lower-triangular tile set
// {(off + tr, off + tc) : 0 <= tc <= tr < m}, units u = first, first + step, ...  Processed in
// batches of B tiles with every fragment load issued before the DMMAs (ILP: one tile's
// LDS -> DMMA -> DMMA -> LDS/STS chain is ~150 cycles).
template <int NT, int B>
__device__ __forceinline__ void tile_update_tri(double* DL, int off, int m, int first, int step, int p0, int lane) {
  constexpr int LD = FactorShape<NT>::LD;
  const int units = m * (m + 1) / 2;
  for (int u0 = first; u0 < units; u0 += B * step) {
    double a0[B], a1[B], b0[B], b1[B];
    int tr[B], tc[B];
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int u = u0 + q * step;
      tri_decode(u < units ? u : 0, tr[q], tc[q]);
      tr[q] += off;
      tc[q] += off;
      const double* pa = DL + (tr[q] * 8 + (lane >> 2)) * LD + p0 + (lane & 3);
      const double* pb = DL + (tc[q] * 8 + (lane >> 2)) * LD + p0 + (lane & 3);
      a0[q] = pa[0];
      a1[q] = pa[4];
      b0[q] = pb[0];
      b1[q] = pb[4];
    }
#pragma unroll
    for (int q = 0; q < B; ++q) {
      if (u0 + q * step >= units) continue;
      double acc[2] = {0.0, 0.0};
      dmma(acc, a0[q], b0[q]);
      dmma(acc, a1[q], b1[q]);
      sub_frag<LD>(DL, tr[q], tc[q], lane, acc);
    }
  }
}


// Recursive doubling on DMMA, run by the NWA warps of group A (named barrier kBarA), turning
// L with inverted 8x8 diagonal tiles into the full inverse Linv, in place:
//   [[A,0],[B,C]]^{-1} = [[Ai,0],[-Ci B Ai, Ci]]   for blocks of 8, 16, 32 rows.
template <int NT, int NWT = FactorShape<NT>::NWA>
__device__ __forceinline__ void trtri_doubling(double* DL, int warp, int lane) {
  using S = FactorShape<NT>;
  constexpr int LD = S::LD;
  constexpr int NWA = NWT;  // warps running the inverse (named barrier kBarA over them)
  constexpr int MAXV = (NT * NT / 256 + NWA - 1) / NWA > 0 ? (NT * NT / 256 + NWA - 1) / NWA : 1;

  // ---- recursive doubling: [[A,0],[B,C]]^{-1} = [[Ai,0],[-Ci B Ai, Ci]] on DMMA ----
#pragma unroll
  for (int b = 8; 2 * b <= NT; b *= 2) {
    const int tpb = b / 8;
    const int units = (NT / (2 * b)) * tpb * tpb;
#pragma unroll
    for (int phase = 0; phase < 2; ++phase) {
      double acc[MAXV][2];
      int i0v[MAXV], trv[MAXV], tcv[MAXV];
      bool ok[MAXV];
#pragma unroll
      for (int q = 0; q < MAXV; ++q) {
        const int u = warp + q * NWA;
        ok[q] = u < units;
        const int pair = u / (tpb * tpb), rem = u % (tpb * tpb);
        i0v[q] = pair * 2 * b;
        trv[q] = rem / tpb;
        tcv[q] = rem % tpb;
        acc[q][0] = acc[q][1] = 0.0;
      }
      for (int k0 = 0; k0 < b; k0 += 4) {
#pragma unroll
        for (int q = 0; q < MAXV; ++q) {
          if (!ok[q]) continue;
          const int i0 = i0v[q];
          if (phase == 0) {  // T = B * Ainv  (Ainv[k][c] == 0 for k < c)
            if (k0 < tcv[q] * 8) continue;
            const double a = DL[(i0 + b + trv[q] * 8 + (lane >> 2)) * LD + i0 + k0 + (lane & 3)];
            const double bb = DL[(i0 + k0 + (lane & 3)) * LD + i0 + tcv[q] * 8 + (lane >> 2)];
            dmma(acc[q], a, bb);
          } else {  // B <- -Cinv * T  (Cinv[r][k] == 0 for k > r)
            if (k0 > trv[q] * 8 + 4) continue;
            const double a = DL[(i0 + b + trv[q] * 8 + (lane >> 2)) * LD + i0 + b + k0 + (lane & 3)];
            const double bb = DL[(i0 + k0 + (lane & 3)) * LD + i0 + b + tcv[q] * 8 + (lane >> 2)];
            dmma(acc[q], a, bb);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < MAXV; ++q) {
        if (!ok[q]) continue;
        const int i0 = i0v[q];
        if (phase == 0) {  // strictly-upper scratch block (rows i0.., cols i0+b..)
          double* dst = DL + (i0 + trv[q] * 8 + (lane >> 2)) * LD + i0 + b + tcv[q] * 8 + 2 * (lane & 3);
          *reinterpret_cast<double2*>(dst) = make_double2(acc[q][0], acc[q][1]);
        } else {
          double* dst = DL + (i0 + b + trv[q] * 8 + (lane >> 2)) * LD + i0 + tcv[q] * 8 + 2 * (lane & 3);
          *reinterpret_cast<double2*>(dst) = make_double2(-acc[q][0], -acc[q][1]);
        }
      }
      named_sync(kBarA, NWA * 32);
    }
  }
}

// ------------------------------------------------------------------------------------------
// In-place Cholesky + triangular inverse of the NT x NT tile DL (lower triangle is read), run by
// the NWA warps of group A (named barrier kBarA).  Returns the 1-based first non-positive pivot
// (reference _first_bad_pivot, bt/kernels.py:136-152; failure test is `pivot <= 0` like the
// LAPACK/OpenBLAS path, so NaN propagates silently), or 0 -- uniform over group A.
//
// Panel-blocked right-looking Cholesky with look-ahead: warp 0 factors panel p (panel_chain)
// while the other warps of the group apply panel p-1's update to the column blocks >= p+1
// (batched DMMA tiles) and invert panel p-1's 8x8 diagonal tile (trtri leaf).  Only the update of
// column block p+1 by panel p sits between two pivot chains.
// INVERSE = true : the full inverse is finished by recursive doubling on DMMA (DL -> Linv).
// INVERSE = false: DL holds L with its 8x8 diagonal tiles replaced by their inverses.
// ------------------------------------------------------------------------------------------
template <int NT, bool INVERSE = true>
__device__ int potrf_trtri(double* DL, int* s_fail, unsigned long long* leaf_bars = nullptr) {
  using S = FactorShape<NT>;
  constexpr int LD = S::LD;
  constexpr int NWA = S::NWA;
  constexpr int NP = NT / 8;
  constexpr int MAXV = S::MAXV;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  BTD_PHASE_INIT();

  for (int p = 0; p < NP; ++p) {
    const int p0 = p * 8;
    if (warp == 0) {
      const int f = (p0 + 32 < NT) ? panel_chain<NT, true, true>(DL, p0, lane)
                                   : panel_chain<NT, false, true>(DL, p0, lane);
      if (lane == 0) *s_fail = f;
      BTD_PHASE(6);
    } else if (p > 0) {
      // helpers: leaf of panel p-1 (warp 1), and panel p-1's update of the column blocks >= p+1
      // (warps 2.. when there are at least two more helpers: the leaf is as long as a few tiles)
      constexpr int T0 = NWA >= 3 ? 2 : 1;
      if (warp == 1) {
        leaf_inverse<NT>(DL, p0 - 8, lane);
        if (leaf_bars) {  // publish leaf p-1 (streaming consumers, btd_factor3.cuh)
          __syncwarp();
          if (lane == 0) {
            __threadfence_block();
            mbar_arrive(&leaf_bars[p - 1]);
          }
        }
      }
      if (warp >= T0) tile_update_tri<NT, 4>(DL, p + 1, NP - p - 1, warp - T0, NWA - T0, p0 - 8, lane);
    }
    named_sync(kBarA, NWA * 32);
    BTD_PHASE(4);
    const int fail = *s_fail;
    if (fail) {
      if (leaf_bars && tid == 0)  // release the consumers of the leaves that will never come
        for (int q = p; q < NP; ++q) mbar_arrive(&leaf_bars[q]);
      return fail;
    }
    // critical: panel p's update of column block p+1 (tiles (tr, p+1), tr >= p+1)
    for (int tr = p + 1 + warp; tr < NP; tr += NWA) tile_update<NT>(DL, tr, p + 1, p0, lane);
    if (NWA == 1 && p + 2 < NP)  // no helpers: the rest of panel p's update runs here
      tile_update_tri<NT, 4>(DL, p + 2, NP - p - 2, 0, 1, p0, lane);
    named_sync(kBarA, NWA * 32);
    BTD_PHASE(5);
  }
  // remaining leaves: the last panel's (and all of them when group A is a single warp)
  for (int lf = (NWA > 1 ? NP - 1 : 0) + warp; lf < NP; lf += NWA) {
    leaf_inverse<NT>(DL, lf * 8, lane);
    if (leaf_bars) {
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        mbar_arrive(&leaf_bars[lf]);
      }
    }
  }
  if constexpr (!INVERSE) {
    if (!leaf_bars) named_sync(kBarA, NWA * 32);
    return 0;
  } else {
  named_sync(kBarA, NWA * 32);
  BTD_PHASE(9);
  trtri_doubling<NT>(DL, warp, lane);
  BTD_PHASE(10);
  return 0;
  }
}

// Pt = Xt * Linv^T, in place on the 16 XP rows owned by this warp (the warp reads only its own rows,
// so it overwrites them after a __syncwarp); both 8-row halves at once, so every Linv^T fragment
// feeds two DMMAs (0.56 fragment loads per DMMA instead of 1.1).
template <int NT>
__device__ __forceinline__ void pt_gemm(double* XP, const double* DL, int row0, int lane) {
  using S = FactorShape<NT>;
  constexpr int LD = S::LD;
  constexpr int NCT = NT / 8;
  const double* pb = DL + (lane >> 2) * LD + (lane & 3);
  double acc[2][NCT][2];
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int c = 0; c < NCT; ++c) acc[rt][c][0] = acc[rt][c][1] = 0.0;
  const double* pa = XP + (row0 + (lane >> 2)) * LD + (lane & 3);
#pragma unroll
  for (int k0 = 0; k0 < NT; k0 += 4) {
    const double a0 = pa[k0], a1 = pa[8 * LD + k0];
#pragma unroll
    for (int ct = 0; ct < NCT; ++ct) {
      if (ct * 8 + 7 < k0) continue;  // Linv[c][k] == 0 for k > c
      const double b = pb[ct * 8 * LD + k0];
      dmma(acc[0][ct], a0, b);
      dmma(acc[1][ct], a1, b);
    }
  }
  __syncwarp();
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int ct = 0; ct < NCT; ++ct)
      *reinterpret_cast<double2*>(XP + (row0 + rt * 8 + (lane >> 2)) * LD + ct * 8 + 2 * (lane & 3)) =
          make_double2(acc[rt][ct][0], acc[rt][ct][1]);
}

// Fill block of the next step:  Gt = -Pt2 * Pt1^T, one 8-row pass of Pt2 rows [row0, row0+8).
// to_global == false: in place over the pass rows (a pass reads only its own Pt2 rows and Pt1);
// to_global == true : last row of the segment, write S_sub = -(Y_L^T Y_R)^T = -Y_R^T Y_L.
template <int NT>
__device__ __forceinline__ void fill_band(double* XP, int row0, int lane, bool to_global, double* ssub, int n) {
  using S = FactorShape<NT>;
  constexpr int LD = S::LD;
  constexpr int NCT = NT / 8;
  const double* pb = XP + (lane >> 2) * LD + (lane & 3);  // Pt1 rows as the col-major B operand
  {
    constexpr int rt = 0;
    double acc[NCT][2];
#pragma unroll
    for (int c = 0; c < NCT; ++c) acc[c][0] = acc[c][1] = 0.0;
    const double* pa = XP + (NT + row0 + rt * 8 + (lane >> 2)) * LD + (lane & 3);
#pragma unroll 4
    for (int k0 = 0; k0 < NT; k0 += 4) {
      const double a0 = pa[k0];
#pragma unroll
      for (int ct = 0; ct < NCT; ++ct) dmma(acc[ct], a0, pb[ct * 8 * LD + k0]);
    }
    __syncwarp();
    const int r = row0 + rt * 8 + (lane >> 2);
#pragma unroll
    for (int ct = 0; ct < NCT; ++ct) {
      const int c = ct * 8 + 2 * (lane & 3);
      if (!to_global) {
        double2 v;
        v.x = -acc[ct][0];
        v.y = -acc[ct][1];
        *reinterpret_cast<double2*>(XP + (NT + r) * LD + c) = v;
      } else if (r < n) {
        if (c < n) ssub[(size_t)c * n + r] = -acc[ct][0];
        if (c + 1 < n) ssub[(size_t)(c + 1) * n + r] = -acc[ct][1];
      }
    }
  }
}

// acc += Pt[R-tile] * Pt[C-tile]^T over k = 0..NT (one TS x TS warp tile of the lower 2NT x 2NT product)
template <int NT>
__device__ __forceinline__ void syrk_tile(const double* XP, int R, int C, double (&acc)[FactorShape<NT>::SUB][FactorShape<NT>::SUB][2],
                                          int lane) {
  using S = FactorShape<NT>;
  constexpr int LD = S::LD, TS = S::TS, SUB = S::SUB;
  const bool diag = (R == C);
  const double* pa = XP + (R * TS + (lane >> 2)) * LD + (lane & 3);
  const double* pb = XP + (C * TS + (lane >> 2)) * LD + (lane & 3);
#pragma unroll 4
  for (int k0 = 0; k0 < NT; k0 += 4) {
    double a[SUB], b[SUB];
#pragma unroll
    for (int i = 0; i < SUB; ++i) {
      a[i] = pa[i * 8 * LD + k0];
      b[i] = pb[i * 8 * LD + k0];
    }
#pragma unroll
    for (int i = 0; i < SUB; ++i)
#pragma unroll
      for (int jj = 0; jj < SUB; ++jj)
        if (!diag || jj <= i) dmma(acc[i][jj], a[i], b[jj]);
  }
}

// S_L += P2^T P2 over the SL tiles owned by warp `w` of a group of `nw` warps; S_L accumulates
// across the segment's steps in its global output slot (L2 resident): keeping it in registers
// would cost 32 registers for the whole kernel.
template <int NT>
__device__ __forceinline__ void sl_update(const double* XP, double* sl, int n, bool first, int w, int nw, int lane) {
  using S = FactorShape<NT>;
  constexpr int TS = S::TS, SUB = S::SUB, HALF = S::HALF, NSL = S::NSL;
  for (int t = w; t < NSL; t += nw) {
    int rr, cc;
    tri_decode(t, rr, cc);
    double acc[SUB][SUB][2];
#pragma unroll
    for (int i = 0; i < SUB; ++i)
#pragma unroll
      for (int jj = 0; jj < SUB; ++jj) {
        const int r = rr * TS + i * 8 + (lane >> 2);
        const int c = cc * TS + jj * 8 + 2 * (lane & 3);
        const double* src = sl + (size_t)r * n + c;
        acc[i][jj][0] = (!first && r < n && c < n) ? src[0] : 0.0;
        acc[i][jj][1] = (!first && r < n && c + 1 < n) ? src[1] : 0.0;
      }
    syrk_tile<NT>(XP, HALF + rr, HALF + cc, acc, lane);
#pragma unroll
    for (int i = 0; i < SUB; ++i)
#pragma unroll
      for (int jj = 0; jj < SUB; ++jj) {
        if (rr == cc && jj > i) continue;
        const int r = rr * TS + i * 8 + (lane >> 2);
        const int c = cc * TS + jj * 8 + 2 * (lane & 3);
        double* dst = sl + (size_t)r * n + c;
        if (r < n && c < n) dst[0] = acc[i][jj][0];
        if (r < n && c + 1 < n) dst[1] = acc[i][jj][1];
      }
  }
}

// Logical warp index of hardware warp `hw` for factor_level_kernel<64> (see there).  Reads
// %warpid: hardware warp slot on the SM, sub-partition = slot % 4.
template <int NW, int NWA>
__device__ __forceinline__ int level_warp_roles(int hw, int lane) {
  __shared__ int s_wid[NW];
  unsigned wid;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  if (lane == 0) s_wid[hw] = (int)wid;
  __syncthreads();
  int lo = s_wid[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) lo = min(lo, s_wid[w]);
  const int sc = (lo / NW) & 1, so = sc ^ 1;  // this CTA's chain sub-partition, the other CTA's
  // order: warps on sc, then on so, then the rest (hardware order within a class); the position
  // in that order is the logical index (group A = the first NWA, the chain = the first)
  auto key = [&](int w) {
    const int sp = s_wid[w] & 3;
    return ((sp == sc ? 0 : sp == so ? 1 : 2) << 8) | w;
  };
  const int mk = key(hw);
  int mine = 0;
#pragma unroll
  for (int v = 0; v < NW; ++v) mine += key(v) < mk;
  return mine;
}

template <int NT>
__global__ void __launch_bounds__(FactorShape<NT>::NTHREADS, FactorShape<NT>::MINB)
    factor_level_kernel(FactorArgs args) {
  using S = FactorShape<NT>;
  constexpr int LD = S::LD, NTHREADS = S::NTHREADS, NW = S::NW, NWA = S::NWA, NWB = S::NWB;
  constexpr int TS = S::TS, SUB = S::SUB, ND = S::ND;
  extern __shared__ __align__(16) double smem[];
  double* XP = smem;                // 2NT x LD : [X1 | Pt1] rows 0..NT-1, [Gt | Pt2] rows NT..2NT-1
  double* DL = smem + 2 * NT * LD;  // NT x LD  : D -> L -> Linv
  __shared__ int s_fail, s_fail_a;

  const int k = args.k0 + blockIdx.x;
  if (cta_superseded(args.err, args.level, 0, k)) return;
  const bool coupled = !args.base;
  const long long start = coupled ? (long long)args.seps[k] + 1 : 0;
  const long long stop = coupled ? (long long)args.seps[k + 1] : args.N;
  const int J = (int)(stop - start);
  const int n = args.n;
  const size_t bs = (size_t)n * n;
  const int tid = threadIdx.x, lane = tid & 31;
  // Logical warp roles by SM sub-partition (NT = 64, two CTAs per SM): the pivot chain (logical
  // warp 0) runs on sub-partition `sc` (0 or 1 by the CTA's warp slots on the SM, so the two
  // resident CTAs' chains sit on different sub-partitions), the rest of group A are this CTA's
  // warps on the two chain sub-partitions, and group B -- the DMMA work that runs concurrently
  // with the chains -- are its warps on the other two.  Every role below is keyed on `warp`.
  const int warp = NT == 64 ? level_warp_roles<NW, NWA>(tid >> 5, lane) : tid >> 5;
  const bool in_a = warp < NWA;
  const int wb = warp - NWA;  // warp index inside group B
  double* sl = args.Sl + (size_t)k * bs;

  // ---- prologue: D_0, X1_0 (A_{1,0} or C_R), Gt_0 = C_L^T ----
  stage_block_async<NT, LD, NTHREADS>(DL, args.diag + start * bs, n);
  if (J > 1)
    stage_block_async<NT, LD, NTHREADS>(XP, args.sub + start * bs, n);
  else if (coupled)
    stage_block_async<NT, LD, NTHREADS>(XP, args.sub + (stop - 1) * bs, n);
  cp_async_commit();
  // Gt_0 = C_L^T and the hierarchy's copies of C_L, C_R: needed only from phase 2 of step 0, so
  // group B does them while the first pivot chain runs (single-warp CTAs: here)
  auto coupling_work = [&](int t, int nt) {
    stage_block_transposed_part<NT, LD>(XP + NT * LD, args.sub + (start - 1) * bs, n, t, nt);
    copy_block_part(args.Lsub + (start - 1) * bs, args.sub + (start - 1) * bs, n, t, nt);  // C_L
    copy_block_part(args.Lsub + (stop - 1) * bs, args.sub + (stop - 1) * bs, n, t, nt);    // C_R
  };
  if (coupled && NWB == 0) coupling_work(tid, NTHREADS);
  cp_async_wait_all();
  for (int r = n + tid; r < NT; r += NTHREADS) DL[r * LD + r] = 1.0;
  __syncthreads();
  BTD_PHASE_INIT();

  for (int j = 0; j < J; ++j) {
    const bool last = (j == J - 1);
    // ================= phase 1: A factors D_j ; B finishes step j-1 =================
    int fail = 0;
    constexpr bool kChain = NT >= 32;
    if constexpr (kChain) {
      // single-warp left-looking pivot chain (btd_chain.cuh), then the inverse by recursive
      // doubling on the whole of group A
      if (in_a) {
        if (warp == 0) {
          const int f = chain_potrf<LD, NT>(DL, lane);
          if (lane == 0) s_fail_a = f;
        }
        named_sync(kBarA, NWA * 32);
        fail = s_fail_a;
        if (!fail) trtri_doubling<NT>(DL, warp, lane);
      }
    } else {
      if (in_a) fail = potrf_trtri<NT>(DL, &s_fail);
    }
    if (NWB == 0) __syncthreads();  // single-warp CTA: group B work runs after the factor
    constexpr int SKIPB = 0;
    if (j == 0 && coupled && NWB > 0 && !in_a) coupling_work((warp - NWA) * 32 + lane, NWB * 32);
    if (j > 0 && (NWB == 0 || (!in_a && wb >= SKIPB))) {
      const int w = NWB ? wb - SKIPB : 0, nw = NWB ? NWB - SKIPB : 1, nb = NWB ? (NWB - SKIPB) * 32 : 32;
      const int gt = NWB ? (warp - NWA - SKIPB) * 32 + lane : tid;
      if (coupled) {
        sl_update<NT>(XP, sl, n, j == 1, w, nw, lane);
        named_sync(kBarB, nb);
        for (int rb = w; rb < NT / 8; rb += nw) fill_band<NT>(XP, rb * 8, lane, false, nullptr, n);
        named_sync(kBarB, nb);
      }
      // L_{j,j-1} (Pt1 of step j-1) -> global, then stage the next X1 over it
      if (n == NT) {  // 16-byte copies, no index division
        double* dst = args.Lsub + (start + j - 1) * bs;
        for (int e = gt; e < NT * NT / 2; e += nb) {
          const int r = e / (NT / 2), c = 2 * (e % (NT / 2));
          *reinterpret_cast<double2*>(dst + r * NT + c) = *reinterpret_cast<const double2*>(XP + r * LD + c);
        }
      } else {
        for (int e = gt; e < n * n; e += nb) args.Lsub[(start + j - 1) * bs + e] = XP[(e / n) * LD + e % n];
      }
      named_sync(kBarB, nb);
      const double* nx = !last ? args.sub + (start + j) * bs : (coupled ? args.sub + (stop - 1) * bs : nullptr);
      if (nx) {
        if ((n & 1) == 0) {
          for (int idx = gt; idx < NT * NT / 2; idx += nb) {
            const int r = idx / (NT / 2), c = (idx % (NT / 2)) * 2;
            const bool ok = r < n && c < n;
            cp_async16(XP + r * LD + c, ok ? (const void*)(nx + (size_t)r * n + c) : (const void*)nx, ok ? 16 : 0);
          }
        } else {
          for (int idx = gt; idx < NT * NT; idx += nb) {
            const int r = idx / NT, c = idx % NT;
            const bool ok = r < n && c < n;
            cp_async8(XP + r * LD + c, ok ? (const void*)(nx + (size_t)r * n + c) : (const void*)nx, ok ? 8 : 0);
          }
        }
        cp_async_commit();
      }
    }
    if (warp == 0 && lane == 0) s_fail = fail;  // logical warp 0 (the chain) is in group A
    __syncthreads();
    BTD_PHASE(1);
    if (s_fail) {
      if (tid == 0 && s_fail <= n) report_npd(args.err, args.level, j, k, s_fail);
      return;
    }
    // ================= phase 2: all warps ==========================================
    store_packed_lower<NT, LD, NTHREADS>(args.Linv + (start + j) * (size_t)packed_offset_(n), DL, n);
    if (last && !coupled) break;
    cp_async_wait_all();
    __syncthreads();
    if (coupled || warp * 16 < NT) pt_gemm<NT>(XP, DL, warp * 16, lane);
    if (!coupled && NW * 16 < NT) pt_gemm<NT>(XP, DL, (warp + NW) * 16, lane);  // single-warp base
    __syncthreads();
    BTD_PHASE(2);
    if (!last) {
      stage_block_async<NT, LD, NTHREADS>(DL, args.diag + (start + j + 1) * bs, n);
      cp_async_commit();
    }
    // D_{j+1} = A_{j+1,j+1} - P1^T P1  (or S_R at the last row of a coupled segment)
    if constexpr (NT == 64) {
      // 36 lower 8x8 tiles balanced over the 8 warps (4-5 each, max 5 DMMAs per k step instead of
      // 8 for the warps that held two 16x16 tiles): warps 2p, 2p+1 share the tile rows 7-p and p,
      // (7-p, 0..7-p) then (p, 0..p), split 5 / 4.
      const int pr = warp >> 1, first = (warp & 1) * 5;
      double dacc[5][2];
      int dtr[5], dtc[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        const int idx = first + i;
        const bool hi = idx <= 7 - pr;
        dtr[i] = idx < 9 ? (hi ? 7 - pr : pr) : -1;
        dtc[i] = hi ? idx : idx - (8 - pr);
        dacc[i][0] = dacc[i][1] = 0.0;
      }
      const double* base = XP + (lane >> 2) * LD + (lane & 3);
      // a warp's tiles lie in at most two tile rows (7 - pr and pr): one A fragment load per row
      // and k step, shared by the tiles of that row (7 instead of 10 fragment loads per k step)
      bool rhi[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) rhi[i] = dtr[i] == 7 - pr;
      const double* pah = base + (7 - pr) * 8 * LD;
      const double* pal = base + pr * 8 * LD;
#pragma unroll 4
      for (int k0 = 0; k0 < NT; k0 += 4) {
        const double ah = pah[k0], al = pal[k0];
#pragma unroll
        for (int i = 0; i < 5; ++i) {
          if (dtr[i] < 0) continue;
          dmma(dacc[i], rhi[i] ? ah : al, base[dtc[i] * 8 * LD + k0]);
        }
      }
      cp_async_wait_all();
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        if (dtr[i] < 0) continue;
        const int r = dtr[i] * 8 + (lane >> 2), c = dtc[i] * 8 + 2 * (lane & 3);
        if (!last) {
          double2* dst = reinterpret_cast<double2*>(DL + r * LD + c);
          double2 v = *dst;
          v.x = (r == c && r >= n) ? 1.0 : v.x - dacc[i][0];
          v.y = (r == c + 1 && r >= n) ? 1.0 : v.y - dacc[i][1];
          *dst = v;
        } else if (r < n) {
          double* dst = args.Sr + (size_t)k * bs + (size_t)r * n;
          if (c < n) dst[c] = dacc[i][0];
          if (c + 1 < n) dst[c + 1] = dacc[i][1];
        }
      }
      __syncthreads();
      BTD_PHASE(3);
      continue;
    }
    double acc[S::MAXD][SUB][SUB][2];
    int drr[S::MAXD], dcc[S::MAXD];
#pragma unroll
    for (int s = 0; s < S::MAXD; ++s) {
      const int dd = warp + s * NW;
      drr[s] = -1;
#pragma unroll
      for (int i = 0; i < SUB; ++i)
#pragma unroll
        for (int jj = 0; jj < SUB; ++jj) acc[s][i][jj][0] = acc[s][i][jj][1] = 0.0;
      if (dd < ND) {
        tri_decode(dd, drr[s], dcc[s]);
        syrk_tile<NT>(XP, drr[s], dcc[s], acc[s], lane);
      }
    }
    cp_async_wait_all();
    __syncthreads();
#pragma unroll
    for (int s = 0; s < S::MAXD; ++s) {
      if (drr[s] < 0) continue;
      const int rr = drr[s], cc = dcc[s];
#pragma unroll
      for (int i = 0; i < SUB; ++i)
#pragma unroll
        for (int jj = 0; jj < SUB; ++jj) {
          if (rr == cc && jj > i) continue;
          const int r = rr * TS + i * 8 + (lane >> 2);
          const int c = cc * TS + jj * 8 + 2 * (lane & 3);
          if (!last) {
            double2* dst = reinterpret_cast<double2*>(DL + r * LD + c);
            double2 v = *dst;
            v.x = (r == c && r >= n) ? 1.0 : v.x - acc[s][i][jj][0];
            v.y = (r == c + 1 && r >= n) ? 1.0 : v.y - acc[s][i][jj][1];
            *dst = v;
          } else if (r < n) {
            double* dst = args.Sr + (size_t)k * bs + (size_t)r * n;
            if (c < n) dst[c] = acc[s][i][jj][0];
            if (c + 1 < n) dst[c + 1] = acc[s][i][jj][1];
          }
        }
    }
    __syncthreads();
    BTD_PHASE(3);
  }

  if (coupled) {  // the last row's S_L update and S_sub = -Y_R^T Y_L[last]
    sl_update<NT>(XP, sl, n, J == 1, warp, NW, lane);
    for (int rb = warp; rb < NT / 8; rb += NW)
      fill_band<NT>(XP, rb * 8, lane, true, args.Ssub + (size_t)k * bs, n);
  }
}

// Next-level diagonal: S_diag[p] = (A[s_p] - S_L[p]) - S_R[p-1]  (reference order, bt/schur.py:186-188).
// S_L[p] already sits in next_diag[p]; only the lower triangle is formed (the kernels never read
// the upper triangle of a diagonal block).
__global__ void assemble_schur_diag_kernel(const double* diag, const int* seps, double* next_diag,
                                           const double* Sr, int K, int n, const DevErr* err) {
  if (error_raised(err)) return;
  // flattened grid-stride over P blocks x n^2 elements (a CTA per separator wastes most threads
  // at small n: 116510 separators x 64 elements at n = 8)
  const size_t bs = (size_t)n * n;
  const size_t total = (size_t)(K + 1) * bs;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int p = (int)(e / bs);
    const int i = (int)(e % bs);
    const int r = i / n, c = i % n;
    if (c > r) continue;
    double v = diag[(size_t)seps[p] * bs + i];
    if (p < K) v -= next_diag[e];
    if (p > 0) v -= Sr[e - bs];
    next_diag[e] = v;
  }
}

// The same for even n, a warp per block row: 16-byte accesses over the row's lower part (columns
// 0..r, plus the pair partner of column r, which lands in the never-read upper triangle), no
// per-element index division.
__global__ void assemble_schur_diag_rows_kernel(const double* diag, const int* seps, double* next_diag,
                                                const double* Sr, int K, int n, const DevErr* err) {
  if (error_raised(err)) return;
  const long long rows = (long long)(K + 1) * n;
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const size_t bs = (size_t)n * n;
  for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < rows; w += nw) {
    const int p = (int)(w / n), r = (int)(w % n);
    const double* a = diag + (size_t)seps[p] * bs + (size_t)r * n;
    double* o = next_diag + (size_t)p * bs + (size_t)r * n;
    const double* sr = Sr + ((size_t)p - 1) * bs + (size_t)r * n;
    for (int c = 2 * lane; c <= r; c += 64) {
      double2 v = *reinterpret_cast<const double2*>(a + c);
      if (p < K) {
        const double2 t = *reinterpret_cast<const double2*>(o + c);
        v.x -= t.x;
        v.y -= t.y;
      }
      if (p > 0) {
        const double2 t = *reinterpret_cast<const double2*>(sr + c);
        v.x -= t.x;
        v.y -= t.y;
      }
      *reinterpret_cast<double2*>(o + c) = v;
    }
  }
}

// Upper triangle of every n x n block := its lower triangle (debug export of Schur diagonals).
__global__ void mirror_lower_kernel(double* blocks, long long P, int n) {
  const size_t bs = (size_t)n * n, total = (size_t)P * bs;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const size_t b = e / bs;
    const int i = (int)(e % bs), r = i / n, c = i % n;
    if (c > r) blocks[e] = blocks[b * bs + (size_t)c * n + r];
  }
}

__global__ void fill_separators_kernel(int* seps, int P, int N, int step) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < P) seps[k] = (k == P - 1) ? N - 1 : k * step;
}

__global__ void init_err_kernel(DevErr* err) {
  err->key = kNoErr;
  err->level = 0x7fffffff;
  err->pad = 0;
}

}  // namespace btd
