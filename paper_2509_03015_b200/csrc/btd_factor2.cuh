// Paired-segment level elimination for 32 < n <= 64: one CTA interleaves TWO segments so that the
// latency-bound Cholesky of one segment's diagonal block runs while the DMMA work of the other
// segment's previous step fills the fp64 pipe.
//
// Same algebra as factor_level_kernel (btd_factor.cuh, "Y-form", reference chain
// permute_split / factorize_btd_batch / solve_btd_batch(F) / compute_schur, bt/schur.py:98-193,
// bt/block_cholesky.py:24-68), different schedule.  Per step j of a segment:
//   potrf  (group A, 4 warps):  D_j -> L_j -> Linv_j (potrf_trtri), Linv_j -> HBM (packed)
//   gemm   (group B, 8 warps):  Pt = [X1; Gt] Linv_j^T ; S_L += Pt2 Pt2^T ; D_{j+1} = A - Pt1 Pt1^T ;
//                               Gt_{j+1} = -Pt2 Pt1^T ; L_{j+1,j} = Pt1 -> HBM ; stage the next X1
// and the two segments (slots) alternate:  phase t:  A: potrf(slot t%2, step t/2)
//                                                     B: gemm (slot (t+1)%2, step (t-1)/2)
// so every phase costs max(potrf, gemm) instead of potrf + gemm.  The per-step dependency
// potrf(j) -> gemm(j) -> potrf(j+1) of one segment is preserved by the phase barrier.
//
// Shared memory: two slots of [XP (2NT x LD) | DL (NT x LD)] = 209 KB at NT = 64 (1 CTA / SM).
#pragma once

#include "btd_factor.cuh"

namespace btd {

template <int NT>
struct PairShape {
  using S = FactorShape<NT>;
  static constexpr int LD = S::LD;
  static constexpr int NWA = S::NWA;  // potrf group (potrf_trtri is written for S::NWA warps)
  static constexpr int NWB = NT / 8;  // gemm group: one 16-row band of the 2NT-row XP per warp
  static constexpr int NW = NWA + NWB;
  static constexpr int NTHREADS = 32 * NW;
  static constexpr int NB = 32 * NWB;
  static constexpr size_t SLOT = (size_t)3 * NT * LD;  // doubles
  static constexpr size_t SMEM = 2 * SLOT * sizeof(double);
  static constexpr int NUNITS = S::ND + S::NSL;  // D-update tiles + S_L tiles
  static constexpr int MAXQ = (NUNITS + NWB - 1) / NWB;
  static_assert(2 * NT / 16 == NWB, "pt_gemm: 16 rows per gemm warp");
  static_assert(NT / 8 == NWB, "fill_band: 8 rows per gemm warp");
};

// cp.async staging of an n x n row-major block into an NT x LD tile by `nb` threads (index gt).
template <int NT, int LD>
__device__ __forceinline__ void stage_block_async_part(double* sm, const double* g, int n, int gt, int nb) {
  if ((n & 1) == 0) {
    for (int idx = gt; idx < NT * (NT / 2); idx += nb) {
      const int r = idx / (NT / 2), c = (idx % (NT / 2)) * 2;
      const bool ok = r < n && c < n;
      cp_async16(sm + r * LD + c, ok ? (const void*)(g + (size_t)r * n + c) : (const void*)g, ok ? 16 : 0);
    }
  } else {
    for (int idx = gt; idx < NT * NT; idx += nb) {
      const int r = idx / NT, c = idx % NT;
      const bool ok = r < n && c < n;
      cp_async8(sm + r * LD + c, ok ? (const void*)(g + (size_t)r * n + c) : (const void*)g, ok ? 8 : 0);
    }
  }
}

// S_L tile t (16x16 tile of the lower triangle) += Pt2 Pt2^T, read-modify-write in its global
// (L2-resident) slot; `first` starts from zero.
template <int NT>
__device__ __forceinline__ void sl_tile(const double* XP, double* sl, int n, bool first, int t, int lane) {
  using S = FactorShape<NT>;
  constexpr int TS = S::TS, SUB = S::SUB, HALF = S::HALF;
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

// Group B: the DMMA work of step j of one segment (XP/DL of its slot).  wb = warp index in group B,
// gt = thread index in group B.
template <int NT>
__device__ __forceinline__ void pair_gemm(const FactorArgs& a, double* XP, double* DL, long long start, long long stop,
                                          int j, int k, int wb, int gt, int lane) {
  using S = FactorShape<NT>;
  using P = PairShape<NT>;
  constexpr int LD = S::LD, TS = S::TS, SUB = S::SUB, ND = S::ND, NB = P::NB, MAXQ = P::MAXQ;
  const int n = a.n;
  const size_t bs = (size_t)n * n;
  const int J = (int)(stop - start);
  const bool last = (j == J - 1);

  cp_async_wait_all();  // this thread's X1 staging (issued two phases ago)
  named_sync(kBarB, NB);
  pt_gemm<NT>(XP, DL, wb * 16, lane);  // Pt = [X1; Gt] Linv^T, in place
  named_sync(kBarB, NB);
  if (!last) {  // DL is free (Linv_j is in HBM): stage A_{j+1,j+1} under the Schur products
    stage_block_async_part<NT, LD>(DL, a.diag + (start + j + 1) * bs, n, gt, NB);
    cp_async_commit();
  }
  // D_{j+1} tiles (kept in registers) and S_L tiles (read-modify-write), interleaved over the warps
  double acc[2][SUB][SUB][2];
  int drr[2], dcc[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    drr[q] = -1;
#pragma unroll
    for (int i = 0; i < SUB; ++i)
#pragma unroll
      for (int jj = 0; jj < SUB; ++jj) acc[q][i][jj][0] = acc[q][i][jj][1] = 0.0;
  }
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) {
    const int u = wb + q * P::NWB;
    if (u < ND) {
      if (q < 2) {
        tri_decode(u, drr[q], dcc[q]);
        syrk_tile<NT>(XP, drr[q], dcc[q], acc[q], lane);
      }
    } else if (u < P::NUNITS) {
      sl_tile<NT>(XP, a.Sl + (size_t)k * bs, n, j == 0, u - ND, lane);
    }
  }
  named_sync(kBarB, NB);  // S_L has read Pt2: the fill may overwrite it
  fill_band<NT>(XP, wb * 8, lane, last, a.Ssub + (size_t)k * bs, n);
  cp_async_wait_all();
  named_sync(kBarB, NB);  // A_{j+1,j+1} landed; the fill has read Pt1
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    if (drr[q] < 0) continue;
    const int rr = drr[q], cc = dcc[q];
#pragma unroll
    for (int i = 0; i < SUB; ++i)
#pragma unroll
      for (int jj = 0; jj < SUB; ++jj) {
        if (rr == cc && jj > i) continue;
        const int r = rr * TS + i * 8 + (lane >> 2);
        const int c = cc * TS + jj * 8 + 2 * (lane & 3);
        if (!last) {
          double* dst = DL + r * LD + c;
          dst[0] = (r == c && r >= n) ? 1.0 : dst[0] - acc[q][i][jj][0];
          dst[1] = (r == c + 1 && r >= n) ? 1.0 : dst[1] - acc[q][i][jj][1];
        } else if (r < n) {
          double* dst = a.Sr + (size_t)k * bs + (size_t)r * n;
          if (c < n) dst[c] = acc[q][i][jj][0];
          if (c + 1 < n) dst[c + 1] = acc[q][i][jj][1];
        }
      }
  }
  if (last) return;
  // L_{j+1,j} = Pt1 -> hierarchy, then the next X1 (A_{j+2,j+1}, or C_R for the last row) over it
  if ((n & 1) == 0) {
    const int cpr = n / 2;
    for (int e = gt; e < n * cpr; e += NB) {
      const int r = e / cpr, c = (e % cpr) * 2;
      *reinterpret_cast<double2*>(a.Lsub + (start + j) * bs + (size_t)r * n + c) =
          *reinterpret_cast<const double2*>(XP + r * LD + c);
    }
  } else {
    for (int e = gt; e < n * n; e += NB) a.Lsub[(start + j) * bs + e] = XP[(e / n) * LD + e % n];
  }
  named_sync(kBarB, NB);
  const double* nx = (j + 1 < J - 1) ? a.sub + (start + j + 1) * bs : a.sub + (stop - 1) * bs;
  stage_block_async_part<NT, LD>(XP, nx, n, gt, NB);
  cp_async_commit();
}

template <int NT>
__global__ void __launch_bounds__(PairShape<NT>::NTHREADS, 1) factor_pair_kernel(FactorArgs args) {
  using S = FactorShape<NT>;
  using P = PairShape<NT>;
  constexpr int LD = S::LD, NTHREADS = P::NTHREADS, NWA = P::NWA;
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_fail_a;  // potrf_trtri's group-internal flag
  __shared__ int s_fail;    // phase result: failing pivot
  __shared__ int s_fail_j, s_fail_k;

  if (npd_superseded(args.err, args.level, 0, 2 * blockIdx.x)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool in_a = warp < NWA;
  const int n = args.n;
  const size_t bs = (size_t)n * n;
  const int pk = packed_offset_(n);

  long long start[2], stop[2];
  int J[2], kseg[2];
  double* XPs[2];
  double* DLs[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    kseg[s] = 2 * blockIdx.x + s;
    const bool ok = kseg[s] < args.K;
    start[s] = ok ? (long long)args.seps[kseg[s]] + 1 : 0;
    stop[s] = ok ? (long long)args.seps[kseg[s] + 1] : 0;
    J[s] = (int)(stop[s] - start[s]);
    XPs[s] = smem + s * P::SLOT;
    DLs[s] = XPs[s] + 2 * NT * LD;
  }

  // ---- prologue (all threads): D_0, X1_0 (A_{1,0} or C_R), Gt_0 = C_L^T, coupling copies ----
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    if (J[s] <= 0) continue;
    stage_block_async_part<NT, LD>(DLs[s], args.diag + start[s] * bs, n, tid, NTHREADS);
    const double* x1 = J[s] > 1 ? args.sub + start[s] * bs : args.sub + (stop[s] - 1) * bs;
    stage_block_async_part<NT, LD>(XPs[s], x1, n, tid, NTHREADS);
    cp_async_commit();
    stage_block_transposed<NT, LD, NTHREADS>(XPs[s] + NT * LD, args.sub + (start[s] - 1) * bs, n);
    copy_block<NTHREADS>(args.Lsub + (start[s] - 1) * bs, args.sub + (start[s] - 1) * bs, n);  // C_L
    copy_block<NTHREADS>(args.Lsub + (stop[s] - 1) * bs, args.sub + (stop[s] - 1) * bs, n);    // C_R
  }
  cp_async_wait_all();
  if (tid == 0) s_fail = 0;
#pragma unroll
  for (int s = 0; s < 2; ++s)
    for (int r = n + tid; r < NT; r += NTHREADS) DLs[s][r * LD + r] = 1.0;
  __syncthreads();

  const int jmax = J[0] > J[1] ? J[0] : J[1];
  const int phases = 2 * jmax + 1;
  for (int t = 0; t < phases; ++t) {
#ifdef BTD_PHASE_PROF
    const long long ph0 = clock64();
#endif
    // (runtime slot selects written as ternaries: no local-memory arrays)
    if (in_a) {
      const bool s1 = t & 1;
      const int j = t >> 1;
      if (j < (s1 ? J[1] : J[0])) {
        double* DL = s1 ? DLs[1] : DLs[0];
        const int fail = potrf_trtri<NT>(DL, &s_fail_a);
        if (fail) {
          if (tid == 0) {
            s_fail = fail;
            s_fail_j = j;
            s_fail_k = s1 ? kseg[1] : kseg[0];
          }
        } else {
          store_packed_lower<NT, LD, 32 * NWA>(args.Linv + ((s1 ? start[1] : start[0]) + j) * (size_t)pk, DL, n);
        }
      }
    } else if (t >= 1) {
      const bool s1 = !(t & 1);
      const int j = (t - 1) >> 1;
      if (j < (s1 ? J[1] : J[0]))
        pair_gemm<NT>(args, s1 ? XPs[1] : XPs[0], s1 ? DLs[1] : DLs[0], s1 ? start[1] : start[0],
                      s1 ? stop[1] : stop[0], j, s1 ? kseg[1] : kseg[0], warp - NWA, tid - 32 * NWA, lane);
    }
#ifdef BTD_PHASE_PROF
    if (blockIdx.x == 0 && (tid == 0 || tid == 32 * NWA)) atomicAdd(&g_phase_cycles[tid == 0 ? 11 : 12], (unsigned long long)(clock64() - ph0));
#endif
    if (tid == 0 && s_fail == 0 && (t & 1)) {  // another segment's failure makes the rest moot
      bool moot = true;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int jn = (t + 1 - s) >> 1;  // next potrf step of slot s
        if (jn < J[s] && !npd_superseded(args.err, args.level, jn, kseg[s])) moot = false;
      }
      if (moot) s_fail = -1;
    }
    __syncthreads();
#ifdef BTD_PHASE_PROF
    if (blockIdx.x == 0 && tid == 0) atomicAdd(&g_phase_cycles[13], (unsigned long long)(clock64() - ph0));
#endif
    if (s_fail) {
      if (tid == 0 && s_fail > 0 && s_fail <= n) report_npd(args.err, args.level, s_fail_j, s_fail_k, s_fail);
      return;
    }
  }
}

}  // namespace btd
