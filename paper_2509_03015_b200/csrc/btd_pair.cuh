// Pair-slot level elimination for 32 < n <= 64 on wide levels (the level-0 kernel of BASELINE
// config 2): one persistent 16-warp CTA per SM keeps TWO segments ("slots") in flight and
// ping-pongs them, so the latency-bound pivot chain of one slot runs while the DMMA-bound rest of
// the other slot's step runs -- on different SM sub-partitions.
//
// Same Y-form algebra as factor_level_kernel / factor_stream_kernel (the reference chain
// permute_split / factorize_btd_batch / solve_btd_batch(F) / compute_schur, bt/schur.py:98-193,
// bt/block_cholesky.py:24-68), same outputs (packed Linv, L_sub, S_L, S_R, S_sub).
//
// Warp roles by SM sub-partition (warp w runs on SMSP w % 4):
//   warp 0            chain  : Cholesky of D_j of the chain slot, one warp, left-looking
//                              (chain_potrf64: L with inverted 8x8 diagonal tiles)
//   warps 4, 8, 12    helpers: staging of the chain slot (D_0 and C_L^T of a new segment, the next
//                              X1 = A_{j+1,j} / C_R), L2 prefetch of A_{j+1,j+1}; no fp64 work
//   the other 12      bulk   : everything else of the bulk slot's step j, on SMSPs 1-3 only, so
//                              the DMMA stream never delays the pivot chain:
//     (a) blocked triangular solve [X1; Gt; I] L_j^{-T} in registers (24 8-row tiles, 2 per warp):
//         Pt1 = L_{j+1,j} (-> smem + L_sub), Pt2 = Y_L[j]^T (-> smem), Pt3 = Linv_j^T (-> packed)
//     (b) 36 units: D_{j+1} = A_{j+1,j+1} - Pt1 Pt1^T (-> DL, or S_R at the last row),
//         S_L += Pt2 Pt2^T (global, L2 resident), Gt_{j+1} = -Pt2 Pt1^T (or S_sub at the last row)
// Phase t: slot t % 2 is the chain slot, the other the bulk slot; __syncthreads ends a phase.
#pragma once

#include "btd_factor3.cuh"

namespace btd {

struct PairShape {
  static constexpr int NT = 64, LD = 68;
  static constexpr int NW = 16, NTHREADS = 32 * NW;
  static constexpr int NBULK = 12;
  static constexpr int SLOT = 3 * NT * LD;  // DL (NT x LD) + XP (2 NT x LD) doubles per slot
  static constexpr size_t SMEM = (size_t)2 * SLOT * sizeof(double);
};

constexpr int kBarBulk = 4;   // the 12 bulk warps
constexpr int kBarStage = 5;  // chain warp + helpers: a new segment's blocks have landed

// TRSM tile assignment, two 8-row tiles per bulk warp, balanced per sub-partition (DMMA counts:
// X / G band 72, identity band b: 72, 56, 42, 30, 20, 12, 6, 2).  Encoding: type * 8 + band,
// type 0 = X (Pt1), 1 = G (Pt2), 2 = Y (identity -> Linv^T).  Indexed by bulk warp bi (SMSP bi%3+1).
__device__ __constant__ const unsigned char kTrsmTiles[12][2] = {
    {8 + 0, 8 + 1}, {8 + 2, 8 + 3}, {8 + 4, 8 + 5},        // SMSP 1, 2, 3
    {0 + 7, 16 + 0}, {0 + 6, 16 + 1}, {8 + 6, 8 + 7},      // SMSP 1, 2, 3
    {0 + 0, 16 + 7}, {0 + 1, 16 + 6}, {0 + 5, 16 + 2},     // SMSP 1, 2, 3
    {0 + 3, 16 + 4}, {0 + 4, 16 + 3}, {0 + 2, 16 + 5}};    // SMSP 1, 2, 3

__device__ __forceinline__ int pair_bulk_index(int warp) { return warp - warp / 4 - 1; }  // warp % 4 != 0

// one 8-row tile of the triangular solve: state + activity
struct TrsmTile {
  double v[8][2];
  int type, band;
};

__device__ __forceinline__ void trsm_tile_load(TrsmTile& t, const double* XP, int lane) {
  const int r = 8 * t.band + (lane >> 2);
  if (t.type == 2) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int col = c * 8 + 2 * (lane & 3);
      t.v[c][0] = (col == r) ? 1.0 : 0.0;
      t.v[c][1] = (col + 1 == r) ? 1.0 : 0.0;
    }
  } else {
    const double* src = XP + (t.type * 64 + r) * PairShape::LD + 2 * (lane & 3);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double2 x = *reinterpret_cast<const double2*>(src + c * 8);
      t.v[c][0] = x.x;
      t.v[c][1] = x.y;
    }
  }
}

// [T0; T1] <- [T0; T1] L^{-T} (L in DL with inverted diagonal tiles), column block by column block
__device__ __forceinline__ void trsm_two_tiles(TrsmTile& t0, TrsmTile& t1, const double* DL, int lane) {
  constexpr int LD = PairShape::LD;
  const int f0 = t0.type == 2 ? t0.band : 0, f1 = t1.type == 2 ? t1.band : 0;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const double* lp = DL + (8 * p + (lane >> 2)) * LD + 8 * p + (lane & 3);
    const double lb0 = lp[0], lb1 = lp[4];  // B = Linv_pp^T
    const bool a0 = p >= f0, a1 = p >= f1;
    double n00 = 0.0, n01 = 0.0, n10 = 0.0, n11 = 0.0;
    if (a0) {
      double x0, x1, acc[2] = {0.0, 0.0};
      c2a(t0.v[p][0], t0.v[p][1], lane, x0, x1);
      dmma(acc, x0, lb0);
      dmma(acc, x1, lb1);
      t0.v[p][0] = acc[0];
      t0.v[p][1] = acc[1];
      c2a(-acc[0], -acc[1], lane, n00, n01);
    }
    if (a1) {
      double x0, x1, acc[2] = {0.0, 0.0};
      c2a(t1.v[p][0], t1.v[p][1], lane, x0, x1);
      dmma(acc, x0, lb0);
      dmma(acc, x1, lb1);
      t1.v[p][0] = acc[0];
      t1.v[p][1] = acc[1];
      c2a(-acc[0], -acc[1], lane, n10, n11);
    }
#pragma unroll
    for (int c = p + 1; c < 8; ++c) {  // B = L_cp^T
      const double* q = DL + (8 * c + (lane >> 2)) * LD + 8 * p + (lane & 3);
      const double b0 = q[0], b1 = q[4];
      if (a0) {
        dmma(t0.v[c], n00, b0);
        dmma(t0.v[c], n01, b1);
      }
      if (a1) {
        dmma(t1.v[c], n10, b0);
        dmma(t1.v[c], n11, b1);
      }
    }
  }
}

// results: Pt1 -> XP lo (+ L_sub unless last), Pt2 -> XP hi, Pt3 = Linv^T -> packed Linv
__device__ __forceinline__ void trsm_tile_store(const TrsmTile& t, double* XP, double* lsub, double* linv, int n,
                                                int lane) {
  constexpr int LD = PairShape::LD;
  const int r = 8 * t.band + (lane >> 2);
  if (t.type < 2) {
    double* dst = XP + (t.type * 64 + r) * LD + 2 * (lane & 3);
#pragma unroll
    for (int c = 0; c < 8; ++c) *reinterpret_cast<double2*>(dst + c * 8) = make_double2(t.v[c][0], t.v[c][1]);
    if (t.type == 0 && lsub && r < n) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int col = c * 8 + 2 * (lane & 3);
        if ((n & 1) == 0) {
          if (col < n) *reinterpret_cast<double2*>(lsub + (size_t)r * n + col) = make_double2(t.v[c][0], t.v[c][1]);
        } else {
          if (col < n) lsub[(size_t)r * n + col] = t.v[c][0];
          if (col + 1 < n) lsub[(size_t)r * n + col + 1] = t.v[c][1];
        }
      }
    }
  } else {  // Pt3[r][col] = Linv[col][r]: packed row col holds columns 0..col (+ a zero pad for even col)
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = c * 8 + 2 * (lane & 3) + h;
        const int len = ((col + 2) >> 1) << 1;
        if (col < n && r < len) linv[packed_offset_(col) + r] = (r <= col) ? t.v[c][h] : 0.0;
      }
  }
}

// acc(16 x 16 lower-triangle tile (rr, cc) of X X^T) over k = 0..64, X = XP rows [R0 + 16 rr ...]
__device__ __forceinline__ void pair_syrk16(const double* XP, int R, int C, double (&acc)[2][2][2], int lane) {
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
  syrk_tile<64>(XP, R, C, acc, lane);
}

struct PairSlot {
  int k;           // segment (-1: none)
  int j, J;        // next step, segment length
  long long start, stop;
  int iter;        // segments taken by this slot so far
  bool fresh;      // segment not started: its chain phase stages D_0 / C_L^T first
  bool has_chain;  // a successful chain result waits for this slot's bulk phase
};

__global__ void __launch_bounds__(PairShape::NTHREADS, 1) factor_pair_kernel(FactorArgs args) {
  using PS = PairShape;
  constexpr int NT = PS::NT, LD = PS::LD;
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_fail[2];
  __shared__ int s_skip;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int role = (warp & 3) ? 2 : (warp == 0 ? 0 : 1);  // 0 chain, 1 helper, 2 bulk
  const int n = args.n;
  const size_t bs = (size_t)n * n;
  const int pk = packed_offset_(n);
  const int kend = args.kend ? args.kend : args.K;
  const int G = gridDim.x;

  PairSlot slot[2];
  for (int s = 0; s < 2; ++s) {
    slot[s].k = -1;
    slot[s].iter = 0;
    slot[s].fresh = false;
    slot[s].has_chain = false;
  }
  // next segment of slot s: k0 + blockIdx.x + (2 i + s) G
  auto take = [&](int s) -> bool {
    const long long kk = (long long)args.k0 + blockIdx.x + (long long)(2 * slot[s].iter + s) * G;
    slot[s].iter++;
    if (kk >= kend) {
      slot[s].k = -1;
      return false;
    }
    slot[s].k = (int)kk;
    slot[s].start = (long long)args.seps[kk] + 1;
    slot[s].stop = (long long)args.seps[kk + 1];
    slot[s].J = (int)(slot[s].stop - slot[s].start);
    slot[s].j = 0;
    slot[s].fresh = true;
    slot[s].has_chain = false;
    return true;
  };
  bool more[2] = {true, true};
  for (int t = 0;; ++t) {
    const int cs = t & 1, bsl = cs ^ 1;
    // ---- uniform bookkeeping: the chain slot takes a new segment when it has none ----
    if (slot[cs].k < 0 && more[cs] && !slot[cs].has_chain) {
      while (true) {
        if (!take(cs)) {
          more[cs] = false;
          break;
        }
        // a failure recorded at an earlier (step, member) makes this segment irrelevant
        if (tid == 0) s_skip = npd_superseded(args.err, args.level, 0, slot[cs].k) ? 1 : 0;
        __syncthreads();
        const int skip = s_skip;
        __syncthreads();
        if (!skip) break;
      }
    }
    const bool chain_on = slot[cs].k >= 0 && !slot[cs].has_chain;
    const bool bulk_on = slot[bsl].k >= 0 && slot[bsl].has_chain;
    if (!chain_on && !bulk_on && !more[0] && !more[1] && slot[0].k < 0 && slot[1].k < 0) break;

    double* cDL = smem + cs * PS::SLOT;
    double* cXP = cDL + NT * LD;
    double* bDL = smem + bsl * PS::SLOT;
    double* bXP = bDL + NT * LD;

    if (role == 0 || role == 1) {
      // ================= chain slot =================
      if (chain_on) {
        PairSlot& S = slot[cs];
        const bool last = S.j == S.J - 1;
        const int hidx = role == 1 ? ((warp / 4 - 1) * 32 + lane) : 0;  // helper thread 0..95
        if (S.fresh) {
          if (role == 1) {
            stage_block_async_part<NT, LD>(cDL, args.diag + S.start * bs, n, hidx, 96);
            cp_async_commit();
            // Gt_0 = C_L^T (XP hi), and the hierarchy's copies of both coupling blocks
            const double* cl = args.sub + (S.start - 1) * bs;
            for (int idx = hidx; idx < NT * NT; idx += 96) {
              const int c = idx / NT, r = idx % NT;
              cXP[(NT + r) * LD + c] = (r < n && c < n) ? cl[(size_t)c * n + r] : 0.0;
            }
            for (int e = hidx; e < n * n; e += 96) {
              args.Lsub[(S.start - 1) * bs + e] = cl[e];
              args.Lsub[(S.stop - 1) * bs + e] = args.sub[(S.stop - 1) * bs + e];
            }
            cp_async_wait_all();
            for (int r = n + hidx; r < NT; r += 96) cDL[r * LD + r] = 1.0;
          }
          named_sync(kBarStage, 128);
        }
        if (role == 0) {
          const int fail = chain_potrf64<LD, NT>(cDL, lane);
          if (lane == 0) {
            s_fail[cs] = fail;
            if (fail && fail <= n) report_npd(args.err, args.level, S.j, S.k, fail);
          }
        } else {
          // X1 of this step (A_{j+1,j}, or C_R at the last row) -> XP lo for the bulk phase
          const double* x1 = !last ? args.sub + (S.start + S.j) * bs : args.sub + (S.stop - 1) * bs;
          stage_block_async_part<NT, LD>(cXP, x1, n, hidx, 96);
          cp_async_commit();
          if (!last && hidx == 0) prefetch_l2(args.diag + (S.start + S.j + 1) * bs, (unsigned)(bs * sizeof(double)));
          cp_async_wait_all();
        }
      }
    } else if (bulk_on) {
      // ================= bulk slot =================
      PairSlot& S = slot[bsl];
      const bool last = S.j == S.J - 1;
      const int bi = pair_bulk_index(warp);
      double* sl = args.Sl + (size_t)S.k * bs;
      // (a) triangular solve of the two owned tiles
      {
        TrsmTile t0, t1;
        t0.type = kTrsmTiles[bi][0] >> 3;
        t0.band = kTrsmTiles[bi][0] & 7;
        t1.type = kTrsmTiles[bi][1] >> 3;
        t1.band = kTrsmTiles[bi][1] & 7;
        trsm_tile_load(t0, bXP, lane);
        trsm_tile_load(t1, bXP, lane);
        trsm_two_tiles(t0, t1, bDL, lane);
        double* lsub = last ? nullptr : args.Lsub + (S.start + S.j) * bs;
        double* linv = args.Linv + (S.start + S.j) * (size_t)pk;
        trsm_tile_store(t0, bXP, lsub, linv, n, lane);
        trsm_tile_store(t1, bXP, lsub, linv, n, lane);
      }
      named_sync(kBarBulk, 32 * PS::NBULK);
      // (b) units bi + 24 (Gt), bi + 12, bi: 0..9 D 16x16 tiles, 10..19 S_L tiles, 20..35 Gt halves
      // Gt results wait in registers for the barrier: unit bi + 24 always, bi + 12 when bi >= 8
      double gacc[2][4][2];
      bool gheld[2] = {false, false};
#pragma unroll
      for (int q = 2; q >= 0; --q) {
        const int u = bi + 12 * q;
        if (u >= 20) {  // Gt half-band: rows 8g.., columns 32h..32h+31 of -Pt2 Pt1^T
          const int g = (u - 20) >> 1, h = (u - 20) & 1;
          double acc[4][2];
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[c][0] = acc[c][1] = 0.0;
          const double* pa = bXP + (NT + 8 * g + (lane >> 2)) * LD + (lane & 3);
          const double* pb = bXP + (32 * h + (lane >> 2)) * LD + (lane & 3);
#pragma unroll 4
          for (int k0 = 0; k0 < NT; k0 += 4) {
            const double a = pa[k0];
#pragma unroll
            for (int c = 0; c < 4; ++c) dmma(acc[c], a, pb[c * 8 * LD + k0]);
          }
          if (last) {  // S_sub = -(Pt2 Pt1^T)^T = -Y_R^T Y_L[last]
            const int r = 8 * g + (lane >> 2);
            double* ss = args.Ssub + (size_t)S.k * bs;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int col = 32 * h + c * 8 + 2 * (lane & 3);
              if (r < n) {
                if (col < n) ss[(size_t)col * n + r] = -acc[c][0];
                if (col + 1 < n) ss[(size_t)(col + 1) * n + r] = -acc[c][1];
              }
            }
          } else {
            if (q >= 1) {
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                gacc[2 - q][c][0] = -acc[c][0];
                gacc[2 - q][c][1] = -acc[c][1];
              }
              gheld[2 - q] = true;
            }
          }
        } else {
          const bool is_d = u < 10;
          int rr, cc;
          tri_decode(is_d ? u : u - 10, rr, cc);
          // prefetched addends: A_{j+1,j+1} (D) or the running S_L (S_L), 16 x 16 tile fragments
          double old[2][2][2];
          const double* src = is_d ? args.diag + (S.start + S.j + 1) * bs : sl;
          const bool load = is_d ? !last : S.j > 0;
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              const int r = rr * 16 + i * 8 + (lane >> 2), c = cc * 16 + jj * 8 + 2 * (lane & 3);
              old[i][jj][0] = (load && r < n && c < n) ? src[(size_t)r * n + c] : 0.0;
              old[i][jj][1] = (load && r < n && c + 1 < n) ? src[(size_t)r * n + c + 1] : 0.0;
            }
          double acc[2][2][2];
          pair_syrk16(bXP, is_d ? rr : 4 + rr, is_d ? cc : 4 + cc, acc, lane);
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              if (rr == cc && jj > i) continue;
              const int r = rr * 16 + i * 8 + (lane >> 2), c = cc * 16 + jj * 8 + 2 * (lane & 3);
              if (!is_d) {  // S_L += Pt2 Pt2^T
                if (r < n && c < n) sl[(size_t)r * n + c] = old[i][jj][0] + acc[i][jj][0];
                if (r < n && c + 1 < n) sl[(size_t)r * n + c + 1] = old[i][jj][1] + acc[i][jj][1];
              } else if (!last) {  // D_{j+1} = A - Pt1 Pt1^T (identity on the padded diagonal)
                double2 v;
                v.x = (r == c && r >= n) ? 1.0 : old[i][jj][0] - acc[i][jj][0];
                v.y = (r == c + 1 && r >= n) ? 1.0 : old[i][jj][1] - acc[i][jj][1];
                *reinterpret_cast<double2*>(bDL + r * LD + c) = v;
              } else if (r < n) {  // S_R = Y_R^T Y_R
                double* dst = args.Sr + (size_t)S.k * bs + (size_t)r * n;
                if (c < n) dst[c] = acc[i][jj][0];
                if (c + 1 < n) dst[c + 1] = acc[i][jj][1];
              }
            }
        }
      }
      if (!last) {
        named_sync(kBarBulk, 32 * PS::NBULK);  // every read of Pt2 done: Gt_{j+1} replaces it
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (!gheld[q]) continue;
          const int u = bi + 12 * (2 - q);
          const int g = (u - 20) >> 1, h = (u - 20) & 1;
          double* dst = bXP + (NT + 8 * g + (lane >> 2)) * LD + 32 * h + 2 * (lane & 3);
#pragma unroll
          for (int c = 0; c < 4; ++c)
            *reinterpret_cast<double2*>(dst + c * 8) = make_double2(gacc[q][c][0], gacc[q][c][1]);
        }
      }
    }
    __syncthreads();  // ---- end of phase ----
    // uniform state updates
    if (chain_on) {
      PairSlot& S = slot[cs];
      S.fresh = false;
      if (s_fail[cs]) {
        S.k = -1;  // abandoned (failure reported)
      } else {
        S.has_chain = true;
      }
    }
    if (bulk_on) {
      PairSlot& S = slot[bsl];
      S.has_chain = false;
      if (++S.j == S.J) S.k = -1;
    }
  }
}

}  // namespace btd
