// Single-warp Cholesky of one 32 x 32 or 64 x 64 diagonal block (the pivot chain of
// factor_level_kernel and factor_stream_kernel).
//
// Left-looking over eight 8-column panels, so one warp needs no barrier at all:
//   1. panel p -= L[:, 0:8p] L[panel rows, 0:8p]^T            (DMMA tiles, independent rows)
//   2. the 8 x 8 diagonal tile is factored REDUNDANTLY in every lane's registers: the per-column
//      dependency is rcp(d) + one FMA (no shuffles, no shared-memory round trip)
//   3. rows below the tile: L_ip = A_ip L_pp^{-T} by forward substitution, one row per lane
//   4. the tile's inverse ("leaf") replaces the tile in place; 1 / L_ii goes to column NT
// Output format = potrf_trtri<64, false> (btd_factor.cuh): L with inverted 8 x 8 diagonal tiles
// (left-looking never reads a finished diagonal tile, so the leaves can be written at once).
// Failure rule as everywhere: a pivot that is not > 0 (NaN included) -> 1-based pivot returned,
// the block's contents are then undefined.
// Included by btd_factor.cuh after the helpers it uses (dmma, sub_frag, rcp_nr, rsqrt_nr).
#pragma once

namespace btd {

// leaf_bar0 (optional, > 0): panel p's leaf and the rows below it are published on the named
// barrier leaf_bar0 + p (bar.arrive by this warp, `leaf_count` threads in total with the consumers'
// bar.sync): a streaming consumer may start that column block of its triangular solve.  On a
// failure every remaining barrier is arrived on so no consumer waits forever.
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

template <int LD, int NT>
__device__ __forceinline__ int chain_potrf(double* DL, int lane, int leaf_bar0 = 0, int leaf_count = 0) {
  static_assert(NT == 32 || NT == 64, "chain_potrf factors 32 x 32 or 64 x 64 tiles");
  constexpr int NP = NT / 8;
  int fail = 0;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const int p0 = 8 * p;
    // ---- 1. left-looking update of panel p by panels 0..p-1 ----
    if (p > 0) {
      double acc[NP][2];
#pragma unroll
      for (int tr = p; tr < NP; ++tr) acc[tr][0] = acc[tr][1] = 0.0;
      const double* pb = DL + (p0 + (lane >> 2)) * LD + (lane & 3);
#pragma unroll
      for (int k0 = 0; k0 < p0; k0 += 4) {
        const double b = pb[k0];
#pragma unroll
        for (int tr = p; tr < NP; ++tr) dmma(acc[tr], DL[(tr * 8 + (lane >> 2)) * LD + k0 + (lane & 3)], b);
      }
#pragma unroll
      for (int tr = p; tr < NP; ++tr) sub_frag<LD>(DL, tr, p, lane, acc[tr]);
      __syncwarp();
    }
    // ---- 2. redundant factorization of the diagonal tile ----
    double a[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j) a[i][j] = DL[(p0 + i) * LD + p0 + j];
    double rinv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double d = a[k][k];
      if (fail == 0 && !(d > 0.0)) fail = p0 + k + 1;
      const double dinv = rcp_nr(d);
      rinv[k] = rsqrt_nr(d);
      double t[8];
#pragma unroll
      for (int i = k + 1; i < 8; ++i) t[i] = a[i][k] * dinv;
      // the next pivot first: it is the only update on the chain
      if (k + 1 < 8) a[k + 1][k + 1] = fma(-t[k + 1], a[k + 1][k], a[k + 1][k + 1]);
#pragma unroll
      for (int i = k + 1; i < 8; ++i)
#pragma unroll
        for (int j = k + 1; j <= i; ++j)
          if (!(i == k + 1 && j == k + 1)) a[i][j] = fma(-t[i], a[j][k], a[i][j]);
    }
    if (fail) {  // uniform over the warp (every lane factored the same tile)
      if (leaf_bar0)
        for (int q = p; q < NP; ++q) named_arrive(leaf_bar0 + q, leaf_count);
      return fail;
    }
    double lt[8][8];  // L_pp (normalized)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#pragma unroll
      for (int j = 0; j < i; ++j) lt[i][j] = a[i][j] * rinv[j];
      lt[i][i] = a[i][i] * rinv[i];
    }
    // ---- 3. rows below the tile: l = x L_pp^{-T} (forward substitution) ----
#pragma unroll
    for (int h = 0; h < NT / 32; ++h) {
      const int r = p0 + 8 + lane + 32 * h;
      if (r < NT) {
        double x[8];
        double* row = DL + r * LD + p0;
#pragma unroll
        for (int c = 0; c < 8; c += 2) {
          const double2 v = *reinterpret_cast<const double2*>(row + c);
          x[c] = v.x;
          x[c + 1] = v.y;
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          x[c] *= rinv[c];
#pragma unroll
          for (int m = c + 1; m < 8; ++m) x[m] = fma(-x[c], lt[m][c], x[m]);
        }
#pragma unroll
        for (int c = 0; c < 8; c += 2) *reinterpret_cast<double2*>(row + c) = make_double2(x[c], x[c + 1]);
      }
    }
    // ---- 4. leaf: lane c < 8 computes column c of L_pp^{-1} ----
    __syncwarp();  // every lane has read the diagonal tile (step 2) before lanes 0-7 overwrite it
    if (lane < 8) {
      const int c = lane;
      double x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = (i == c) ? rinv[i] : 0.0;
#pragma unroll
      for (int i = 1; i < 8; ++i) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int m = 0; m < i; ++m) {
          if (m & 1)
            s1 = fma(lt[i][m], x[m], s1);
          else
            s0 = fma(lt[i][m], x[m], s0);
        }
        if (i > c) x[i] = -(s0 + s1) * rinv[i];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) DL[(p0 + i) * LD + p0 + c] = x[i];
      DL[(p0 + c) * LD + NT] = rinv[c];
    }
    __syncwarp();
    if (leaf_bar0) named_arrive(leaf_bar0 + p, leaf_count);
  }
  return 0;
}

template <int LD, int NT>
__device__ __forceinline__ int chain_potrf64(double* DL, int lane, int leaf_bar0 = 0, int leaf_count = 0) {
  return chain_potrf<LD, NT>(DL, lane, leaf_bar0, leaf_count);
}

}  // namespace btd
