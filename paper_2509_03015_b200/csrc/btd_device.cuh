// Device-side helpers shared by the block-tridiagonal factor/solve kernels (sm_100a).
//
// fp64 on B200: tcgen05 has no .kind::f64 (ptxas rejects it), so the fp64 tensor path is the
// warp-synchronous `mma.sync.m8n8k4.f64` (SASS DMMA). Measured on this pool's B200:
// DMMA 37.1 TFLOP/s, DFMA 34.1 TFLOP/s (profiles/fp64_peak_r01.json).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace btd {

// ---------------------------------------------------------------------------------------------
// Device error word.  The reference raises NotPositiveDefinite for the earliest block step j of
// the failing level, lowest member at that step, with the 1-based pivot of that block
// (bt/block_cholesky.py:24-42, bt/kernels.py:87-101,136-181).  We pack (j, member, pivot) so that
// a single 64-bit atomicMin selects exactly that failure.
// ---------------------------------------------------------------------------------------------
struct DevErr {
  unsigned long long key;  // (block << 43) | (member << 16) | pivot ; ~0ull == no error
  int level;               // recursion level of the failure (INT_MAX == none)
  int pad;
};

constexpr unsigned long long kNoErr = ~0ull;
constexpr long long kMaxBlockCoord = (1ll << 20) - 1;
constexpr long long kMaxMemberCoord = (1ll << 27) - 1;

__device__ __forceinline__ void report_npd(DevErr* e, int level, long long block, long long member,
                                           int pivot) {
  unsigned long long j = (unsigned long long)(block < kMaxBlockCoord ? block : kMaxBlockCoord);
  unsigned long long m = (unsigned long long)(member < kMaxMemberCoord ? member : kMaxMemberCoord);
  unsigned long long key = (j << 43) | (m << 16) | (unsigned long long)(pivot & 0xffff);
  atomicMin(&e->key, key);
  atomicMin(&e->level, level);
}

__device__ __forceinline__ bool error_raised(const DevErr* e) {
  return *((volatile const unsigned long long*)&e->key) != kNoErr;
}

// A factor kernel of level `level` may skip its remaining work only when the error already recorded
// can no longer be superseded: it comes from an earlier level, or from an earlier (step, member) of
// this level than the step `j` this segment would run next (the reference reports the earliest
// step, then the lowest member).  Skipping on any error would lose an earlier failure of a CTA that
// starts after another CTA of the same level failed.
__device__ __forceinline__ bool npd_superseded(const DevErr* e, int level, long long j, long long member) {
  const unsigned long long key = *((volatile const unsigned long long*)&e->key);
  if (key == kNoErr) return false;
  const int lvl = *((volatile const int*)&e->level);
  if (lvl < level) return true;
  const long long jerr = (long long)(key >> 43);
  const long long merr = (long long)((key >> 16) & ((1ull << 27) - 1));
  return j > jerr || (j == jerr && member > merr);
}

// CTA-uniform form of npd_superseded for a kernel's entry check: the error word can be written by
// another CTA (of this or a concurrently running launch) while this CTA starts, so threads reading
// it separately could disagree and some would exit while the others wait at a barrier.  Thread 0
// decides for the CTA.  Call once, at kernel entry, from every thread.
__device__ __forceinline__ bool cta_superseded(const DevErr* e, int level, long long j, long long member) {
  __shared__ int s_superseded;
  if (threadIdx.x == 0) s_superseded = npd_superseded(e, level, j, member) ? 1 : 0;
  __syncthreads();
  return s_superseded != 0;
}

// ---------------------------------------------------------------------------------------------
// fp64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col).
// Fragment ownership (lane l): a = A[l/4][l%4], b = B[l%4][l/4], d = {D[l/4][2(l%4)], D[l/4][2(l%4)+1]}.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------------------------
// cp.async (LDGSTS) staging with zero fill.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------------------------
// mbarrier + TMA 1D bulk copy (cp.async.bulk, SASS UBLKCP): one thread moves a whole contiguous
// block global->shared; completion is tracked by transaction bytes on an mbarrier.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// The same with an L2 eviction-priority hint (createpolicy): evict_last for data that is read
// again soon (a solve's forward-sweep blocks, re-read by the backward sweep), evict_first for the
// last use.
__device__ __forceinline__ unsigned long long l2_policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                                 unsigned long long policy) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Scalar global load with an L2 eviction-priority policy (see l2_policy_*).
__device__ __forceinline__ double ld_hint(const double* p, unsigned long long policy) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(policy));
  return v;
}

// Bulk prefetch of a contiguous global range into L2 (cp.async.bulk.prefetch.L2, no completion
// tracking): used to pull the next step's diagonal block into L2 while the Cholesky runs.
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes & ~15u) : "memory");
}

// Stage an n x n row-major global block into an NT x LD shared tile, zero-padding rows/cols >= n.
template <int NT, int LD, int NTHREADS>
__device__ __forceinline__ void stage_block_async(double* sm, const double* g, int n) {
  if ((n & 1) == 0) {
    constexpr int CPR = NT / 2;
    for (int idx = threadIdx.x; idx < NT * CPR; idx += NTHREADS) {
      const int r = idx / CPR, c = (idx % CPR) * 2;
      const bool ok = (r < n) && (c < n);
      cp_async16(sm + r * LD + c, ok ? (const void*)(g + (size_t)r * n + c) : (const void*)g, ok ? 16 : 0);
    }
  } else {
    for (int idx = threadIdx.x; idx < NT * NT; idx += NTHREADS) {
      const int r = idx / NT, c = idx % NT;
      const bool ok = (r < n) && (c < n);
      cp_async8(sm + r * LD + c, ok ? (const void*)(g + (size_t)r * n + c) : (const void*)g, ok ? 8 : 0);
    }
  }
}

// Synchronous transposed staging: sm[r][c] = g[c][r] (zero padded).
template <int NT, int LD, int NTHREADS>
__device__ __forceinline__ void stage_block_transposed(double* sm, const double* g, int n) {
  for (int idx = threadIdx.x; idx < NT * NT; idx += NTHREADS) {
    const int c = idx / NT, r = idx % NT;  // read g row c (coalesced along r)
    sm[r * LD + c] = (r < n && c < n) ? g[(size_t)c * n + r] : 0.0;
  }
}

// Store the n x n leading part of a shared tile to a row-major global block.
// lower_only: write zeros above the diagonal (triangular factors).
template <int NT, int LD, int NTHREADS>
__device__ __forceinline__ void store_block(double* g, const double* sm, int n, bool lower_only) {
  if (n == NT) {
    constexpr int CPR = NT / 2;
    for (int idx = threadIdx.x; idx < NT * CPR; idx += NTHREADS) {
      const int r = idx / CPR, c = (idx % CPR) * 2;
      double2 v = *reinterpret_cast<const double2*>(sm + r * LD + c);
      if (lower_only) {
        if (c > r) v.x = 0.0;
        if (c + 1 > r) v.y = 0.0;
      }
      *reinterpret_cast<double2*>(g + (size_t)r * NT + c) = v;
    }
  } else if ((n & 1) == 0) {
    const int cpr = n / 2;
    for (int idx = threadIdx.x; idx < n * cpr; idx += NTHREADS) {
      const int r = idx / cpr, c = (idx % cpr) * 2;
      double2 v = *reinterpret_cast<const double2*>(sm + r * LD + c);
      if (lower_only) {
        if (c > r) v.x = 0.0;
        if (c + 1 > r) v.y = 0.0;
      }
      *reinterpret_cast<double2*>(g + (size_t)r * n + c) = v;
    }
  } else {
    for (int idx = threadIdx.x; idx < n * n; idx += NTHREADS) {
      const int r = idx / n, c = idx % n;
      g[(size_t)r * n + c] = (lower_only && c > r) ? 0.0 : sm[r * LD + c];
    }
  }
}

// Store the lower triangle of the n x n leading part of a shared tile in packed row-major form
// (row r at offset O_r, length L_r = 2 ceil((r+1)/2), zero padded; see packed_row_offset in
// btd_solve2.cuh): the inverse Cholesky factors are stored this way.
__host__ __device__ __forceinline__ int packed_offset_(int r) {
  const int k = r >> 1;
  return (r & 1) ? 2 * (k + 1) * (k + 1) : 2 * k * (k + 1);
}
template <int NT, int LD, int NTHREADS>
__device__ __forceinline__ void store_packed_lower(double* g, const double* sm, int n) {
  if ((n & 1) == 0 && NT <= 64) {
    // even n: a warp per row, a lane per column pair -- one 16-byte shared load and one 16-byte
    // global store per pair (packed rows start at even offsets; the block stride is even)
    constexpr int NWARPS = NTHREADS / 32;
    const int lane = threadIdx.x & 31;
    for (int r = threadIdx.x >> 5; r < n; r += NWARPS) {
      const int len = ((r + 2) >> 1) << 1, c = 2 * lane;
      if (c < len) {
        const double2 v = *reinterpret_cast<const double2*>(sm + r * LD + c);
        *reinterpret_cast<double2*>(g + packed_offset_(r) + c) = make_double2(v.x, c + 1 <= r ? v.y : 0.0);
      }
    }
    return;
  }
  // (r, c) for c <= r, plus the zero pad (r, r+1) of even rows
  for (int e = threadIdx.x; e < n * (n + 1); e += NTHREADS) {
    const int r = e / (n + 1), c = e % (n + 1);
    const int len = ((r + 2) >> 1) << 1;
    if (c < len) g[packed_offset_(r) + c] = (c <= r) ? sm[r * LD + c] : 0.0;
  }
}

// Plain global->global copy of an n x n block (used to keep the coupling blocks in the hierarchy).
template <int NTHREADS>
__device__ __forceinline__ void copy_block(double* dst, const double* src, int n) {
  const int tot = n * n;
  for (int i = threadIdx.x; i < tot; i += NTHREADS) dst[i] = src[i];
}

// The same by `nb` threads (index t), 16-byte accesses with 4 loads in flight when n is even.
__device__ __forceinline__ void copy_block_part(double* dst, const double* src, int n, int t, int nb) {
  const int tot = n * n;
  if ((n & 1) == 0) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
    double2* d2 = reinterpret_cast<double2*>(dst);
    const int h = tot / 2;
    int i = t;
    for (; i + 3 * nb < h; i += 4 * nb) {
      const double2 a = s2[i], b = s2[i + nb], c = s2[i + 2 * nb], d = s2[i + 3 * nb];
      d2[i] = a;
      d2[i + nb] = b;
      d2[i + 2 * nb] = c;
      d2[i + 3 * nb] = d;
    }
    for (; i < h; i += nb) d2[i] = s2[i];
  } else {
    for (int i = t; i < tot; i += nb) dst[i] = src[i];
  }
}

// Transposed staging sm[r][c] = g[c][r] (zero padded) by `nb` threads (index t), 4 loads in flight.
template <int NT, int LD>
__device__ __forceinline__ void stage_block_transposed_part(double* sm, const double* g, int n, int t, int nb) {
  int idx = t;
  for (; idx + 3 * nb < NT * NT; idx += 4 * nb) {
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = idx + q * nb, c = e / NT, r = e % NT;
      v[q] = (r < n && c < n) ? g[(size_t)c * n + r] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = idx + q * nb, c = e / NT, r = e % NT;
      sm[r * LD + c] = v[q];
    }
  }
  for (; idx < NT * NT; idx += nb) {
    const int c = idx / NT, r = idx % NT;
    sm[r * LD + c] = (r < n && c < n) ? g[(size_t)c * n + r] : 0.0;
  }
}

}  // namespace btd
