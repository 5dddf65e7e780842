// C-ABI implementation: recursion planning, workspace layout and kernel launches.
// See include/blocktri_b200.h for the reference interface each entry point replaces.
#include "../../include/blocktri_b200.h"

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "btd_factor.cuh"
#include "btd_factor3.cuh"
#include "btd_solve.cuh"
#include "btd_solve2.cuh"
#include "btd_solve3.cuh"
#include "btd_big.cuh"
#include "btd_spmv.cuh"
#include "btd_small.cuh"
#include "btd_kalman.cuh"
#include "btd_seam.cuh"

namespace {

// every kernel this library launches (btd_launch_count: bench.py gpu_launches)
std::atomic<long long> g_launches{0};

constexpr size_t kAlign = 256;
size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

struct LevelPlan {
  int64_t N = 0;  // blocks of this level's matrix
  int64_t P = 0;  // separators (= blocks of the next level)
  int64_t K = 0;  // segments
  int64_t step = 0;  // rho + 1: separators are k * step (k < P-1) and N-1 (plan_partition, closed form)
  int64_t sep(int64_t k) const { return k == P - 1 ? N - 1 : k * step; }
  int64_t max_segment() const {  // longest segment (the tail absorbs the gap)
    if (K < 1) return 0;
    const int64_t regular = K > 1 ? step - 1 : 0;
    return std::max(regular, sep(K) - sep(K - 1) - 1);
  }
  // persistent offsets
  size_t off_seps = 0, off_linv = 0, off_lsub = 0;
  // factor-scratch offsets: next level matrix + S_R scratch
  size_t off_next_diag = 0, off_next_sub = 0, off_sr = 0;
};

}  // namespace

struct btd_hierarchy {
  int64_t N = 0, n = 0;
  btd_config cfg{};
  int nt = 0;
  std::vector<LevelPlan> levels;
  int64_t base_N = 0;
  bool overflow = false;
  size_t off_err = 0, off_base_linv = 0, off_base_lsub = 0;
  bool big = false;              // n > 64: tiled path (btd_big.cuh), Linv stored full n x n
  bool partial = false;          // sharded chunk: exactly `levels` local levels, no base
  int64_t kmax = 1;              // most segments of any level (big-path workspaces)
  size_t off_big_ws = 0;         // factor scratch: WD | WX | WP per segment
  size_t off_splitk = 0;         // factor scratch: split-k partials of the base GEMMs
  size_t persistent_bytes = 0, scratch_bytes = 0;
  char* persistent = nullptr;
  bool factored = false;
  bool pending_check = false;
  // optional per-launch timing of the factor kernels (btd_profile_kernels)
  bool profile = false;
  std::vector<cudaEvent_t> ev;
  int nev = 0;
  cudaStream_t copy_stream = nullptr;  // btd_factorize_from_host
  // n > 64: wide levels run as two half-level launch sequences on two streams, so one half's
  // Cholesky kernels overlap the other half's tile GEMMs
  cudaStream_t aux_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_half[2] = {nullptr, nullptr};  // host input: the two halves' H2D copies landed
  ~btd_hierarchy() {
    for (cudaEvent_t e : ev_half)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (aux_stream) cudaStreamDestroy(aux_stream);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
  }
};

namespace {

enum SolvePhase : int { kPhaseFull = 0, kPhaseDown = 1, kPhaseUp = 2 };

void prof_mark(btd_hierarchy* h, cudaStream_t s) {
  if (!h->profile) return;
  if (h->nev >= (int)h->ev.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    h->ev.push_back(e);
  }
  cudaEventRecord(h->ev[h->nev++], s);
}

void set_status(btd_status* st, int code, const char* fmt, ...) __attribute__((format(printf, 3, 4)));
void set_status(btd_status* st, int code, const char* fmt, ...) {
  if (!st) return;
  st->code = code;
  st->pivot = -1;
  st->level = st->member = st->block = -1;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(st->message, sizeof(st->message), fmt, ap);
  va_end(ap);
}

void clear_status(btd_status* st) {
  if (!st) return;
  st->code = BTD_OK;
  st->pivot = -1;
  st->level = st->member = st->block = -1;
  st->message[0] = '\0';
}

int cuda_fail(btd_status* st, cudaError_t e, const char* where) {
  set_status(st, BTD_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
  return BTD_ERR_CUDA;
}

bool config_ok(const btd_config* c) {
  return c && c->crossover >= 1 && c->segment_length >= 1 && c->max_levels >= 1;
}

// plan_partition (bt/schur.py:75-95): separators at 0, rho+1, 2(rho+1), ...; the last block is always
// a separator; a regular separator adjacent to it is dropped so the tail segment absorbs the gap.
std::vector<int64_t> plan_separators(int64_t N, int64_t rho) {
  const int64_t step = rho + 1;
  std::vector<int64_t> s((size_t)((N + step - 1) / step));
  for (size_t k = 0; k < s.size(); ++k) s[k] = (int64_t)k * step;
  s.reserve(s.size() + 1);
  if (s.back() != N - 1) {
    if (s.back() == N - 2) s.pop_back();
    s.push_back(N - 1);
  }
  return s;
}

// _should_recurse (bt/schur.py:321-326)
bool should_recurse(int64_t N, const btd_config& cfg) {
  if (N < 3) return false;
  if (cfg.auto_crossover) return plan_separators(N, cfg.segment_length).size() - 1 >= 2;
  return N > cfg.crossover;
}

// ---- per-device launch state --------------------------------------------------------------
// The dynamic shared-memory attribute and the SM count are per device, and one process may drive
// several GPUs from several threads: both are cached per (kernel, device) under a mutex.
constexpr int kMaxDevices = 64;

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

int device_sms() {
  static std::atomic<int> cache[kMaxDevices];
  const int d = current_device();
  int v = (d >= 0 && d < kMaxDevices) ? cache[d].load(std::memory_order_relaxed) : 0;
  if (!v) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v < 1) v = 148;
    if (d >= 0 && d < kMaxDevices) cache[d].store(v, std::memory_order_relaxed);
  }
  return v;
}

std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, int> g_smem_set;       // (kernel, device) -> configured bytes
std::map<std::pair<const void*, int>, int> g_blocks_per_sm;  // (kernel, device) -> occupancy

// cudaFuncAttributeMaxDynamicSharedMemorySize >= smem for `fn` on the current device
cudaError_t ensure_smem(const void* fn, size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  const int d = current_device();
  std::lock_guard<std::mutex> lk(g_attr_mu);
  int& have = g_smem_set[{fn, d}];
  if (have >= (int)smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) have = (int)smem;
  return e;
}

// resident CTAs per SM of `fn` on the current device (after ensure_smem)
int resident_blocks(const void* fn, int threads, size_t smem) {
  const int d = current_device();
  std::lock_guard<std::mutex> lk(g_attr_mu);
  auto it = g_blocks_per_sm.find({fn, d});
  if (it != g_blocks_per_sm.end()) return it->second;
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, threads, smem) != cudaSuccess || b < 1) {
    cudaGetLastError();
    b = 1;
  }
  g_blocks_per_sm[{fn, d}] = b;
  return b;
}

// grid of a flattened grid-stride elementwise kernel (256 threads per CTA)
unsigned flat_grid(int64_t elements) {
  const int sms = device_sms();
  const int64_t want = (elements + 255) / 256;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 16));
}

// Next-level diagonal blocks (btd_factor.cuh): a warp per block row for even n >= 32 (cfg2 level 0
// 131 -> 106 us); the flat element kernel for small blocks (a warp per 8-double row idles 28 lanes:
// cfg3 level 0 40 -> 187 us).
void launch_assemble(const double* diag, const int* seps, double* next_diag, const double* Sr, int K, int64_t n,
                     btd::DevErr* err, cudaStream_t s) {
  const int64_t P = (int64_t)K + 1;
  if ((n & 1) == 0 && n >= 32) {
    const int64_t warps = P * n;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, (int64_t)device_sms() * 16));
    btd::assemble_schur_diag_rows_kernel<<<grid, 256, 0, s>>>(diag, seps, next_diag, Sr, K, (int)n, err);
  } else {
    btd::assemble_schur_diag_kernel<<<flat_grid(P * n * n), 256, 0, s>>>(diag, seps, next_diag, Sr, K, (int)n, err);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

int pick_nt(int64_t n) {
  if (n <= 8) return 8;
  if (n <= 16) return 16;
  if (n <= 32) return 32;
  if (n <= 64) return 64;
  return 0;
}

template <int NT>
cudaError_t launch_factor(const btd::FactorArgs& a, unsigned grid, cudaStream_t s) {
  using S = btd::FactorShape<NT>;
  constexpr size_t smem = S::SMEM;
  cudaError_t e = ensure_smem((const void*)btd::factor_level_kernel<NT>, smem);
  if (e != cudaSuccess) return e;
  btd::factor_level_kernel<NT><<<grid, S::NTHREADS, smem, s>>>(a); g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// Streaming schedule (btd_factor3.cuh) at NT = 64 for levels that fit in one wave of one CTA per
// SM (and the base): its per-step latency is lower than factor_level_kernel's, but with one CTA
// per SM it sustains less DMMA throughput on wide levels (measured: level 0 of cfg2 9.1 ms vs
// 6.6 ms), where two factor_level_kernel CTAs per SM hide each other's pivot chains better.
bool use_stream(int nt, const btd::FactorArgs& a) {
  if (nt != 64) return false;
  return a.base || a.K <= device_sms();
}

cudaError_t launch_stream64(const btd::FactorArgs& a, unsigned grid, cudaStream_t s) {
  using SS = btd::StreamShape;
  cudaError_t e = ensure_smem((const void*)btd::factor_stream_kernel, SS::SMEM);
  if (e != cudaSuccess) return e;
  btd::factor_stream_kernel<<<grid, SS::NTHREADS, SS::SMEM, s>>>(a); g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// Small-block kernels (btd_small.cuh) at NT = 8: an 8-lane group per segment.
bool use_small(int nt) { return nt == 8; }

cudaError_t dispatch_factor(int nt, const btd::FactorArgs& a, unsigned grid, cudaStream_t s) {
  if (use_small(nt)) {
    const unsigned g = a.base ? 1u : (grid + 15) / 16;
    cudaError_t e = ensure_smem((const void*)btd::factor_small_kernel, btd::kS2Smem);
    if (e != cudaSuccess) return e;
    btd::factor_small_kernel<<<g, btd::kSmallThreads, btd::kS2Smem, s>>>(a);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
  }
  if (use_stream(nt, a)) return launch_stream64(a, grid, s);
  switch (nt) {
    case 8: return launch_factor<8>(a, grid, s);
    case 16: return launch_factor<16>(a, grid, s);
    case 32: return launch_factor<32>(a, grid, s);
    case 64: return launch_factor<64>(a, grid, s);
  }
  return cudaErrorInvalidValue;
}

template <int NT, int DC>
cudaError_t launch_solve(const btd::SolveArgs& a, unsigned grid_x, cudaStream_t s) {
  dim3 grid(grid_x, (unsigned)((a.d + DC - 1) / DC));
  btd::solve_level_kernel<NT, DC><<<grid, btd::SolveShape<NT>::NTHREADS, 0, s>>>(a); g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <int NT>
cudaError_t dispatch_solve_dc(const btd::SolveArgs& a, unsigned grid_x, cudaStream_t s) {
  if (a.d == 1) return launch_solve<NT, 1>(a, grid_x, s);
  if (a.d == 2) return launch_solve<NT, 2>(a, grid_x, s);
  return launch_solve<NT, 4>(a, grid_x, s);
}

template <int NT, int DC, bool WIDE>
cudaError_t launch_stream_v(const btd::SolveArgs& a, cudaStream_t s) {
  using T = btd::TmaShape<NT, DC, WIDE>;
  const void* fn = (const void*)btd::solve_tma_kernel<NT, DC, WIDE>;
  cudaError_t e = ensure_smem(fn, T::SMEM);
  if (e != cudaSuccess) return e;
  const long long cap = (long long)resident_blocks(fn, T::NTHREADS, T::SMEM) * device_sms();
  const unsigned gx = (unsigned)(a.K < cap ? a.K : cap);
  dim3 grid(gx, (unsigned)((a.d + DC - 1) / DC));
  btd::solve_tma_kernel<NT, DC, WIDE><<<grid, T::NTHREADS, T::SMEM, s>>>(a); g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// Wide levels (at least as many segments as SMs) at n = 64 run two CTAs per SM; narrow levels and
// the base keep one CTA per SM with a deeper ring (more prefetch for the lone segment).
template <int NT, int DC>
cudaError_t launch_stream(const btd::SolveArgs& a, cudaStream_t s) {
  if constexpr (NT == 64) {
    if (a.mode != btd::kSolveBase && a.K >= device_sms()) return launch_stream_v<NT, DC, true>(a, s);
  }
  return launch_stream_v<NT, DC, false>(a, s);
}

template <int NT>
cudaError_t dispatch_stream_dc(const btd::SolveArgs& a, cudaStream_t s) {
  if (a.d == 1) return launch_stream<NT, 1>(a, s);
  if (a.d == 2) return launch_stream<NT, 2>(a, s);
  return launch_stream<NT, 4>(a, s);
}

cudaError_t dispatch_stream(int nt, const btd::SolveArgs& a, cudaStream_t s) {
  switch (nt) {
    case 8: return dispatch_stream_dc<8>(a, s);
    case 16: return dispatch_stream_dc<16>(a, s);
    case 32: return dispatch_stream_dc<32>(a, s);
    case 64: return dispatch_stream_dc<64>(a, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_solve_small(const btd::SolveArgs& a, cudaStream_t s) {
  const unsigned gx = a.mode == btd::kSolveBase ? 1u : (unsigned)((a.K + 15) / 16);
  const int dc = a.d == 1 ? 1 : a.d == 2 ? 2 : 4;
  dim3 grid(gx, (unsigned)((a.d + dc - 1) / dc));
  if (dc == 1) btd::solve_small_kernel<1><<<grid, btd::kSmallThreads, btd::SS2<1>::SMEM, s>>>(a);
  else if (dc == 2) btd::solve_small_kernel<2><<<grid, btd::kSmallThreads, btd::SS2<2>::SMEM, s>>>(a);
  else btd::solve_small_kernel<4><<<grid, btd::kSmallThreads, btd::SS2<4>::SMEM, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t dispatch_solve(int nt, const btd::SolveArgs& a, unsigned grid_x, cudaStream_t s) {
  switch (nt) {
    case 8: return dispatch_solve_dc<8>(a, grid_x, s);
    case 16: return dispatch_solve_dc<16>(a, grid_x, s);
    case 32: return dispatch_solve_dc<32>(a, grid_x, s);
    case 64: return dispatch_solve_dc<64>(a, grid_x, s);
  }
  return cudaErrorInvalidValue;
}

void decode_error(const btd::DevErr& e, btd_status* st) {
  const long long j = (long long)(e.key >> 43);
  const long long member = (long long)((e.key >> 16) & ((1ull << 27) - 1));
  const int pivot = (int)(e.key & 0xffff);
  set_status(st, BTD_ERR_NOT_POSITIVE_DEFINITE,
             "matrix is not positive definite at pivot %d, block %lld, member %lld, level %d", pivot, j, member,
             e.level);
  st->pivot = pivot;
  st->block = j;
  st->member = member;
  st->level = e.level;
}

int finish_check(btd_hierarchy* h, cudaStream_t stream, btd_status* st) {
  // the error word lands in a pinned per-thread word (a pageable destination goes through a driver
  // staging copy, on the critical path between the last factor kernel and the caller's next launch);
  // consumed before this thread's next factorization, so one word per thread serves every device
  thread_local btd::DevErr* pinned = nullptr;
  if (!pinned && cudaHostAlloc((void**)&pinned, sizeof(btd::DevErr), cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    pinned = nullptr;
  }
  btd::DevErr local;
  btd::DevErr* dst = pinned ? pinned : &local;
  cudaError_t e = cudaMemcpyAsync(dst, h->persistent + h->off_err, sizeof(btd::DevErr), cudaMemcpyDeviceToHost, stream);
  if (e != cudaSuccess) return cuda_fail(st, e, "btd_factorize(copy error word)");
  e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return cuda_fail(st, e, "btd_factorize(sync)");
  const btd::DevErr herr = *dst;
  h->pending_check = false;
  if (herr.key != btd::kNoErr) {
    h->factored = false;
    decode_error(herr, st);
    return BTD_ERR_NOT_POSITIVE_DEFINITE;
  }
  if (h->overflow) {
    h->factored = false;
    set_status(st, BTD_ERR_LEVEL_OVERFLOW, "recursion needs more than max_levels=%lld levels",
               (long long)h->cfg.max_levels);
    return BTD_ERR_LEVEL_OVERFLOW;
  }
  h->factored = true;
  return BTD_OK;
}


// =============================================================================================
// n > 64: host sequencing of the tiled path (btd_big.cuh)
// =============================================================================================
btd::Operand opnd(const double* base, long long stride, int ld, int index, int delta = 0, int row0 = 0,
                  int trans = 0) {
  btd::Operand o;
  o.base = base;
  o.stride = stride;
  o.ld = ld;
  o.index = index;
  o.delta = delta;
  o.row0 = row0;
  o.col0 = 0;
  o.trans = trans;
  return o;
}

struct BigCtx {
  const int* seps;
  long long N;
  int base_mode, K;  // K: segments of this launch sequence, starting at segment k0
  const btd::DevErr* err;
  cudaStream_t s;
  int k0 = 0;
  int Kws = 0;  // segments the per-segment workspaces are laid out for (0: K)
  // segment lengths present in this launch sequence (regular plan: all segments but the last
  // have the same length); 0 = unknown (every launch is issued)
  int jreg = 0, jtail = 0;
  double* part = nullptr;  // split-k partials workspace (single-segment sequences: the serial base)
  size_t part_doubles = 0;
  int level = INT_MAX;     // factor level (INT_MAX: solve sequences)
};

// split-k partials of the base solve's n x d products: 8 splits of ceil(n/64) x ceil(d/64) tiles
size_t big_solve_part_doubles(int64_t n, int64_t d) {
  return (size_t)8 * ((n + 63) / 64) * ((d + 63) / 64) * 64 * 64;
}

void set_lengths(BigCtx& c, const LevelPlan& lp) {
  if (lp.K < 1) return;
  c.jreg = (int)(lp.sep(1) - lp.sep(0) - 1);
  c.jtail = (int)(lp.sep(lp.K) - lp.sep(lp.K - 1) - 1);
}

// Does any segment of the sequence do work at step j for this activity?  Launches that would only
// start CTAs to exit (e.g. the last-row products at every other step) are skipped on the host.
bool big_any_active(const BigCtx& c, int j, int act) {
  if (!c.jreg) return true;
  auto hit = [&](int J) {
    switch (act) {
      case btd::kActNotLast: return j < J - 1;
      case btd::kActLast: return j == J - 1;
      case btd::kActBeforeSecondLast: return j < J - 2;
      case btd::kActSecondLast: return j == J - 2;
      default: return j < J;
    }
  };
  return hit(c.jreg) || hit(c.jtail);
}

cudaError_t big_gemm(const BigCtx& c, int j, int act, btd::Operand A, btd::Operand B, btd::Operand Cin,
                     btd::Operand Cout, int m, int n, int k, double alpha, double beta, int lower = 0, int tri = 0,
                     int store_trans = 0) {
  if (!big_any_active(c, j, act)) return cudaSuccess;
  const int smem = 4 * btd::GSTAGE * (int)sizeof(double);  // 2 stages x (A, B) tiles
  {
    const void* fns[4] = {(const void*)btd::bt_gemm_kernel<false, false>, (const void*)btd::bt_gemm_kernel<false, true>,
                          (const void*)btd::bt_gemm_kernel<true, false>, (const void*)btd::bt_gemm_kernel<true, true>};
    for (const void* f : fns) {
      cudaError_t e = ensure_smem(f, smem);
      if (e != cudaSuccess) return e;
    }
  }
  btd::GemmArgs g{};
  g.A = A;
  g.B = B;
  g.Cin = Cin;
  g.Cout = Cout;
  g.seps = c.seps;
  g.N = c.N;
  g.base_mode = c.base_mode;
  g.j = j;
  g.act = act;
  g.level = c.level;
  g.m = m;
  g.n = n;
  g.k = k;
  g.alpha = alpha;
  g.beta = beta;
  g.lower_only = lower;
  g.tri = tri;
  g.store_trans = store_trans;
  g.tiles_n = (n + btd::BT - 1) / btd::BT;
  g.k0 = c.k0;
  g.err = c.err;
  const int tiles = ((m + btd::BT - 1) / btd::BT) * g.tiles_n;
  // split-k when the grid is far too small for the machine (the serial base: one segment) and k is
  // long enough to pay for the extra reduce launch (measured: a loss at k = 128/256, a gain at 1024)
  g.ksplit = 1;
  constexpr int mink = 512;
  if (c.part && c.K == 1 && k >= mink) {
    const int sms = device_sms();
    int ks = std::min(8, std::max(1, sms / std::max(1, 2 * tiles)));
    ks = std::min(ks, std::max(1, k / btd::BK));
    while (ks > 1 && (size_t)tiles * ks * btd::BT * btd::BT > c.part_doubles) --ks;
    g.ksplit = ks;
    g.part = c.part;
  }
  dim3 grid((unsigned)(tiles * g.ksplit), (unsigned)c.K);
  if (!A.trans && !B.trans) btd::bt_gemm_kernel<false, false><<<grid, btd::BTHREADS, smem, c.s>>>(g);
  else if (!A.trans) btd::bt_gemm_kernel<false, true><<<grid, btd::BTHREADS, smem, c.s>>>(g);
  else if (!B.trans) btd::bt_gemm_kernel<true, false><<<grid, btd::BTHREADS, smem, c.s>>>(g);
  else btd::bt_gemm_kernel<true, true><<<grid, btd::BTHREADS, smem, c.s>>>(g);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (g.ksplit > 1) {
    btd::bt_gemm_reduce_kernel<<<dim3((unsigned)tiles, (unsigned)c.K), btd::BTHREADS, 0, c.s>>>(g);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  return cudaGetLastError();
}

cudaError_t big_copy(const BigCtx& c, int j, int act, btd::Operand src, btd::Operand dst, int rows, int cols) {
  if (!big_any_active(c, j, act)) return cudaSuccess;
  btd::CopyArgs a{};
  a.src = src;
  a.dst = dst;
  a.seps = c.seps;
  a.N = c.N;
  a.base_mode = c.base_mode;
  a.j = j;
  a.act = act;
  a.level = c.level;
  a.rows = rows;
  a.cols = cols;
  a.k0 = c.k0;
  a.err = c.err;
  const long long tot = (long long)rows * cols;
  dim3 grid((unsigned)std::min<long long>((tot + 255) / 256, 64), (unsigned)c.K);
  btd::bt_copy_kernel<<<grid, 256, 0, c.s>>>(a); g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// CTAs per segment for big_potrf_kernel: 1 on wide levels; on narrow levels (the serial base, a
// level with fewer segments than SMs) a cluster of up to 8 CTAs shares each block's tile GEMMs.
int big_potrf_cluster(int K, int n, int sms) {
  const int NB = n / btd::BT;
  const int maxc = std::max(1, std::min(8, NB * (NB - 1) / 2));  // more CTAs than trailing tiles idle
  if (K >= sms) return 1;
  return std::max(1, std::min(maxc, sms / std::max(K, 1)));
}

// Split a wide n > 64 level into two half-level launch sequences on two streams: each half's
// big_potrf_kernel (latency-bound, < 2 waves) overlaps the other half's tile GEMMs.
bool big_split_level(int64_t K) { return K >= 2 * (int64_t)device_sms(); }

cudaError_t ensure_aux(btd_hierarchy* h) {
  cudaError_t e = cudaSuccess;
  if (!h->aux_stream) e = cudaStreamCreateWithFlags(&h->aux_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess && !h->ev_fork) e = cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess && !h->ev_join) e = cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming);
  return e;
}

// Blocked Cholesky + inverse of the n x n working blocks of one step (replaces big_potrf_kernel when
// big_seq_potrf says so): per 64-column block kb the diagonal tile (big_diag_potrf_kernel), the
// panel L_ib = A_ib Linv_kk^T and the trailing update A_ij -= L_ib L_jb^T as batched tile GEMMs;
// then the inverse row by row, Linv[i][0:i] = -Linv_ii (L[i][0:i] Linv[0:i][0:i]) with the inner
// product parked transposed in the unused strict upper tiles of the working block.
cudaError_t big_potrf_seq(const BigCtx& c, int level, int j, int n, double* WD, double* Linv, btd::DevErr* err) {
  using namespace btd;
  const int NB = n / BT;
  const long long nn = (long long)n * n;
  auto D_at = [&](int r0, int c0, int trans = 0) {
    Operand o = opnd(WD, nn, n, kIdxSeg);
    o.row0 = r0;
    o.col0 = c0;
    o.trans = trans;
    return o;
  };
  auto L_at = [&](int r0, int c0, int trans = 0) {
    Operand o = opnd(Linv, nn, n, kIdxSegRow);
    o.row0 = r0;
    o.col0 = c0;
    o.trans = trans;
    return o;
  };
  BigDiagArgs a{};
  a.D = opnd(WD, nn, n, kIdxSeg);
  a.Linv = opnd(Linv, nn, n, kIdxSegRow);
  a.seps = c.seps;
  a.N = c.N;
  a.base_mode = c.base_mode;
  a.j = j;
  a.n = n;
  a.level = level;
  a.k0 = c.k0;
  a.err = err;
  cudaError_t e;
  for (int kb = 0; kb < NB; ++kb) {
    a.kb = kb;
    big_diag_potrf_kernel<<<(unsigned)c.K, 128, 0, c.s>>>(a); g_launches.fetch_add(1, std::memory_order_relaxed);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (kb + 1 == NB) break;
    const int r0 = (kb + 1) * BT, rows = n - r0;
    e = big_gemm(c, j, kActAll, D_at(r0, kb * BT), L_at(kb * BT, kb * BT, 1), D_at(r0, kb * BT), D_at(r0, kb * BT),
                 rows, BT, BT, 1.0, 0.0);
    if (e != cudaSuccess) return e;
    e = big_gemm(c, j, kActAll, D_at(r0, kb * BT), D_at(r0, kb * BT, 1), D_at(r0, r0), D_at(r0, r0), rows, rows, BT,
                 -1.0, 1.0, 1);
    if (e != cudaSuccess) return e;
  }
  for (int ib = 1; ib < NB; ++ib) {
    const int w = ib * BT;
    // T = L[ib][0:ib] Linv[0:ib][0:ib] (Linv lower: tri 4), stored transposed at D[0:w][w:w+64]
    e = big_gemm(c, j, kActAll, D_at(w, 0), L_at(0, 0), D_at(0, w), D_at(0, w), BT, w, w, 1.0, 0.0, 0, 4, 1);
    if (e != cudaSuccess) return e;
    // Linv[ib][0:ib] = -Linv_ii T  (Linv_ii lower: tri 2)
    e = big_gemm(c, j, kActAll, L_at(w, w), D_at(0, w, 1), L_at(w, 0), L_at(w, 0), BT, w, BT, -1.0, 0.0, 0, 2);
    if (e != cudaSuccess) return e;
  }
  if (NB > 1) {
    big_zero_upper_kernel<<<dim3((unsigned)(NB * (NB - 1) / 2), (unsigned)c.K), 256, 0, c.s>>>(a);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    e = cudaGetLastError();
  }
  return e;
}

// big_potrf_seq (batched tile launches) vs big_potrf_kernel (one CTA / cluster per block)
bool big_seq_potrf(int n, int K) {
  (void)K;
  // measured: the per-launch cost of the k = 64 tile GEMMs loses below n = 1024 (cfg4 factor
  // 38.6 vs 33.3 ms, n = 512 53 vs 47 ms) and wins at n = 1024 (111 vs 129 ms)
  return n >= 1024;
}

// One level (coupled) or the base (base_mode) of the tiled factorization.
cudaError_t big_factor_level(const BigCtx& c, int level, int Jmax, int n, const double* diag, const double* sub,
                             double* Linv, double* Lsub, double* Sl, double* Sr, double* Ssub, char* ws,
                             btd::DevErr* err) {
  using namespace btd;
  const long long nn = (long long)n * n;
  const size_t Kws = (size_t)(c.Kws ? c.Kws : c.K);  // the same layout for both halves of a split level
  double* WD = (double*)ws;
  double* WX = WD + Kws * nn;
  double* WP = WX + Kws * 2 * nn;
  const bool coupled = !c.base_mode;
  const Operand oWD = opnd(WD, nn, n, kIdxSeg), oWP = opnd(WP, 2 * nn, n, kIdxSeg);
  const Operand oWXhi = opnd(WX, 2 * nn, n, kIdxSeg, 0, n), oWPhi = opnd(WP, 2 * nn, n, kIdxSeg, 0, n);
  const Operand oLinv = opnd(Linv, nn, n, kIdxSegRow);
  cudaError_t e;
#define BIG_CHECK(x)              \
  do {                            \
    e = (x);                      \
    if (e != cudaSuccess) return e; \
  } while (0)
  // ---- prologue ----
  // X1 (A_{j+1,j}, or C_R at the last row) is read by the P1 product straight from `sub`; only the
  // fill coupling Gt lives in the workspace (rows n..2n of WX)
  BIG_CHECK(big_copy(c, 0, kActAll, opnd(diag, nn, n, kIdxSegRow), oWD, n, n));
  if (coupled) {
    BIG_CHECK(big_copy(c, 0, kActAll, opnd(sub, nn, n, kIdxSegStart, 0, 0, 1), oWXhi, n, n));  // C_L^T
    BIG_CHECK(big_copy(c, 0, kActAll, opnd(sub, nn, n, kIdxSegStart), opnd(Lsub, nn, n, kIdxSegStart), n, n));
    BIG_CHECK(big_copy(c, 0, kActAll, opnd(sub, nn, n, kIdxSegStop, -1), opnd(Lsub, nn, n, kIdxSegStop, -1), n, n));
  }
  const Operand oLinvT = opnd(Linv, nn, n, kIdxSegRow, 0, 0, 1);
  const Operand oL1 = opnd(Lsub, nn, n, kIdxSegRow), oL1t = opnd(Lsub, nn, n, kIdxSegRow, 0, 0, 1);
  for (int j = 0; j < Jmax; ++j) {
    if (big_seq_potrf(n, c.K)) {
      BIG_CHECK(big_potrf_seq(c, level, j, n, WD, Linv, err));
    } else {
      BigPotrfArgs a{};
      a.D = oWD;
      a.Linv = oLinv;
      a.seps = c.seps;
      a.N = c.N;
      a.base_mode = c.base_mode;
      a.j = j;
      a.n = n;
      a.level = level;
      a.k0 = c.k0;
      a.err = err;
      const int smem = (BT * FactorShape<64>::LD + 4 * GSTAGE) * (int)sizeof(double);
      BIG_CHECK(ensure_smem((const void*)big_potrf_kernel, smem));
      const int sms = device_sms();
      // a cluster of CTAs per segment when the level is too narrow to fill the SMs
      a.csize = big_potrf_cluster(c.K, n, sms);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3((unsigned)(c.K * a.csize));
      cfg.blockDim = dim3(BTHREADS);
      cfg.dynamicSmemBytes = (size_t)smem;
      cfg.stream = c.s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = (unsigned)a.csize;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      BIG_CHECK(cudaLaunchKernelEx(&cfg, big_potrf_kernel, a)); g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    // P1 = X1 Linv^T: inside the segment it is L_{j+1,j}, written straight into the hierarchy's Lsub
    // slot; at the last row it is Y_R = C_R Linv^T (workspace WP).  P2 = Gt Linv^T -> WP rows n..2n.
    BIG_CHECK(big_gemm(c, j, kActNotLast, opnd(sub, nn, n, kIdxSegRow), oLinvT, oL1, oL1, n, n, n, 1.0, 0.0, 0, 1));
    if (coupled) {
      BIG_CHECK(big_gemm(c, j, kActLast, opnd(sub, nn, n, kIdxSegStop, -1), oLinvT, oWP, oWP, n, n, n, 1.0, 0.0, 0, 1));
      BIG_CHECK(big_gemm(c, j, kActAll, oWXhi, oLinvT, oWPhi, oWPhi, n, n, n, 1.0, 0.0, 0, 1));
      // fill block G^T = -P2 P1^T, or at the last row S_sub = (-P2 P1^T)^T
      const Operand oP1t = opnd(WP, 2 * nn, n, kIdxSeg, 0, 0, 1);
      BIG_CHECK(big_gemm(c, j, kActNotLast, oWPhi, oL1t, oWXhi, oWXhi, n, n, n, -1.0, 0.0));
      BIG_CHECK(big_gemm(c, j, kActLast, oWPhi, oP1t, opnd(Ssub, nn, n, kIdxSeg), opnd(Ssub, nn, n, kIdxSeg), n, n, n,
                         -1.0, 0.0, 0, 0, 1));
      // S_L (+)= P2 P2^T
      const Operand oSl = opnd(Sl, nn, n, kIdxSeg);
      BIG_CHECK(big_gemm(c, j, kActAll, oWPhi, opnd(WP, 2 * nn, n, kIdxSeg, 0, n, 1), oSl, oSl, n, n, n, 1.0,
                         j > 0 ? 1.0 : 0.0, 1));
      // S_R = P1 P1^T at the last row
      BIG_CHECK(big_gemm(c, j, kActLast, oWP, oP1t, opnd(Sr, nn, n, kIdxSeg), opnd(Sr, nn, n, kIdxSeg), n, n, n, 1.0,
                         0.0, 1));
    }
    // D_{j+1} = A_{j+1,j+1} - P1 P1^T
    BIG_CHECK(big_gemm(c, j, kActNotLast, oL1, oL1t, opnd(diag, nn, n, kIdxSegRow, 1), oWD, n, n, n, -1.0, 1.0, 1));
  }
  return cudaSuccess;
}

// One level pass of the tiled solve.  mode: down (fold), up (boundary + solution), base.
// n > 64 with d <= 4 on a level with many segments: solve_wide_kernel (btd_solve3.cuh), one CTA
// per segment streaming the blocks, instead of tile GEMMs that would fill d of 64 output columns.
// Narrow levels and the serial base keep the GEMM path (one CTA per segment would stream whole
// blocks through a single SM).
// 5 <= d <= 8: solve_dmma_kernel (btd_solve3.cuh), one CTA per segment, the block products on
// DMMA with the matrix fragments read from global memory ((512, 128, 8): solve 4.63 -> 3.28 ms).
// Wider right-hand sides keep the tile GEMMs: with one CTA per 8-column slice every slice re-reads
// the blocks (cfg4, d = 64: 15.2 -> 34 ms measured).
bool use_wide_solve(int n, int d, int64_t K) {
  if (d >= 5 && d <= 8 && n % 64 == 0) return true;
  // blocks of <= 128 KB (n <= 128) stream fast enough through one SM even on narrow levels and
  // the serial base; n = 192, 256 only when the level has many segments
  return d <= 4 && (n <= 128 || (n <= 256 && K >= 64));
}

template <int DC>
cudaError_t launch_wide_dc(const btd::SolveArgs& a, cudaStream_t s) {
  const size_t smem = (size_t)5 * a.n * DC * sizeof(double);
  cudaError_t e = ensure_smem((const void*)btd::solve_wide_kernel<DC>, smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)(a.mode == btd::kSolveBase ? 1 : a.K), (unsigned)((a.d + DC - 1) / DC));
  btd::solve_wide_kernel<DC><<<grid, btd::kWideThreads, smem, s>>>(a); g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_wide(const btd::SolveArgs& a, cudaStream_t s) {
  if (a.d >= 5) {
    const size_t smem = (size_t)5 * a.n * btd::kDmmaDS * sizeof(double);
    cudaError_t e = ensure_smem((const void*)btd::solve_dmma_kernel, smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((a.d + btd::kDmmaDS - 1) / btd::kDmmaDS), (unsigned)(a.mode == btd::kSolveBase ? 1 : a.K));
    btd::solve_dmma_kernel<<<grid, btd::kWideThreads, smem, s>>>(a);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
  }
  if (a.d == 1) return launch_wide_dc<1>(a, s);
  if (a.d == 2) return launch_wide_dc<2>(a, s);
  return launch_wide_dc<4>(a, s);
}

cudaError_t big_solve_level(const BigCtx& c, int mode, int Jmax, int n, int d, const double* rhs, const double* Linv,
                            const double* Lsub, double* x, const double* xsep, double* fl, double* fr, double* Tws,
                            double* Uws) {
  using namespace btd;
  const long long nn = (long long)n * n, ps = (long long)n * d;
  const Operand oT = opnd(Tws, ps, d, kIdxSeg), oU = opnd(Uws, ps, d, kIdxSeg);
  const Operand oX0 = opnd(x, ps, d, kIdxSegRow), oXm1 = opnd(x, ps, d, kIdxSegRow, -1), oXp1 = opnd(x, ps, d, kIdxSegRow, 1);
  const Operand oR0 = opnd(rhs, ps, d, kIdxSegRow);
  cudaError_t e;
  // forward: z_j = Linv_j (b_j - L_{j,j-1} z_{j-1})
  for (int j = 0; j < Jmax; ++j) {
    if (j == 0)
      BIG_CHECK(big_copy(c, 0, kActAll, oR0, oT, n, d));
    else
      BIG_CHECK(big_gemm(c, j, kActAll, opnd(Lsub, nn, n, kIdxSegRow, -1), oXm1, oR0, oT, n, d, n, -1.0, 1.0));
    BIG_CHECK(big_gemm(c, j, kActAll, opnd(Linv, nn, n, kIdxSegRow), oT, oX0, oX0, n, d, n, 1.0, 0.0, 0, 2));
  }
  // backward: w_j = Linv_j^T (z_j - L_{j+1,j}^T w_{j+1})
  const Operand oLinvT = opnd(Linv, nn, n, kIdxSegRow, 0, 0, 1);
  for (int j = Jmax - 1; j >= 0; --j) {
    // last row of the segment: w = Linv^T z
    BIG_CHECK(big_gemm(c, j, kActLast, oLinvT, oX0, oU, oU, n, d, n, 1.0, 0.0, 0, 3));
    if (mode != kSolveDown) BIG_CHECK(big_copy(c, j, kActLast, oU, oX0, n, d));
    if (mode == kSolveDown)  // f_R = C_R w_last
      BIG_CHECK(big_gemm(c, j, kActLast, opnd(Lsub, nn, n, kIdxSegStop, -1), oU, opnd(fr, ps, d, kIdxSeg),
                         opnd(fr, ps, d, kIdxSeg), n, d, n, 1.0, 0.0));
    // other rows: t = z_j - L_{j+1,j}^T w_{j+1} ; w_j = Linv_j^T t
    const Operand oW1 = mode == kSolveDown ? oU : oXp1;
    BIG_CHECK(big_gemm(c, j, kActNotLast, opnd(Lsub, nn, n, kIdxSegRow, 0, 0, 1), oW1, oX0, oT, n, d, n, -1.0, 1.0));
    BIG_CHECK(big_gemm(c, j, kActNotLast, oLinvT, oT, mode == kSolveDown ? oU : oX0, mode == kSolveDown ? oU : oX0, n,
                       d, n, 1.0, 0.0, 0, 3));
  }
  if (mode == kSolveDown)  // f_L = C_L^T w_0
    BIG_CHECK(big_gemm(c, 0, kActAll, opnd(Lsub, nn, n, kIdxSegStart, 0, 0, 1), oU, opnd(fl, ps, d, kIdxSeg),
                       opnd(fl, ps, d, kIdxSeg), n, d, n, 1.0, 0.0));
  return cudaSuccess;
#undef BIG_CHECK
}

// reduced level-(L+1) system of a partial (sharded) hierarchy -> caller buffers
cudaError_t export_reduced(const btd_hierarchy* h, const double* cd, const double* cs, double* red_diag,
                           double* red_sub, cudaStream_t stream) {
  const size_t bb = (size_t)h->n * h->n * sizeof(double);
  cudaError_t e = cudaMemcpyAsync(red_diag, cd, (size_t)h->base_N * bb, cudaMemcpyDeviceToDevice, stream);
  if (e == cudaSuccess && h->base_N > 1)
    e = cudaMemcpyAsync(red_sub, cs, (size_t)(h->base_N - 1) * bb, cudaMemcpyDeviceToDevice, stream);
  return e;
}

}  // namespace

namespace {

// ---------------------------------------------------------------------------------------------
// CUDA graphs: the whole launch sequence of a factorization (every level, the assemblies and the
// base) or of a solve is captured once per (shape, config, buffer addresses) and replayed with
// one cudaGraphLaunch.  torch's caching allocator hands the same addresses back to repeated
// factorizations of the same shape, so steady-state calls hit the cache.  BTD_GRAPHS=0 disables.
// ---------------------------------------------------------------------------------------------
struct GraphKey {  // all 8-byte fields: no padding, so memcmp ordering is well defined
  int64_t kind;  // 0 factor, 1 + phase: solve
  int64_t N, n, crossover, rho, max_levels, auto_cross, nlevels, extra;
  const void* ptr[7];
  int64_t device = 0;
  bool operator<(const GraphKey& o) const {
    return std::memcmp(this, &o, sizeof(GraphKey)) < 0;
  }
};
struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  long long launches = 0;
  unsigned long long last_use = 0;
};
std::mutex g_graph_mu;
std::map<GraphKey, GraphEntry> g_graphs;
unsigned long long g_graph_clock = 0;
std::atomic<long long> g_graph_replays{0};  // graph launches served from the cache (btd_graph_replays)
constexpr size_t kMaxGraphs = 32;

std::atomic<int> g_graphs_on{-1};  // -1: not read from BTD_GRAPHS yet

bool graphs_enabled() {
  int v = g_graphs_on.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* ev = getenv("BTD_GRAPHS");
    v = (ev && ev[0] == '0') ? 0 : 1;
    g_graphs_on.store(v, std::memory_order_relaxed);
  }
  return v == 1;
}

// The launch sequence is recorded on a private capture stream (the caller's stream may be the
// legacy default stream, which cannot be captured -- torch's default) and the instantiated graph is
// launched into the caller's stream, so stream order is what the caller sees either way.
template <class F>
int run_graphed(GraphKey key, cudaStream_t stream, btd_status* st, F&& enqueue) {
  if (!graphs_enabled()) return enqueue(stream);
  int dev = 0;
  cudaGetDevice(&dev);
  key.device = dev;
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    auto it = g_graphs.find(key);
    if (it != g_graphs.end()) {
      it->second.last_use = ++g_graph_clock;
      cudaError_t e = cudaGraphLaunch(it->second.exec, stream);
      if (e != cudaSuccess) return cuda_fail(st, e, "cudaGraphLaunch");
      g_launches.fetch_add(it->second.launches, std::memory_order_relaxed);
      g_graph_replays.fetch_add(1, std::memory_order_relaxed);
      return BTD_OK;
    }
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (stream && (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)) {
    cudaGetLastError();
    return enqueue(stream);  // the caller is capturing already: just record into its graph
  }
  cudaStream_t cap = nullptr;
  if (cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    return enqueue(stream);
  }
  const long long before = g_launches.load();
  if (cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    cudaStreamDestroy(cap);
    return enqueue(stream);
  }
  const int rc = enqueue(cap);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(cap, &graph);
  cudaStreamDestroy(cap);
  const long long launches = g_launches.load() - before;
  g_launches.fetch_sub(launches, std::memory_order_relaxed);  // counted when the graph runs
  if (rc != BTD_OK || e != cudaSuccess || !graph) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    clear_status(st);
    return enqueue(stream);  // nothing ran during the failed capture: run the sequence directly
  }
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return enqueue(stream);
  }
  e = cudaGraphLaunch(exec, stream);
  if (e != cudaSuccess) {
    cudaGraphExecDestroy(exec);
    return cuda_fail(st, e, "cudaGraphLaunch");
  }
  g_launches.fetch_add(launches, std::memory_order_relaxed);
  std::lock_guard<std::mutex> lk(g_graph_mu);
  if (g_graphs.size() >= kMaxGraphs) {  // evict the least recently used graph
    auto lru = g_graphs.begin();
    for (auto it = g_graphs.begin(); it != g_graphs.end(); ++it)
      if (it->second.last_use < lru->second.last_use) lru = it;
    cudaGraphExecDestroy(lru->second.exec);
    g_graphs.erase(lru);
  }
  GraphEntry& ent = g_graphs[key];
  if (ent.exec) cudaGraphExecDestroy(ent.exec);  // another thread captured the same key meanwhile
  ent.exec = exec;
  ent.launches = launches;
  ent.last_use = ++g_graph_clock;
  return BTD_OK;
}

}  // namespace

extern "C" {

const char* btd_version(void) { return "blocktri_b200 0.1.0 (sm_100a)"; }

void btd_default_config(btd_config* cfg) {
  if (!cfg) return;
  cfg->crossover = 64;
  cfg->segment_length = 8;
  cfg->max_levels = 32;
  cfg->auto_crossover = 0;
  cfg->reserved = 0;
}

int btd_plan_separators(int64_t num_blocks, const btd_config* cfg, int64_t* separators_out, int64_t* count_out,
                        btd_status* st) {
  clear_status(st);
  if (!config_ok(cfg)) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "crossover, segment_length and max_levels must be >= 1");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  if (num_blocks < 3) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "cannot partition fewer than 3 block rows, got %lld",
               (long long)num_blocks);
    return BTD_ERR_INVALID_ARGUMENT;
  }
  std::vector<int64_t> s = plan_separators(num_blocks, cfg->segment_length);
  if (count_out) *count_out = (int64_t)s.size();
  if (separators_out) std::copy(s.begin(), s.end(), separators_out);
  return BTD_OK;
}

static int create_impl(int64_t num_blocks, int64_t block_size, const btd_config* cfg, int64_t forced_levels,
                       btd_hierarchy** out, btd_status* st) {
  clear_status(st);
  if (!out) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "out is NULL");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  *out = nullptr;
  if (!config_ok(cfg)) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "crossover, segment_length and max_levels must be >= 1");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  if (num_blocks < 1 || block_size < 1) {
    set_status(st, BTD_ERR_DIMENSION_MISMATCH, "need num_blocks >= 1 and block_size >= 1, got (%lld, %lld)",
               (long long)num_blocks, (long long)block_size);
    return BTD_ERR_DIMENSION_MISMATCH;
  }
  if (num_blocks >= (int64_t)INT_MAX) {
    set_status(st, BTD_ERR_UNSUPPORTED, "num_blocks must be < 2^31");
    return BTD_ERR_UNSUPPORTED;
  }
  const int nt = pick_nt(block_size);
  const bool big = !nt && block_size % 64 == 0 && block_size <= 1024;
  if (!nt && !big) {
    set_status(st, BTD_ERR_UNSUPPORTED,
               "block size %lld has no sm_100a kernel in this build (n <= 64, or a multiple of 64 up to 1024)",
               (long long)block_size);
    return BTD_ERR_UNSUPPORTED;
  }
  btd_hierarchy* h = new (std::nothrow) btd_hierarchy();
  if (!h) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "out of host memory");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  h->N = num_blocks;
  h->n = block_size;
  h->cfg = *cfg;
  h->nt = nt;
  h->big = big;
  const size_t bb = (size_t)block_size * block_size * sizeof(double);
  const size_t pb = big ? bb : (size_t)btd::packed_stride((int)block_size) * sizeof(double);

  // ---- recursion plan (recursive_factorize level loop, bt/schur.py:298-318) ----
  int64_t cur = num_blocks;
  h->partial = forced_levels >= 0;
  while (true) {
    if (h->partial) {
      if ((int64_t)h->levels.size() == forced_levels) break;
      if (cur < 3) {
        delete h;
        set_status(st, BTD_ERR_INVALID_ARGUMENT, "chunk too short for %lld local levels", (long long)forced_levels);
        return BTD_ERR_INVALID_ARGUMENT;
      }
    } else {
      if (!should_recurse(cur, *cfg)) break;
      if ((int64_t)h->levels.size() >= cfg->max_levels) {
        h->overflow = true;
        break;
      }
    }
    LevelPlan lp;
    lp.N = cur;
    lp.step = cfg->segment_length + 1;
    {  // separator count of plan_partition without materialising the list (bt/schur.py:75-95)
      int64_t P0 = (cur + lp.step - 1) / lp.step;  // 0, step, 2 step, ... < cur
      const int64_t last = (P0 - 1) * lp.step;
      if (last != cur - 1) {
        if (last == cur - 2) --P0;
        ++P0;
      }
      lp.P = P0;
    }
    lp.K = lp.P - 1;
    const int64_t maxlen = lp.max_segment();
    if (maxlen > btd::kMaxBlockCoord) {
      delete h;
      set_status(st, BTD_ERR_UNSUPPORTED, "segment length %lld exceeds the device error-coordinate range",
                 (long long)maxlen);
      return BTD_ERR_UNSUPPORTED;
    }
    h->levels.push_back(std::move(lp));
    cur = h->levels.back().P;
  }
  h->base_N = cur;

  // ---- persistent layout: error word, per level seps/Linv/Lsub, base Linv/Lsub ----
  size_t off = 0;
  h->off_err = off;
  off = align_up(off + sizeof(btd::DevErr));
  for (auto& lp : h->levels) {
    lp.off_seps = off;
    off = align_up(off + (size_t)lp.P * sizeof(int));
    lp.off_linv = off;
    off = align_up(off + (size_t)lp.N * pb);
    lp.off_lsub = off;
    off = align_up(off + (size_t)(lp.N - 1) * bb);
  }
  if (!h->overflow && !h->partial) {
    h->off_base_linv = off;
    off = align_up(off + (size_t)h->base_N * pb);
    h->off_base_lsub = off;
    off = align_up(off + (size_t)std::max<int64_t>(h->base_N - 1, 1) * bb);
  }
  h->persistent_bytes = off;

  // ---- factor scratch: per level, the next level's matrix and the S_R scratch ----
  size_t so = 0;
  for (auto& lp : h->levels) {
    lp.off_next_diag = so;
    so = align_up(so + (size_t)lp.P * bb);
    lp.off_next_sub = so;
    so = align_up(so + (size_t)(lp.P - 1) * bb);
    lp.off_sr = so;
    so = align_up(so + (size_t)lp.K * bb);
    h->kmax = std::max<int64_t>(h->kmax, lp.K);
  }
  if (big) {
    h->off_big_ws = so;
    so = align_up(so + (size_t)h->kmax * 5 * bb);
    h->off_splitk = so;  // split-k partials of the base's n x n products (8 splits)
    so = align_up(so + (size_t)8 * bb);
  }
  h->scratch_bytes = std::max<size_t>(so, kAlign);
  *out = h;
  return BTD_OK;
}

int btd_create(int64_t num_blocks, int64_t block_size, const btd_config* cfg, btd_hierarchy** out, btd_status* st) {
  return create_impl(num_blocks, block_size, cfg, -1, out, st);
}

int btd_create_partial(int64_t num_blocks, int64_t block_size, const btd_config* cfg, int64_t local_levels,
                       btd_hierarchy** out, btd_status* st) {
  if (local_levels < 1) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "local_levels must be >= 1");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  return create_impl(num_blocks, block_size, cfg, local_levels, out, st);
}

void btd_destroy(btd_hierarchy* h) { delete h; }

int btd_num_levels(const btd_hierarchy* h, int64_t* num_levels, int64_t* base_blocks, int32_t* overflow) {
  if (!h) return BTD_ERR_INVALID_ARGUMENT;
  if (num_levels) *num_levels = (int64_t)h->levels.size();
  if (base_blocks) *base_blocks = h->base_N;
  if (overflow) *overflow = h->overflow ? 1 : 0;
  return BTD_OK;
}

int btd_level_info(const btd_hierarchy* h, int64_t level, int64_t* num_blocks, int64_t* num_separators,
                   int64_t* separators_out) {
  if (!h || level < 0 || level >= (int64_t)h->levels.size()) return BTD_ERR_INVALID_ARGUMENT;
  const LevelPlan& lp = h->levels[level];
  if (num_blocks) *num_blocks = lp.N;
  if (num_separators) *num_separators = lp.P;
  if (separators_out)
    for (int64_t k = 0; k < lp.P; ++k) separators_out[k] = lp.sep(k);
  return BTD_OK;
}

int btd_factor_workspace(const btd_hierarchy* h, size_t* persistent_bytes, size_t* scratch_bytes) {
  if (!h) return BTD_ERR_INVALID_ARGUMENT;
  if (persistent_bytes) *persistent_bytes = h->persistent_bytes;
  if (scratch_bytes) *scratch_bytes = h->scratch_bytes;
  return BTD_OK;
}

struct HostSrc {
  const double* diag;
  const double* sub;
  double* dev_diag;
  double* dev_sub;
};

// H2D of diagonal blocks [b0, b0 + nb) from pinned host memory.  Every kernel reads only the lower
// triangle of a diagonal block (potrf, the D / S_L updates and the Schur assembly), so for n >= 32
// the rows are sent in G bands: band g (rows [g n/G, (g+1) n/G)) only its first (g+1) n/G columns,
// the last band in full (G = 4 for n >= 64: 5/8 of the bytes; G = 2 for n >= 32: 3/4), one pitched
// 3D copy per band with rows of >= 128 bytes.  The device copy's remaining upper triangle is never
// read.
cudaError_t copy_diag_h2d(double* dev, const double* host, int64_t b0, int64_t nb, int64_t n, cudaStream_t s) {
  const size_t nn = (size_t)n * n;
  if (nb <= 0) return cudaSuccess;
  int G = n >= 64 ? 4 : n >= 32 ? 2 : 1;
  while (G > 1 && n % G) --G;
  if (G <= 1)
    return cudaMemcpyAsync(dev + b0 * nn, host + b0 * nn, (size_t)nb * nn * sizeof(double), cudaMemcpyHostToDevice, s);
  const size_t pitch = (size_t)n * sizeof(double);
  const int64_t band = n / G;
  for (int g = 0; g < G; ++g) {
    cudaMemcpy3DParms p{};
    p.srcPtr = make_cudaPitchedPtr(const_cast<double*>(host), pitch, (size_t)n, (size_t)n);
    p.dstPtr = make_cudaPitchedPtr(dev, pitch, (size_t)n, (size_t)n);
    p.srcPos = make_cudaPos(0, (size_t)(g * band), (size_t)b0);
    p.dstPos = p.srcPos;
    p.extent = make_cudaExtent((size_t)((g + 1) * band) * sizeof(double), (size_t)band, (size_t)nb);
    p.kind = cudaMemcpyHostToDevice;
    cudaError_t e = cudaMemcpy3DAsync(&p, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t chunked_level0(btd_hierarchy* h, btd::FactorArgs a, const LevelPlan& lp, const HostSrc& src,
                           cudaStream_t stream) {
  if (!h->copy_stream) {
    cudaError_t e = cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
  }
  const size_t nn = (size_t)h->n * h->n;
  const int64_t K = lp.K;
  // chunks of >= ~64 MB: below that the per-chunk copy/event/launch overhead outweighs the overlap
  const int64_t bytes = (2 * lp.N - 1) * (int64_t)nn * (int64_t)sizeof(double);
  const int64_t chunks = std::max<int64_t>(1, std::min<int64_t>({K, (int64_t)16, bytes >> 26}));
  // the copy stream must not overwrite buffers a previous factorization on `stream` still reads
  cudaEvent_t ready;
  cudaError_t e = cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
  if (e != cudaSuccess) return e;
  cudaEventRecord(ready, stream);
  cudaStreamWaitEvent(h->copy_stream, ready, 0);
  cudaEventDestroy(ready);
  int64_t row0 = 0;
  for (int64_t c = 0; c < chunks; ++c) {
    const int64_t ka = K * c / chunks, kb = K * (c + 1) / chunks;
    // segments [ka, kb) read diag/sub rows up to seps[kb] (exclusive for sub, inclusive for the
    // separator diag read by the assembly); the last chunk takes everything that is left
    const int64_t row1 = (c + 1 == chunks) ? lp.N : lp.sep(kb) + 1;
    e = copy_diag_h2d(src.dev_diag, src.diag, row0, row1 - row0, h->n, h->copy_stream);
    const int64_t srow1 = std::min<int64_t>(row1, lp.N - 1);
    if (e == cudaSuccess && srow1 > row0)
      e = cudaMemcpyAsync(src.dev_sub + row0 * nn, src.sub + row0 * nn, (size_t)(srow1 - row0) * nn * sizeof(double),
                          cudaMemcpyHostToDevice, h->copy_stream);
    if (e != cudaSuccess) return e;
    cudaEvent_t ev;
    e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    cudaEventRecord(ev, h->copy_stream);
    cudaStreamWaitEvent(stream, ev, 0);
    cudaEventDestroy(ev);
    btd::FactorArgs ac = a;
    ac.k0 = (int)ka;
    ac.kend = (int)kb;
    if (kb > ka) {
      e = dispatch_factor(h->nt, ac, (unsigned)(kb - ka), stream);
      if (e != cudaSuccess) return e;
    }
    row0 = row1;
  }
  return cudaSuccess;
}

// Host-resident input (btd_factorize_from_host): the level-0 blocks are copied in chunks of whole
// segments on a private copy stream, and each chunk's segments are factored as soon as their
// blocks have landed, so the H2D transfer overlaps the level-0 elimination.

// Every device operation of one factorization, enqueued on `stream` (captured into a CUDA graph by
// factorize_impl when the inputs are device resident).  Host state is not touched here.
static int enqueue_factor(btd_hierarchy* h, const double* diag, const double* sub, char* pers, char* scr,
                          cudaStream_t stream, btd_status* st, double* red_diag, double* red_sub,
                          const HostSrc* host) {
  const int n = (int)h->n;
  btd::DevErr* err = (btd::DevErr*)(pers + h->off_err);
  btd::init_err_kernel<<<1, 1, 0, stream>>>(err); g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(st, e, "btd_factorize(init)");

  // separators of every level, generated on the device from the regular plan (no host sync):
  // s_k = k (rho+1) for k < P-1 and s_{P-1} = N-1 (equivalent to plan_partition, bt/schur.py:75-95).
  for (auto& lp : h->levels) {
    const unsigned blocks = (unsigned)((lp.P + 255) / 256);
    btd::fill_separators_kernel<<<blocks, 256, 0, stream>>>((int*)(pers + lp.off_seps), (int)lp.P, (int)lp.N,
                                                            (int)(h->cfg.segment_length + 1)); g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(st, e, "btd_factorize(seps)");

  // n > 64 with a split level 0: each half's rows are copied on the copy stream and the half's
  // launch sequence starts as soon as they have landed (half A computes while half B copies)
  const bool big_overlap = host && h->big && !h->levels.empty() && big_split_level(h->levels[0].K);
  if (big_overlap) {
    const LevelPlan& lp = h->levels[0];
    const size_t nn = (size_t)h->n * h->n;
    e = ensure_aux(h);
    if (e == cudaSuccess && !h->copy_stream) e = cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i)
      if (!h->ev_half[i]) e = cudaEventCreateWithFlags(&h->ev_half[i], cudaEventDisableTiming);
    // the copy stream must not overwrite buffers earlier work on `stream` still reads
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_fork, stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->copy_stream, h->ev_fork, 0);
    const int64_t rows[3] = {0, lp.sep(lp.K / 2) + 1, h->N};
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
      e = copy_diag_h2d(host->dev_diag, host->diag, rows[i], rows[i + 1] - rows[i], h->n, h->copy_stream);
      const int64_t s1 = std::min<int64_t>(rows[i + 1], h->N - 1);
      if (e == cudaSuccess && s1 > rows[i])
        e = cudaMemcpyAsync(host->dev_sub + rows[i] * nn, host->sub + rows[i] * nn, (size_t)(s1 - rows[i]) * nn * sizeof(double),
                            cudaMemcpyHostToDevice, h->copy_stream);
      if (e == cudaSuccess) e = cudaEventRecord(h->ev_half[i], h->copy_stream);
    }
    if (e != cudaSuccess) return cuda_fail(st, e, "btd_factorize_from_host(copy)");
    host = nullptr;
  } else if (host && (h->big || h->levels.empty())) {  // no chunking: one bulk copy, then the usual path
    const size_t nn = (size_t)h->n * h->n * sizeof(double);
    e = copy_diag_h2d(host->dev_diag, host->diag, 0, h->N, h->n, stream);
    if (e == cudaSuccess && h->N > 1)
      e = cudaMemcpyAsync(host->dev_sub, host->sub, (size_t)(h->N - 1) * nn, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return cuda_fail(st, e, "btd_factorize_from_host(copy)");
    host = nullptr;
  }
  const double* cd = diag;
  const double* cs = sub;
  if (h->big) {
    for (size_t l = 0; l < h->levels.size(); ++l) {
      LevelPlan& lp = h->levels[l];
      int jmax = 0;
      jmax = (int)lp.max_segment();
      BigCtx c{(const int*)(pers + lp.off_seps), lp.N, 0, (int)lp.K, err, stream};
      c.level = (int)l;
      set_lengths(c, lp);
      double* next_diag = (double*)(scr + lp.off_next_diag);
      prof_mark(h, stream);
      auto level_seq = [&](const BigCtx& cc) {
        return big_factor_level(cc, (int)l, jmax, n, cd, cs, (double*)(pers + lp.off_linv),
                                (double*)(pers + lp.off_lsub), next_diag, (double*)(scr + lp.off_sr),
                                (double*)(scr + lp.off_next_sub), scr + h->off_big_ws, err);
      };
      if (big_split_level(lp.K)) {
        e = ensure_aux(h);
        if (e == cudaSuccess) e = cudaEventRecord(h->ev_fork, stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(h->aux_stream, h->ev_fork, 0);
        if (l == 0 && big_overlap) {  // each half waits for its own rows only
          if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, h->ev_half[0], 0);
          if (e == cudaSuccess) e = cudaStreamWaitEvent(h->aux_stream, h->ev_half[1], 0);
        }
        BigCtx ca = c, cb = c;
        ca.Kws = cb.Kws = (int)lp.K;
        ca.K = (int)(lp.K / 2);
        cb.k0 = ca.K;
        cb.K = (int)lp.K - ca.K;
        cb.s = h->aux_stream;
        if (e == cudaSuccess) e = level_seq(ca);
        if (e == cudaSuccess) e = level_seq(cb);
        if (e == cudaSuccess) e = cudaEventRecord(h->ev_join, h->aux_stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, h->ev_join, 0);
      } else {
        e = level_seq(c);
      }
      prof_mark(h, stream);
      if (e != cudaSuccess) return cuda_fail(st, e, "btd_factorize(big level)");
      launch_assemble(cd, (const int*)(pers + lp.off_seps), next_diag, (const double*)(scr + lp.off_sr), (int)lp.K, n,
                      err, stream);
      e = cudaGetLastError();
      if (e != cudaSuccess) return cuda_fail(st, e, "btd_factorize(assemble)");
      cd = next_diag;
      cs = (const double*)(scr + lp.off_next_sub);
    }
    if (h->partial) {
      e = export_reduced(h, cd, cs, red_diag, red_sub, stream);
      if (e != cudaSuccess) return cuda_fail(st, e, "btd_factorize_partial(export)");
    } else if (!h->overflow) {
      BigCtx c{nullptr, h->base_N, 1, 1, err, stream};
      c.level = (int)h->levels.size();
      c.jreg = c.jtail = (int)h->base_N;
      c.part = (double*)(scr + h->off_splitk);
      c.part_doubles = (size_t)8 * h->n * h->n;
      prof_mark(h, stream);
      e = big_factor_level(c, (int)h->levels.size(), (int)h->base_N, n, cd, cs, (double*)(pers + h->off_base_linv),
                           (double*)(pers + h->off_base_lsub), nullptr, nullptr, nullptr, scr + h->off_big_ws, err);
      prof_mark(h, stream);
      if (e != cudaSuccess) return cuda_fail(st, e, "btd_factorize(big base)");
    }
    return BTD_OK;
  }
  for (size_t l = 0; l < h->levels.size(); ++l) {
    LevelPlan& lp = h->levels[l];
    btd::FactorArgs a{};
    a.diag = cd;
    a.sub = cs;
    a.seps = (const int*)(pers + lp.off_seps);
    a.N = lp.N;
    a.n = n;
    a.K = (int)lp.K;
    a.base = 0;
    a.level = (int)l;
    a.Linv = (double*)(pers + lp.off_linv);
    a.Lsub = (double*)(pers + lp.off_lsub);
    a.Sl = (double*)(scr + lp.off_next_diag);
    a.Sr = (double*)(scr + lp.off_sr);
    a.Ssub = (double*)(scr + lp.off_next_sub);
    a.err = err;
    if (l == 0 && host) {
      prof_mark(h, stream);
      e = chunked_level0(h, a, lp, *host, stream);
      prof_mark(h, stream);
      if (e != cudaSuccess) return cuda_fail(st, e, "btd_factorize_from_host(level 0)");
    } else {
      prof_mark(h, stream);
      e = dispatch_factor(h->nt, a, (unsigned)lp.K, stream);
      prof_mark(h, stream);
      if (e != cudaSuccess) return cuda_fail(st, e, "btd_factorize(level kernel)");
    }
    launch_assemble(cd, a.seps, a.Sl, a.Sr, (int)lp.K, n, err, stream);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(st, e, "btd_factorize(assemble)");
    cd = a.Sl;
    cs = a.Ssub;
  }
  if (h->partial) {
    e = export_reduced(h, cd, cs, red_diag, red_sub, stream);
    if (e != cudaSuccess) return cuda_fail(st, e, "btd_factorize_partial(export)");
  } else if (!h->overflow) {
    btd::FactorArgs a{};
    a.diag = cd;
    a.sub = cs;
    a.seps = nullptr;
    a.N = h->base_N;
    a.n = n;
    a.K = 1;
    a.base = 1;
    a.level = (int)h->levels.size();
    a.Linv = (double*)(pers + h->off_base_linv);
    a.Lsub = (double*)(pers + h->off_base_lsub);
    a.err = err;
    prof_mark(h, stream);
    e = dispatch_factor(h->nt, a, 1u, stream);
    prof_mark(h, stream);
    if (e != cudaSuccess) return cuda_fail(st, e, "btd_factorize(base kernel)");
  }
  return BTD_OK;
}

static int factorize_impl(btd_hierarchy* h, const double* diag, const double* sub, void* persistent, void* scratch,
                          void* stream_, int32_t check, btd_status* st, double* red_diag, double* red_sub,
                          const HostSrc* host = nullptr) {
  clear_status(st);
  if (!h || !diag || !persistent || !scratch || (h->N > 1 && !sub)) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "btd_factorize: NULL argument");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  cudaStream_t stream = (cudaStream_t)stream_;
  char* pers = (char*)persistent;
  char* scr = (char*)scratch;
  h->persistent = pers;
  h->factored = false;
  h->nev = 0;
  int rc;
  if (host || h->profile) {  // the host path uses a second stream; profiling records events
    rc = enqueue_factor(h, diag, sub, pers, scr, stream, st, red_diag, red_sub, host);
  } else {
    const GraphKey key{0, h->N, h->n, h->cfg.crossover, h->cfg.segment_length, h->cfg.max_levels,
                       h->cfg.auto_crossover, (int64_t)h->levels.size(), h->partial ? 1 : 0,
                       {diag, sub, pers, scr, red_diag, red_sub, nullptr}};
    rc = run_graphed(key, stream, st, [&](cudaStream_t sq) {
      return enqueue_factor(h, diag, sub, pers, scr, sq, st, red_diag, red_sub, nullptr);
    });
  }
  if (rc != BTD_OK) return rc;
  h->pending_check = true;
  if (check) return finish_check(h, stream, st);
  return BTD_OK;
}

int btd_factorize(btd_hierarchy* h, const double* diag, const double* sub, void* persistent, void* scratch,
                  void* stream, int32_t check, btd_status* st) {
  if (h && h->partial) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "partial hierarchy: use btd_factorize_partial");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  return factorize_impl(h, diag, sub, persistent, scratch, stream, check, st, nullptr, nullptr);
}

int btd_factorize_from_host(btd_hierarchy* h, const double* host_diag, const double* host_sub, double* dev_diag,
                            double* dev_sub, void* persistent, void* scratch, void* stream, int32_t check,
                            btd_status* st) {
  if (!h || h->partial || !host_diag || !dev_diag || (h->N > 1 && (!host_sub || !dev_sub))) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "btd_factorize_from_host: bad arguments");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  HostSrc src{host_diag, host_sub, dev_diag, dev_sub};
  return factorize_impl(h, dev_diag, dev_sub, persistent, scratch, stream, check, st, nullptr, nullptr, &src);
}

int btd_factorize_partial(btd_hierarchy* h, const double* diag, const double* sub, void* persistent, void* scratch,
                          double* reduced_diag, double* reduced_sub, void* stream, int32_t check, btd_status* st) {
  if (!h || !h->partial || !reduced_diag || !reduced_sub) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "btd_factorize_partial needs a partial hierarchy and output buffers");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  return factorize_impl(h, diag, sub, persistent, scratch, stream, check, st, reduced_diag, reduced_sub);
}

int btd_reduced_size(const btd_hierarchy* h, int64_t* num_blocks) {
  if (!h || !num_blocks) return BTD_ERR_INVALID_ARGUMENT;
  *num_blocks = h->base_N;
  return BTD_OK;
}

int btd_check(btd_hierarchy* h, void* stream, btd_status* st) {
  clear_status(st);
  if (!h || !h->persistent) {
    set_status(st, BTD_ERR_NOT_FACTORED, "hierarchy has not been factorized");
    return BTD_ERR_NOT_FACTORED;
  }
  return finish_check(h, (cudaStream_t)stream, st);
}

int btd_solve_workspace(const btd_hierarchy* h, int64_t d, size_t* scratch_bytes) {
  if (!h || d < 1) return BTD_ERR_INVALID_ARGUMENT;
  const size_t pb = (size_t)h->n * d * sizeof(double);
  size_t so = 0;
  for (const auto& lp : h->levels) {
    so = align_up(so + (size_t)lp.P * pb);  // next rhs
    so = align_up(so + (size_t)lp.P * pb);  // next x
    so = align_up(so + (size_t)lp.K * pb);  // f_R
  }
  if (h->big) {  // T, U panels per segment, the boundary-modified rhs of a level, split-k partials
    so = align_up(so + (size_t)h->kmax * pb);
    so = align_up(so + (size_t)h->kmax * pb);
    so = align_up(so + (size_t)h->N * pb);
    so = align_up(so + big_solve_part_doubles(h->n, d) * sizeof(double));
  }
  if (scratch_bytes) *scratch_bytes = std::max<size_t>(so, kAlign);
  return BTD_OK;
}

// Every device operation of one solve, enqueued on `stream` (captured into a CUDA graph by solve_impl).
static int enqueue_solve(const btd_hierarchy* h, const double* rhs, double* x, int64_t d, void* scratch,
                         cudaStream_t stream, btd_status* st, int phase, const double* red_in, double* red_out) {
  const char* pers = h->persistent;
  char* scr = (char*)scratch;
  const btd::DevErr* err = (const btd::DevErr*)(pers + h->off_err);
  const int n = (int)h->n;
  const size_t pb = (size_t)h->n * d * sizeof(double);
  const size_t L = h->levels.size();
  std::vector<double*> rhs_l(L + 1), x_l(L + 1), fr_l(L);
  rhs_l[0] = const_cast<double*>(rhs);
  x_l[0] = x;
  size_t so = 0;
  for (size_t l = 0; l < L; ++l) {
    const LevelPlan& lp = h->levels[l];
    rhs_l[l + 1] = (double*)(scr + so);
    so = align_up(so + (size_t)lp.P * pb);
    x_l[l + 1] = (double*)(scr + so);
    so = align_up(so + (size_t)lp.P * pb);
    fr_l[l] = (double*)(scr + so);
    so = align_up(so + (size_t)lp.K * pb);
  }
  cudaError_t e;
  if (h->big) {
    double* Tws = (double*)(scr + so);
    so = align_up(so + (size_t)h->kmax * pb);
    double* Uws = (double*)(scr + so);
    so = align_up(so + (size_t)h->kmax * pb);
    double* rmod = (double*)(scr + so);
    so = align_up(so + (size_t)h->N * pb);
    double* part = (double*)(scr + so);  // split-k partials (serial base)
    const int dd = (int)d;
    for (size_t l = 0; l < L && phase != kPhaseUp; ++l) {
      const LevelPlan& lp = h->levels[l];
      int jmax = 0;
      jmax = (int)lp.max_segment();
      const int* sp = (const int*)(pers + lp.off_seps);
      BigCtx c{sp, lp.N, 0, (int)lp.K, err, stream};
      set_lengths(c, lp);
      if (use_wide_solve(n, dd, lp.K)) {
        btd::SolveArgs a{};
        a.rhs = rhs_l[l];
        a.Linv = (const double*)(pers + lp.off_linv);
        a.Lsub = (const double*)(pers + lp.off_lsub);
        a.seps = sp;
        a.x = x_l[l];
        a.fl = rhs_l[l + 1];
        a.fr = fr_l[l];
        a.N = lp.N;
        a.n = n;
        a.d = dd;
        a.K = (int)lp.K;
        a.mode = btd::kSolveDown;
        a.err = err;
        e = launch_wide(a, stream);
      } else {
        e = big_solve_level(c, btd::kSolveDown, jmax, n, dd, rhs_l[l], (const double*)(pers + lp.off_linv),
                            (const double*)(pers + lp.off_lsub), x_l[l], nullptr, rhs_l[l + 1], fr_l[l], Tws, Uws);
      }
      if (e != cudaSuccess) return cuda_fail(st, e, "btd_solve(big down)");
      btd::assemble_separator_rhs_kernel<<<flat_grid(lp.P * h->n * d), 256, 0, stream>>>(rhs_l[l], sp, rhs_l[l + 1], fr_l[l],
                                                                              (int)lp.K, n, dd, err); g_launches.fetch_add(1, std::memory_order_relaxed);
      e = cudaGetLastError();
      if (e != cudaSuccess) return cuda_fail(st, e, "btd_solve(assemble)");
    }
    if (phase == kPhaseDown) {
      e = cudaMemcpyAsync(red_out, rhs_l[L], (size_t)h->base_N * pb, cudaMemcpyDeviceToDevice, stream);
      return e == cudaSuccess ? BTD_OK : cuda_fail(st, e, "btd_solve_down(export)");
    }
    if (phase == kPhaseUp) {
      e = cudaMemcpyAsync(x_l[L], red_in, (size_t)h->base_N * pb, cudaMemcpyDeviceToDevice, stream);
      if (e != cudaSuccess) return cuda_fail(st, e, "btd_solve_up(import)");
    } else {
      BigCtx c{nullptr, h->base_N, 1, 1, err, stream};
      c.jreg = c.jtail = (int)h->base_N;
      c.part = part;
      c.part_doubles = big_solve_part_doubles(h->n, d);
      if (use_wide_solve(n, dd, 1)) {
        btd::SolveArgs a{};
        a.rhs = rhs_l[L];
        a.Linv = (const double*)(pers + h->off_base_linv);
        a.Lsub = (const double*)(pers + h->off_base_lsub);
        a.x = x_l[L];
        a.N = h->base_N;
        a.n = n;
        a.d = dd;
        a.K = 1;
        a.mode = btd::kSolveBase;
        a.err = err;
        e = launch_wide(a, stream);
      } else {
        e = big_solve_level(c, btd::kSolveBase, (int)h->base_N, n, dd, rhs_l[L], (const double*)(pers + h->off_base_linv),
                            (const double*)(pers + h->off_base_lsub), x_l[L], nullptr, nullptr, nullptr, Tws, Uws);
      }
      if (e != cudaSuccess) return cuda_fail(st, e, "btd_solve(big base)");
    }
    for (size_t l = L; l-- > 0;) {
      const LevelPlan& lp = h->levels[l];
      int jmax = 0;
      jmax = (int)lp.max_segment();
      const int* sp = (const int*)(pers + lp.off_seps);
      BigCtx c{sp, lp.N, 0, (int)lp.K, err, stream};
      set_lengths(c, lp);
      if (use_wide_solve(n, dd, lp.K)) {
        btd::SolveArgs a{};
        a.rhs = rhs_l[l];
        a.Linv = (const double*)(pers + lp.off_linv);
        a.Lsub = (const double*)(pers + lp.off_lsub);
        a.seps = sp;
        a.xsep = x_l[l + 1];
        a.x = x_l[l];
        a.N = lp.N;
        a.n = n;
        a.d = dd;
        a.K = (int)lp.K;
        a.mode = btd::kSolveUp;
        a.err = err;
        e = launch_wide(a, stream);
        if (e != cudaSuccess) return cuda_fail(st, e, "btd_solve(wide up)");
        continue;
      }
      const long long nn = (long long)n * n, ps = (long long)n * dd;
      const double* Ls = (const double*)(pers + lp.off_lsub);
      // boundary-modified rhs: b_0 -= C_L x_L ; b_last -= C_R^T x_R
      e = cudaMemcpyAsync(rmod, rhs_l[l], (size_t)lp.N * pb, cudaMemcpyDeviceToDevice, stream);
      if (e != cudaSuccess) return cuda_fail(st, e, "btd_solve(big rmod)");
      const btd::Operand rm0 = opnd(rmod, ps, dd, btd::kIdxSegRow), rmL = opnd(rmod, ps, dd, btd::kIdxSegStop, -1);
      e = big_gemm(c, 0, btd::kActAll, opnd(Ls, nn, n, btd::kIdxSegStart), opnd(x_l[l + 1], ps, dd, btd::kIdxSeg), rm0,
                   rm0, n, dd, n, -1.0, 1.0);
      if (e == cudaSuccess)
        e = big_gemm(c, 0, btd::kActAll, opnd(Ls, nn, n, btd::kIdxSegStop, -1, 0, 1),
                     opnd(x_l[l + 1], ps, dd, btd::kIdxSeg, 1), rmL, rmL, n, dd, n, -1.0, 1.0);
      if (e == cudaSuccess)
        e = big_solve_level(c, btd::kSolveUp, jmax, n, dd, rmod, (const double*)(pers + lp.off_linv), Ls, x_l[l],
                            x_l[l + 1], nullptr, nullptr, Tws, Uws);
      // separator rows of the solution
      if (e == cudaSuccess)
        e = big_copy(c, 0, btd::kActAll, opnd(x_l[l + 1], ps, dd, btd::kIdxSeg), opnd(x_l[l], ps, dd, btd::kIdxSegStart),
                     n, dd);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(x_l[l] + (size_t)lp.sep(lp.K) * ps, x_l[l + 1] + (size_t)lp.K * ps, (size_t)pb,
                            cudaMemcpyDeviceToDevice, stream);
      if (e != cudaSuccess) return cuda_fail(st, e, "btd_solve(big up)");
    }
    return BTD_OK;
  }
  for (size_t l = 0; l < L && phase != kPhaseUp; ++l) {
    const LevelPlan& lp = h->levels[l];
    btd::SolveArgs a{};
    a.rhs = rhs_l[l];
    a.Linv = (const double*)(pers + lp.off_linv);
    a.Lsub = (const double*)(pers + lp.off_lsub);
    a.seps = (const int*)(pers + lp.off_seps);
    a.x = x_l[l];
    a.fl = rhs_l[l + 1];
    a.fr = fr_l[l];
    a.N = lp.N;
    a.n = n;
    a.d = (int)d;
    a.K = (int)lp.K;
    a.mode = btd::kSolveDown;
    a.err = err;
    e = use_small(h->nt) ? launch_solve_small(a, stream) : (n == h->nt) ? dispatch_stream(h->nt, a, stream) : dispatch_solve(h->nt, a, (unsigned)lp.K, stream);
    if (e != cudaSuccess) return cuda_fail(st, e, "btd_solve(down)");
    btd::assemble_separator_rhs_kernel<<<flat_grid(lp.P * h->n * d), 256, 0, stream>>>(rhs_l[l], a.seps, rhs_l[l + 1], fr_l[l],
                                                                            (int)lp.K, n, (int)d, err); g_launches.fetch_add(1, std::memory_order_relaxed);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(st, e, "btd_solve(assemble)");
  }
  if (phase == kPhaseDown) {
    e = cudaMemcpyAsync(red_out, rhs_l[L], (size_t)h->base_N * pb, cudaMemcpyDeviceToDevice, stream);
    return e == cudaSuccess ? BTD_OK : cuda_fail(st, e, "btd_solve_down(export)");
  }
  if (phase == kPhaseUp) {
    e = cudaMemcpyAsync(x_l[L], red_in, (size_t)h->base_N * pb, cudaMemcpyDeviceToDevice, stream);
    if (e != cudaSuccess) return cuda_fail(st, e, "btd_solve_up(import)");
  } else {
    btd::SolveArgs a{};
    a.rhs = rhs_l[L];
    a.Linv = (const double*)(pers + h->off_base_linv);
    a.Lsub = (const double*)(pers + h->off_base_lsub);
    a.x = x_l[L];
    a.N = h->base_N;
    a.n = n;
    a.d = (int)d;
    a.K = 1;
    a.mode = btd::kSolveBase;
    a.err = err;
    e = use_small(h->nt) ? launch_solve_small(a, stream) : (n == h->nt) ? dispatch_stream(h->nt, a, stream) : dispatch_solve(h->nt, a, 1u, stream);
    if (e != cudaSuccess) return cuda_fail(st, e, "btd_solve(base)");
  }
  for (size_t l = L; l-- > 0;) {
    const LevelPlan& lp = h->levels[l];
    btd::SolveArgs a{};
    a.rhs = rhs_l[l];
    a.Linv = (const double*)(pers + lp.off_linv);
    a.Lsub = (const double*)(pers + lp.off_lsub);
    a.seps = (const int*)(pers + lp.off_seps);
    a.xsep = x_l[l + 1];
    a.x = x_l[l];
    a.N = lp.N;
    a.n = n;
    a.d = (int)d;
    a.K = (int)lp.K;
    a.mode = btd::kSolveUp;
    a.err = err;
    e = use_small(h->nt) ? launch_solve_small(a, stream) : (n == h->nt) ? dispatch_stream(h->nt, a, stream) : dispatch_solve(h->nt, a, (unsigned)lp.K, stream);
    if (e != cudaSuccess) return cuda_fail(st, e, "btd_solve(up)");
  }
  return BTD_OK;
}

static int solve_impl(const btd_hierarchy* h, const double* rhs, double* x, int64_t d, void* scratch, void* stream_,
                      btd_status* st, int phase, const double* red_in, double* red_out) {
  clear_status(st);
  if (!h || !rhs || !x || !scratch || d < 1) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "btd_solve: NULL argument or d < 1");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  if (!h->factored && !h->pending_check) {
    set_status(st, BTD_ERR_NOT_FACTORED, "hierarchy must be factorized before solving");
    return BTD_ERR_NOT_FACTORED;
  }
  if (d > INT_MAX / 2) {
    set_status(st, BTD_ERR_UNSUPPORTED, "too many rhs columns");
    return BTD_ERR_UNSUPPORTED;
  }
  cudaStream_t stream = (cudaStream_t)stream_;
  const GraphKey key{1 + phase, h->N, h->n, h->cfg.crossover, h->cfg.segment_length, h->cfg.max_levels,
                     h->cfg.auto_crossover, (int64_t)h->levels.size(), d,
                     {h->persistent, rhs, x, scratch, red_in, red_out, (const void*)(intptr_t)h->partial}};
  return run_graphed(key, stream, st, [&](cudaStream_t sq) {
    return enqueue_solve(h, rhs, x, d, scratch, sq, st, phase, red_in, red_out);
  });
}

int btd_solve(const btd_hierarchy* h, const double* rhs, double* x, int64_t d, void* scratch, void* stream,
              btd_status* st) {
  if (h && h->partial) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "partial hierarchy: use btd_solve_down / btd_solve_up");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  return solve_impl(h, rhs, x, d, scratch, stream, st, kPhaseFull, nullptr, nullptr);
}

int btd_solve_down(const btd_hierarchy* h, const double* rhs, double* x, int64_t d, void* scratch,
                   double* reduced_rhs_out, void* stream, btd_status* st) {
  if (!h || !h->partial || !reduced_rhs_out) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "btd_solve_down needs a partial hierarchy and an output buffer");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  return solve_impl(h, rhs, x, d, scratch, stream, st, kPhaseDown, nullptr, reduced_rhs_out);
}

int btd_solve_up(const btd_hierarchy* h, const double* rhs, const double* reduced_x, double* x, int64_t d,
                 void* scratch, void* stream, btd_status* st) {
  if (!h || !h->partial || !reduced_x) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "btd_solve_up needs a partial hierarchy and the reduced solution");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  return solve_impl(h, rhs, x, d, scratch, stream, st, kPhaseUp, reduced_x, nullptr);
}

int btd_level_factor(const btd_hierarchy* h, int64_t level, double* linv_out, double* lsub_out, void* stream,
                     btd_status* st) {
  clear_status(st);
  if (!h || !h->persistent || level < 0 || level > (int64_t)h->levels.size()) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "btd_level_factor: bad level or unfactored hierarchy");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  const size_t bb = (size_t)h->n * h->n * sizeof(double);
  size_t ol, os;
  int64_t N;
  if (level == (int64_t)h->levels.size()) {
    ol = h->off_base_linv;
    os = h->off_base_lsub;
    N = h->base_N;
  } else {
    ol = h->levels[level].off_linv;
    os = h->levels[level].off_lsub;
    N = h->levels[level].N;
  }
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  const size_t pb = (size_t)btd::packed_stride((int)h->n) * sizeof(double);
  if (linv_out) e = cudaMemcpyAsync(linv_out, h->persistent + ol, (size_t)N * pb, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && lsub_out && N > 1)
    e = cudaMemcpyAsync(lsub_out, h->persistent + os, (size_t)(N - 1) * bb, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return cuda_fail(st, e, "btd_level_factor");
  return BTD_OK;
}

int btd_level_schur(const btd_hierarchy* h, int64_t level, const void* scratch, double* diag_out, double* sub_out,
                    void* stream, btd_status* st) {
  clear_status(st);
  if (!h || !scratch || !diag_out || level < 0 || level >= (int64_t)h->levels.size() || !h->factored) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "btd_level_schur: bad level, buffers or unfactored hierarchy");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  const LevelPlan& lp = h->levels[level];
  const size_t bb = (size_t)h->n * h->n * sizeof(double);
  const char* scr = (const char*)scratch;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(diag_out, scr + lp.off_next_diag, (size_t)lp.P * bb, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && lp.P > 1 && sub_out)
    e = cudaMemcpyAsync(sub_out, scr + lp.off_next_sub, (size_t)(lp.P - 1) * bb, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return cuda_fail(st, e, "btd_level_schur(copy)");
  btd::mirror_lower_kernel<<<flat_grid(lp.P * h->n * h->n), 256, 0, s>>>(diag_out, lp.P, (int)h->n);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(st, e, "btd_level_schur(mirror)");
  return BTD_OK;
}

#ifdef BTD_PHASE_PROF
int btd_debug_phase_cycles(unsigned long long* out16, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out16, btd::g_phase_cycles, 16 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(btd::g_phase_cycles, z, sizeof(z));
  }
  return 0;
}
#endif

int btd_profile_kernels(btd_hierarchy* h, int32_t enable) {
  if (!h) return BTD_ERR_INVALID_ARGUMENT;
  h->profile = enable != 0;
  return BTD_OK;
}

int btd_kernel_times(const btd_hierarchy* h, float* ms_out, int64_t cap, int64_t* count) {
  if (!h) return BTD_ERR_INVALID_ARGUMENT;
  const int64_t n = h->nev / 2;
  if (count) *count = n;
  for (int64_t i = 0; i < n && i < cap && ms_out; ++i) {
    cudaError_t e = cudaEventSynchronize(h->ev[2 * i + 1]);
    if (e != cudaSuccess) return BTD_ERR_CUDA;
    cudaEventElapsedTime(&ms_out[i], h->ev[2 * i], h->ev[2 * i + 1]);
  }
  return BTD_OK;
}

long long btd_graph_replays(void) { return g_graph_replays.load(std::memory_order_relaxed); }

int btd_set_graphs(int32_t enable) {
  const int prev = graphs_enabled() ? 1 : 0;
  g_graphs_on.store(enable ? 1 : 0, std::memory_order_relaxed);
  if (!enable) {  // drop the cached executables
    std::lock_guard<std::mutex> lk(g_graph_mu);
    for (auto& kv : g_graphs) cudaGraphExecDestroy(kv.second.exec);
    g_graphs.clear();
  }
  return prev;
}

long long btd_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

// ---------------------------------------------------------------------------------------------
// Block SpMV and fused residual norms (btd_spmv.cuh): btd_matmul bt/core.py:280-288,
// residual_report bt/report.py:20-38.
// ---------------------------------------------------------------------------------------------
static void spmv_grid(int64_t N, int64_t d, long long* rows_per_cta, unsigned* ctas, unsigned* ycols) {
  const int sms = device_sms();
  const long long want = std::min<long long>(N, (long long)sms * 8);
  *rows_per_cta = (N + want - 1) / want;
  *ctas = (unsigned)((N + *rows_per_cta - 1) / *rows_per_cta);
  *ycols = (unsigned)((d + btd::kSpmvMaxD - 1) / btd::kSpmvMaxD);
}

int btd_matmul(const double* diag, const double* sub, int64_t N, int64_t n, const double* x, int64_t d, double* y,
               void* stream, btd_status* st) {
  clear_status(st);
  if (N < 1 || n < 1 || d < 1 || !diag || !x || !y || (N > 1 && !sub)) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "btd_matmul: bad arguments");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  btd::SpmvArgs a{};
  a.diag = diag;
  a.sub = sub;
  a.x = x;
  a.y = y;
  a.N = N;
  a.n = (int)n;
  a.d = (int)d;
  unsigned ctas, ycols;
  spmv_grid(N, d, &a.rows_per_cta, &ctas, &ycols);
  btd::btd_spmv_kernel<<<dim3(ctas, ycols), btd::kSpmvThreads, 0, (cudaStream_t)stream>>>(a); g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(st, e, "btd_matmul");
  return BTD_OK;
}

int btd_residual_workspace(int64_t N, int64_t n, int64_t d, size_t* bytes) {
  (void)n;
  if (N < 1 || d < 1 || !bytes) return BTD_ERR_INVALID_ARGUMENT;
  long long rows;
  unsigned ctas, ycols;
  spmv_grid(N, d, &rows, &ctas, &ycols);
  *bytes = (size_t)ctas * 2 * (size_t)d * sizeof(double);
  return BTD_OK;
}

int btd_residual_norms(const double* diag, const double* sub, int64_t N, int64_t n, const double* x, const double* b,
                       int64_t d, void* workspace, double* norms2, void* stream, btd_status* st) {
  clear_status(st);
  if (N < 1 || n < 1 || d < 1 || !diag || !x || !b || !workspace || !norms2 || (N > 1 && !sub)) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "btd_residual_norms: bad arguments");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  btd::SpmvArgs a{};
  a.diag = diag;
  a.sub = sub;
  a.x = x;
  a.b = b;
  a.partial = (double*)workspace;
  a.N = N;
  a.n = (int)n;
  a.d = (int)d;
  unsigned ctas, ycols;
  spmv_grid(N, d, &a.rows_per_cta, &ctas, &ycols);
  cudaStream_t s = (cudaStream_t)stream;
  btd::btd_spmv_kernel<<<dim3(ctas, ycols), btd::kSpmvThreads, 0, s>>>(a); g_launches.fetch_add(1, std::memory_order_relaxed);
  btd::btd_norm_finish_kernel<<<(unsigned)((2 * d + 127) / 128), 128, 0, s>>>(a.partial, (int)ctas, (int)d, norms2); g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(st, e, "btd_residual_norms");
  return BTD_OK;
}

// ---------------------------------------------------------------------------------------------
// Kalman normal equations (btd_kalman.cuh): build_normal_equations, bt/kalman.py:130-162.
// ---------------------------------------------------------------------------------------------
int btd_kalman_workspace(int64_t horizon, int64_t state_dim, size_t* bytes) {
  if (horizon < 1 || state_dim < 1 || !bytes) return BTD_ERR_INVALID_ARGUMENT;
  *bytes = align_up((size_t)horizon * state_dim * state_dim * sizeof(double)) + kAlign;
  return BTD_OK;
}

int btd_kalman_normal_equations(int64_t horizon, int64_t n, int64_t m, const double* transition,
                                const double* observation, const double* process_cov, const double* meas_cov,
                                const double* observations, const double* prior_offsets, int32_t flags,
                                double* diag, double* sub, double* rhs, void* workspace, void* stream,
                                btd_status* st) {
  clear_status(st);
  const bool diag_r = flags & BTD_KALMAN_DIAG_R;
  if (horizon < 1 || n < 1 || m < 1 || !transition || !observation || !process_cov || !meas_cov ||
      !observations || !prior_offsets || !diag || !rhs || !workspace || (horizon > 1 && !sub)) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "btd_kalman_normal_equations: bad arguments");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  if (n > btd::kKalmanMaxN || (!diag_r && m > btd::kKalmanMaxDenseM)) {
    set_status(st, BTD_ERR_UNSUPPORTED, "Kalman assembly kernel: state_dim <= %d and (dense R) obs_dim <= %d",
               btd::kKalmanMaxN, btd::kKalmanMaxDenseM);
    return BTD_ERR_UNSUPPORTED;
  }
  cudaStream_t s = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  unsigned long long* err = (unsigned long long*)ws;
  double* cross = (double*)(ws + kAlign);
  btd::KalmanArgs a{};
  a.transition = transition;
  a.observation = observation;
  a.process_cov = process_cov;
  a.meas_cov = meas_cov;
  a.observations = observations;
  a.prior = prior_offsets;
  a.N = horizon;
  a.n = (int)n;
  a.m = (int)m;
  a.diag_r = diag_r ? 1 : 0;
  a.shared_h = (flags & BTD_KALMAN_SHARED_H) ? 1 : 0;
  a.shared_q = (flags & BTD_KALMAN_SHARED_Q) ? 1 : 0;
  a.shared_r = (flags & BTD_KALMAN_SHARED_R) ? 1 : 0;
  a.diag = diag;
  a.sub = sub;
  a.rhs = rhs;
  a.cross = cross;
  a.err = err;
  const size_t smem = btd::kalman_smem_doubles((int)n, (int)m, diag_r ? 0 : 1) * sizeof(double);
  cudaError_t e = ensure_smem((const void*)btd::kalman_terms_kernel, smem);
  if (e != cudaSuccess) return cuda_fail(st, e, "btd_kalman_normal_equations(attr)");
  e = cudaMemsetAsync(err, 0xff, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return cuda_fail(st, e, "btd_kalman_normal_equations(init)");
  btd::kalman_terms_kernel<<<(unsigned)horizon, btd::kKalmanThreads, smem, s>>>(a); g_launches.fetch_add(1, std::memory_order_relaxed);
  btd::kalman_finish_kernel<<<flat_grid(horizon * n * n), 256, 0, s>>>(diag, cross, horizon, (int)n, err); g_launches.fetch_add(1, std::memory_order_relaxed);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(st, e, "btd_kalman_normal_equations(launch)");
  unsigned long long key = 0;
  e = cudaMemcpyAsync(&key, err, sizeof(key), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(st, e, "btd_kalman_normal_equations(sync)");
  if (key != btd::kNoErr) {
    const long long k = (long long)(key >> 20);
    const int kind = (int)((key >> 16) & 0xf), pivot = (int)(key & 0xffff);
    set_status(st, BTD_ERR_NOT_POSITIVE_DEFINITE, "%s covariance is not positive definite at pivot %d, step %lld",
               kind == 0 ? "process" : "measurement", pivot, k);
    st->pivot = pivot;
    st->block = k;
    st->member = kind;  // 0: process covariance, 1: measurement covariance
    st->level = -1;
    return BTD_ERR_NOT_POSITIVE_DEFINITE;
  }
  return BTD_OK;
}

// ---------------------------------------------------------------------------------------------
// Accelerator seam (btd_seam.cuh): chol_factor_batch / trsm_lower_batch / gemm_acc_batch,
// bt/kernels.py:164-338.
// ---------------------------------------------------------------------------------------------
static btd::Strides to_strides(const int64_t* s) { return btd::Strides{(long long)s[0], (long long)s[1], (long long)s[2]}; }

size_t btd_seam_error_bytes(void) { return sizeof(btd::SeamErr); }

int btd_seam_error_init(void* err, void* stream) {
  if (!err) return BTD_ERR_INVALID_ARGUMENT;
  btd::seam_err_init_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((btd::SeamErr*)err);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError() == cudaSuccess ? BTD_OK : BTD_ERR_CUDA;
}

int btd_seam_error_read(const void* err, void* stream, btd_status* st) {
  clear_status(st);
  btd::SeamErr h;
  cudaError_t e = cudaMemcpyAsync(&h, err, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(st, e, "btd_seam_error_read");
  if (h.sing != btd::kNoErr) {
    const long long member = (long long)(h.sing >> 24);
    const int row = (int)(h.sing & 0xffffff);
    set_status(st, BTD_ERR_SINGULAR_DIAGONAL, "triangular factor has zero diagonal at row %d, member %lld", row + 1,
               member);
    st->pivot = row + 1;
    st->member = member;
    return BTD_ERR_SINGULAR_DIAGONAL;
  }
  if (h.npd != btd::kNoErr) {
    btd::DevErr de{h.npd, 0, 0};
    decode_error(de, st);
    st->level = -1;
    return BTD_ERR_NOT_POSITIVE_DEFINITE;
  }
  return BTD_OK;
}

int btd_chol_batch(double* blocks, const int64_t strides[3], int64_t count, int64_t n, int64_t block_coord, void* err,
                   void* stream, btd_status* st) {
  clear_status(st);
  if (!err || !strides || count < 0 || n < 1 || n > 0xffff || block_coord < 0 || block_coord > btd::kMaxBlockCoord ||
      count > btd::kMaxMemberCoord || (count > 0 && !blocks)) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "btd_chol_batch: bad arguments");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  if (count == 0) return BTD_OK;
  if (n <= btd::kSeamSmemMaxN) {
    const size_t smem = btd::seam_chol_smem((int)n);
    cudaError_t e = ensure_smem((const void*)btd::seam_chol_smem_kernel, smem);
    if (e != cudaSuccess) return cuda_fail(st, e, "btd_chol_batch(attr)");
    btd::seam_chol_smem_kernel<<<(unsigned)count, btd::kSeamThreads, smem, (cudaStream_t)stream>>>(
        blocks, to_strides(strides), (int)n, (long long)block_coord, (btd::SeamErr*)err);
  } else {
    btd::seam_chol_kernel<<<(unsigned)count, btd::kSeamThreads, 0, (cudaStream_t)stream>>>(
        blocks, to_strides(strides), (int)n, (long long)block_coord, (btd::SeamErr*)err);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BTD_OK : cuda_fail(st, e, "btd_chol_batch");
}

int btd_trsm_batch(const double* factors, const int64_t fstrides[3], double* panels, const int64_t pstrides[3],
                   int64_t count, int64_t n, int64_t cols, int32_t trans, void* err, void* stream, btd_status* st) {
  clear_status(st);
  if (!err || !fstrides || !pstrides || count < 0 || n < 1 || cols < 0 || count > (1ll << 39) || n > (1 << 24) ||
      (count > 0 && (!factors || !panels))) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "btd_trsm_batch: bad arguments");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  if (count == 0) return BTD_OK;
  cudaStream_t s = (cudaStream_t)stream;
  btd::seam_diag_check_kernel<<<(unsigned)count, 128, 0, s>>>(factors, to_strides(fstrides), (int)n, count,
                                                              (btd::SeamErr*)err);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (cols > 0 && n <= btd::kSeamSmemMaxN) {
    const size_t smem = btd::seam_trsm_smem((int)n);
    cudaError_t e = ensure_smem((const void*)btd::seam_trsm_dmma_kernel, smem);
    if (e != cudaSuccess) return cuda_fail(st, e, "btd_trsm_batch(attr)");
    dim3 grid((unsigned)count, (unsigned)((cols + btd::kStCols - 1) / btd::kStCols));
    btd::seam_trsm_dmma_kernel<<<grid, btd::kSeamThreads, smem, s>>>(factors, to_strides(fstrides), panels,
                                                                      to_strides(pstrides), (int)n, (int)cols, trans,
                                                                      (const btd::SeamErr*)err);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  } else if (cols > 0) {
    dim3 grid((unsigned)count, (unsigned)((cols + btd::kSeamThreads - 1) / btd::kSeamThreads));
    btd::seam_trsm_kernel<<<grid, btd::kSeamThreads, 0, s>>>(factors, to_strides(fstrides), panels,
                                                                 to_strides(pstrides), (int)n, (int)cols, trans,
                                                                 (const btd::SeamErr*)err);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BTD_OK : cuda_fail(st, e, "btd_trsm_batch");
}

int btd_gemm_batch(double* out, const int64_t ostrides[3], const double* a, const int64_t astrides[3], const double* b,
                   const int64_t bstrides[3], int64_t count, int64_t m, int64_t q, int64_t p, int32_t trans_a,
                   int32_t trans_b, double alpha, double beta, void* stream, btd_status* st) {
  clear_status(st);
  if (!ostrides || !astrides || !bstrides || count < 0 || m < 0 || q < 0 || p < 0 || count > 65535 ||
      (count > 0 && m > 0 && p > 0 && (!out || ((!a || !b) && q > 0)))) {
    set_status(st, BTD_ERR_INVALID_ARGUMENT, "btd_gemm_batch: bad arguments (at most 65535 members per call)");
    return BTD_ERR_INVALID_ARGUMENT;
  }
  if (count == 0 || m == 0 || p == 0) return BTD_OK;
  btd::Strides as = to_strides(astrides), bs = to_strides(bstrides);
  if (trans_a) std::swap(as.r, as.c);  // op(a)(r, k) = a(k, r)
  if (trans_b) std::swap(bs.r, bs.c);
  const int tiles_m = (int)((m + btd::kSgT - 1) / btd::kSgT), tiles_p = (int)((p + btd::kSgT - 1) / btd::kSgT);
  dim3 grid((unsigned)(tiles_m * tiles_p), (unsigned)count);
  btd::seam_gemm_kernel<<<grid, btd::kSeamThreads, 0, (cudaStream_t)stream>>>(
      out, to_strides(ostrides), a, as, b, bs, (int)m, (int)q, (int)p, tiles_p, alpha, beta);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BTD_OK : cuda_fail(st, e, "btd_gemm_batch");
}

}  // extern "C"
