// Does DFMA run concurrently with DMMA on sm_100a?  And the latency of the approximate fp64
// reciprocal / rsqrt (MUFU.RCP64H / MUFU.RSQ64H) used to shorten the Cholesky pivot chain.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
// mode 0: all warps DMMA; 1: all warps DFMA; 2: even warps DMMA, odd warps DFMA; 3: every warp both
__global__ void mix(double* out, int iters, int mode) {
  const int w = threadIdx.x >> 5;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2], f[16];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0.0;
#pragma unroll
  for (int t = 0; t < 16; ++t) f[t] = t;
  const bool do_mma = mode == 0 || mode == 3 || (mode == 2 && (w & 1) == 0);
  const bool do_fma = mode == 1 || mode == 3 || (mode == 2 && (w & 1) == 1);
  for (int i = 0; i < iters; ++i) {
    if (do_mma) {
#pragma unroll
      for (int t = 0; t < 8; ++t) dmma(c[t][0], c[t][1], a, b);
    }
    if (do_fma) {
#pragma unroll
      for (int t = 0; t < 16; ++t) f[t] = fma(a, f[t], b);
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
#pragma unroll
  for (int t = 0; t < 16; ++t) s += f[t];
  if (s == 12345.0) out[0] = s;
}

__device__ __forceinline__ double rcp_approx(double x) {
  double y;
  asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm volatile("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__global__ void lat(double* out, long long* cyc, double x0, int iters) {
  double x = x0 + threadIdx.x * 1e-20;
  long long t0, t1;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = rcp_approx(x) + 0.5;
  t1 = clock64(); cyc[0] = (t1 - t0) / iters;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = rsqrt_approx(x) + 0.5;
  t1 = clock64(); cyc[1] = (t1 - t0) / iters;
  // full-precision reciprocal: approx + 2 Newton steps
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double y = rcp_approx(x);
    double e = fma(-x, y, 1.0); y = fma(y, e, y);
    e = fma(-x, y, 1.0); y = fma(y, e, y);
    x = y + 0.5;
  }
  t1 = clock64(); cyc[2] = (t1 - t0) / iters;
  // __drcp_rn
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __drcp_rn(x) + 0.5;
  t1 = clock64(); cyc[3] = (t1 - t0) / iters;
  // shfl chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (i & 31)) + 1e-9;
  t1 = clock64(); cyc[4] = (t1 - t0) / iters;
  // rsqrt (libdevice)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = rsqrt(x) + 0.5;
  t1 = clock64(); cyc[5] = (t1 - t0) / iters;
  // lds chain
  __shared__ double sm[64];
  sm[threadIdx.x & 63] = 0.0;
  __syncwarp();
  int idx = 0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { double v = sm[idx]; idx = (int)v; x += v; }
  t1 = clock64(); cyc[6] = (t1 - t0) / iters;
  out[threadIdx.x] = x;
}

int main() {
  double* out; cudaMalloc(&out, 1 << 16);
  long long* cyc; cudaMallocManaged(&cyc, 16 * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"dmma_only", "dfma_only", "split_warps", "same_warp"};
  for (int mode = 0; mode < 4; ++mode) {
    int blocks = sms * 2, wpb = 8, iters = 20000;
    mix<<<blocks, 32 * wpb>>>(out, 100, mode);
    cudaEventRecord(e0);
    mix<<<blocks, 32 * wpb>>>(out, iters, mode);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double wm = mode == 0 ? wpb : mode == 1 ? 0 : mode == 2 ? wpb / 2 : wpb;
    double wf = mode == 1 ? wpb : mode == 0 ? 0 : mode == 2 ? wpb / 2 : wpb;
    double fl_m = 512.0 * 8 * iters * blocks * wm;
    double fl_f = 2.0 * 16 * 32 * iters * (double)blocks * wf;
    printf("{\"mode\":\"%s\",\"ms\":%.3f,\"dmma_tflops\":%.2f,\"dfma_tflops\":%.2f,\"total\":%.2f}\n", names[mode], ms,
           fl_m / ms / 1e9, fl_f / ms / 1e9, (fl_m + fl_f) / ms / 1e9);
  }
  lat<<<1, 32>>>(out, cyc, 1.5, 1000); cudaDeviceSynchronize();
  lat<<<1, 32>>>(out, cyc, 1.5, 1000); cudaDeviceSynchronize();
  printf("{\"rcp_approx\":%lld,\"rsqrt_approx\":%lld,\"rcp_newton2\":%lld,\"drcp_rn\":%lld,\"shfl\":%lld,\"rsqrt\":%lld,\"lds\":%lld}\n",
         cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5], cyc[6]);
  // accuracy of rcp.approx / rsqrt.approx
  return 0;
}
