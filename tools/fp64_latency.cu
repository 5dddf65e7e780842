// Latency microbenchmarks (single warp / single CTA) for the fp64 pivot chain on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double x0, int iters) {
  double x = x0 + threadIdx.x * 1e-20;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = x * 1.0000001;
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0) / iters;
  // rsqrt chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = rsqrt(x) + 0.5;
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0) / iters;
  // division chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 / x + 0.5;
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0) / iters;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = sqrt(x) + 0.5;
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0) / iters;
  // DMMA chain
  double c0 = x, c1 = x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(1e-3), "d"(1e-3));
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0) / iters;
  // MUFU.RSQ64H-only chain via float rsqrt on double->float
  float f = (float)x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) f = rsqrtf(f) + 0.5f;
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0) / iters;
  // barrier (all warps of block)
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0) / iters;
  // smem store->barrier->load round trip
  __shared__ double sm[256];
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { sm[threadIdx.x] = x; __syncthreads(); x = sm[(threadIdx.x + 1) % blockDim.x] + 1e-9; __syncthreads(); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[8] = (t1 - t0) / iters;
  out[threadIdx.x] = x + c0 + c1 + f;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096); cudaMallocManaged(&cyc, 16 * 8);
  for (int th : {32, 256}) {
    lat<<<1, th>>>(out, cyc, 1.5, 1000); cudaDeviceSynchronize();
    lat<<<1, th>>>(out, cyc, 1.5, 1000); cudaDeviceSynchronize();
    printf("{\"threads\":%d,\"dfma\":%lld,\"dmul\":%lld,\"rsqrt_f64\":%lld,\"div_f64\":%lld,\"sqrt_f64\":%lld,\"dmma\":%lld,\"rsqrtf\":%lld,\"bar\":%lld,\"sts_bar_lds_bar\":%lld}\n",
           th, cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5], cyc[6], cyc[7], cyc[8]);
  }
  return 0;
}
