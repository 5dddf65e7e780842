// Microbench of one warp's dependent chains: shfl(double), rsqrt, the 2x2 pivot step.
#include <cstdio>
__global__ void k(double* out, long long* cyc, int iters) {
  double x = 1.0 + threadIdx.x * 1e-3, y = 2.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (i + 1) & 31) + 1e-9;
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { float f = __shfl_sync(0xffffffffu, (float)x, (i + 1) & 31); x = f + 1e-9; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / iters;
  // rsqrt + dmul + dfma (pivot chain of one column)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { double r = rsqrt(x); x = fma(r * r, -1e-3, x) + 1.0; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / iters;
  // full 1-column step: shfl pivot -> rsqrt -> dmul -> dfma
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { double d = __shfl_sync(0xffffffffu, x, i & 7); double r = rsqrt(d); x = fma(r * r, -1e-3, x) + 1.0; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / iters;
  // with a data-dependent branch on the pivot
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { double d = __shfl_sync(0xffffffffu, x, i & 7); if (d <= 0.0) break; double r = rsqrt(d); x = fma(r * r, -1e-3, x) + 1.0; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / iters;
  // smem round trip in-warp: st -> syncwarp -> ld
  __shared__ double sm[32];
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { sm[threadIdx.x] = x; __syncwarp(); x = sm[(threadIdx.x + 1) & 31] + 1e-9; __syncwarp(); }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0) / iters;
  out[threadIdx.x] = x + y;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMallocManaged(&c, 128);
  k<<<1, 32>>>(o, c, 1000); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1000); cudaDeviceSynchronize();
  printf("{\"shfl_f64\":%lld,\"shfl_f32\":%lld,\"rsqrt_step\":%lld,\"col_step\":%lld,\"col_step_branch\":%lld,\"smem_warp_rt\":%lld}\n", c[0], c[1], c[2], c[3], c[4], c[5]);
}
