// fp64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) and DFMA.
// Used to establish the fp64 roofline denominator (MEASURED_PEAKS.json carries no fp64 figure).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = 0.0; c[t][1] = 0.0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) c[t] = t;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 16; ++t) c[t] = fma(a, c[t], b);
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 16; ++t) s += c[t];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int wpb : {4, 8, 16}) {
    int blocks = sms * 2, threads = 32 * wpb, iters = 20000;
    dmma_loop<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)blocks * wpb;
    printf("{\"kind\":\"dmma_m8n8k4\",\"warps_per_block\":%d,\"blocks\":%d,\"tflops\":%.2f}\n", wpb, blocks, flops / ms / 1e9);
  }
  for (int wpb : {4, 8, 16}) {
    int blocks = sms * 2, threads = 32 * wpb, iters = 20000;
    dfma_loop<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16.0 * iters * (double)blocks * threads;
    printf("{\"kind\":\"dfma\",\"warps_per_block\":%d,\"blocks\":%d,\"tflops\":%.2f}\n", wpb, blocks, flops / ms / 1e9);
  }
  return 0;
}
