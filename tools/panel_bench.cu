// Panel factorization variants on one warp (8 columns, 64 rows: lane owns rows l, l+32).
#include <cstdio>
#define FULL 0xffffffffu
template <int V>
__device__ __forceinline__ int panel(double (&va)[8], double (&vb)[8], int lane, double* rinv_out) {
  int fail = 0;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const double d = __shfl_sync(FULL, va[kk], kk);
    double lck[8];
    if (V != 2) {
#pragma unroll
      for (int c = kk + 1; c < 8; ++c) lck[c] = __shfl_sync(FULL, va[kk], c);
    } else {
#pragma unroll
      for (int c = kk + 1; c < 8; ++c) lck[c] = 0.5;
    }
    if (V != 3) { if (d <= 0.0) { fail = kk + 1; break; } }
    const double rinv = (V == 4) ? (double)rsqrtf((float)d) : rsqrt(d);
    const double dinv = rinv * rinv;
#pragma unroll
    for (int c = kk + 1; c < 8; ++c) {
      va[c] = fma(-(va[kk] * lck[c]), dinv, va[c]);
      if (V != 1) vb[c] = fma(-(vb[kk] * lck[c]), dinv, vb[c]);
    }
    va[kk] = (lane == kk) ? d * rinv : va[kk] * rinv;
    vb[kk] *= rinv;
    if (lane == kk) rinv_out[kk] = rinv;
  }
  return fail;
}
template <int V>
__global__ void k(const double* A, double* out, long long* cyc, int reps) {
  __shared__ double rin[8];
  const int lane = threadIdx.x;
  long long tot = 0;
  double va[8], vb[8];
  for (int r = 0; r < reps; ++r) {
    for (int c = 0; c < 8; ++c) { va[c] = A[lane * 8 + c] + r * 1e-12; vb[c] = A[(lane + 32) * 8 + c]; }
    __syncwarp();
    long long t0 = clock64();
    int f = panel<V>(va, vb, lane, rin);
    __syncwarp();
    long long t1 = clock64();
    tot += t1 - t0;
    if (f) out[0] = f;
  }
  for (int c = 0; c < 8; ++c) out[1 + lane * 8 + c] = va[c] + vb[c];
  if (lane == 0) cyc[V] = tot / reps;
}
int main() {
  double hA[64 * 8];
  for (int i = 0; i < 64; ++i) for (int c = 0; c < 8; ++c) hA[i * 8 + c] = (i == c) ? 10.0 : 0.01 * ((i * 7 + c * 3) % 11);
  double *A, *o; long long* cyc; cudaMalloc(&A, sizeof(hA)); cudaMalloc(&o, 8192); cudaMallocManaged(&cyc, 128);
  cudaMemcpy(A, hA, sizeof(hA), cudaMemcpyHostToDevice);
  for (int it = 0; it < 2; ++it) {
    k<0><<<1, 32>>>(A, o, cyc, 100); k<1><<<1, 32>>>(A, o, cyc, 100); k<2><<<1, 32>>>(A, o, cyc, 100);
    k<3><<<1, 32>>>(A, o, cyc, 100); k<4><<<1, 32>>>(A, o, cyc, 100);
    cudaDeviceSynchronize();
  }
  printf("{\"panel_full\":%lld,\"no_vb\":%lld,\"no_lck_shfl\":%lld,\"no_branch\":%lld,\"rsqrtf\":%lld}\n", cyc[0], cyc[1], cyc[2], cyc[3], cyc[4]);
}
