// panel_chain (shuffle chain) vs panel_chain_fast (redundant diagonal tile) from btd_factor.cuh,
// timed in isolation (one warp, one CTA).
#include <cstdio>
#include "../paper_2509_03015_b200/csrc/btd_factor.cuh"
using namespace btd;
template <int NT, int V>
__global__ void k(const double* A, double* out, long long* cyc, int reps, int slot, int p0) {
  constexpr int LD = FactorShape<NT>::LD;
  __shared__ double DL[NT * LD];
  long long tot = 0;
  int f = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < NT * NT; e += 32) DL[(e / NT) * LD + e % NT] = A[e];
    __syncwarp();
    long long t0 = clock64();
    if (V == 0) f += panel_chain<NT, true, false>(DL, p0, threadIdx.x);
    else f += panel_chain<NT, true, true>(DL, p0, threadIdx.x);
    __syncwarp();
    long long t1 = clock64();
    tot += t1 - t0;
  }
  out[threadIdx.x] = DL[threadIdx.x * LD] + f;
  if (threadIdx.x == 0) cyc[slot] = tot / reps;
}
int main() {
  double h[64 * 64];
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) h[i * 64 + j] = (i == j) ? 70.0 : 0.01 * ((i * 7 + j * 3) % 11);
  double *A, *o; long long* c; cudaMalloc(&A, sizeof(h)); cudaMalloc(&o, 8192); cudaMallocManaged(&c, 128);
  cudaMemcpy(A, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int it = 0; it < 2; ++it) {
    k<64, 0><<<1, 32>>>(A, o, c, 50, 0, 0);
    k<64, 1><<<1, 32>>>(A, o, c, 50, 1, 0);
    k<64, 0><<<1, 32>>>(A, o, c, 50, 2, 48);
    k<64, 1><<<1, 32>>>(A, o, c, 50, 3, 48);
    cudaDeviceSynchronize();
  }
  printf("{\"old_p0\":%lld,\"fast_p0\":%lld,\"old_p6\":%lld,\"fast_p6\":%lld}\n", c[0], c[1], c[2], c[3]);
}
