// Microbenchmark: cycles of potrf_trtri<NT> on one CTA (1 CTA alone on an SM), + correctness.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../paper_2509_03015_b200/csrc/btd_factor.cuh"
using namespace btd;

template <int NT>
__global__ void __launch_bounds__(FactorShape<NT>::NTHREADS, FactorShape<NT>::MINB) bench(const double* A, double* out, long long* cyc, int reps) {
  using S = FactorShape<NT>;
  extern __shared__ __align__(16) double smem[];
  double* DL = smem + 2 * NT * S::LD;
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < NT * NT; e += S::NTHREADS) DL[(e / NT) * S::LD + e % NT] = A[e];
    __syncthreads();
    long long t0 = clock64();
    __shared__ int sf; int piv = 0; if (threadIdx.x < FactorShape<NT>::NWA * 32) piv = potrf_trtri<NT>(DL, &sf);
    __syncthreads();
    long long t1 = clock64();
    tot += t1 - t0;
    if (piv) { if (threadIdx.x == 0) cyc[1] = piv; }
  }
  for (int e = threadIdx.x; e < NT * NT; e += S::NTHREADS) out[e] = DL[(e / NT) * S::LD + e % NT];
  if (threadIdx.x == 0) cyc[0] = tot / reps;
}

template <int NT>
void run() {
  using S = FactorShape<NT>;
  double* hA = (double*)malloc(NT * NT * 8);
  double* M = (double*)malloc(NT * NT * 8);
  srand(1);
  for (int i = 0; i < NT * NT; ++i) M[i] = rand() / (double)RAND_MAX - 0.5;
  for (int i = 0; i < NT; ++i) for (int j = 0; j < NT; ++j) { double s = 0; for (int k = 0; k < NT; ++k) s += M[i*NT+k]*M[j*NT+k]; hA[i*NT+j] = s + (i==j ? NT : 0); }
  double *dA, *dO; long long* cyc;
  cudaMalloc(&dA, NT*NT*8); cudaMalloc(&dO, NT*NT*8); cudaMallocManaged(&cyc, 16); cyc[1] = 0;
  cudaMemcpy(dA, hA, NT*NT*8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(bench<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM);
  bench<NT><<<1, S::NTHREADS, S::SMEM>>>(dA, dO, cyc, 20); cudaDeviceSynchronize();
#ifdef BTD_PHASE_PROF
  { unsigned long long z[16] = {0}; cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z)); }
#endif
  bench<NT><<<1, S::NTHREADS, S::SMEM>>>(dA, dO, cyc, 20); cudaError_t e = cudaDeviceSynchronize();
  double* Li = (double*)malloc(NT*NT*8); cudaMemcpy(Li, dO, NT*NT*8, cudaMemcpyDeviceToHost);
  // check Linv * A * Linv^T == I (lower part of Linv only)
  double err = 0;
  for (int i = 0; i < NT; ++i) for (int j = 0; j < NT; ++j) {
    double s = 0;
    for (int a = 0; a <= i; ++a) for (int b = 0; b <= j; ++b) s += Li[i*NT+a] * hA[a*NT+b] * Li[j*NT+b];
    err = fmax(err, fabs(s - (i == j)));
  }
#ifdef BTD_PHASE_PROF
  unsigned long long ph[16]; cudaMemcpyFromSymbol(ph, g_phase_cycles, sizeof(ph));
  unsigned long long z[16] = {0}; cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  printf("per call: chain %llu wait-helpers %llu critical-update %llu leaves %llu combine %llu\n", ph[6]/20, ph[4]/20, ph[5]/20, ph[9]/20, ph[10]/20);
#endif
  printf("{\"NT\":%d,\"cycles\":%lld,\"fail\":%lld,\"err\":%.2e,\"cuda\":\"%s\"}\n", NT, cyc[0], cyc[1], err, cudaGetErrorString(e));
}
int main() { run<8>(); run<16>(); run<32>(); run<64>(); return 0; }
