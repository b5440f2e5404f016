// Microbenchmark: the k_smm_dmma inner product loop (T8 fragments from shared
// memory, 3x3 C tiles, 6 k chunks = one 24x24x24 product) without any copies,
// to separate inner-loop efficiency from the staging pipeline.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1910_13555_b200/csrc/bt_ptx.cuh"

template <int TMT, int TNT, int KT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) inner(double* out, int iters) {
  extern __shared__ __align__(128) double sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int sw_g = ((gq >> 1) & 1) << 2;
  const int la0 = gq * 8 + (tq ^ sw_g), la1 = gq * 8 + ((4 + tq) ^ sw_g);
  const int swt = ((tq >> 1) & 1) << 2;
  const int lb0 = tq * 8 + (gq ^ swt), lb1 = (4 + tq) * 8 + (gq ^ swt);
  double* sA = sm + wid * (TMT + TNT) * KT * 64;
  double* sB = sA + TMT * KT * 64;
  for (int i = threadIdx.x; i < WARPS * (TMT + TNT) * KT * 64; i += blockDim.x) sm[i] = 1e-3 * (i % 7);
  __syncthreads();
  double acc[TMT][TNT][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      double af[2][TMT], bf[2][TNT];
#pragma unroll
      for (int tm = 0; tm < TMT; ++tm) {
        af[0][tm] = sA[((tm * KT + kt) << 6) + la0];
        af[1][tm] = sA[((tm * KT + kt) << 6) + la1];
      }
#pragma unroll
      for (int tn = 0; tn < TNT; ++tn) {
        bf[0][tn] = sB[((kt * TNT + tn) << 6) + lb0];
        bf[1][tn] = sB[((kt * TNT + tn) << 6) + lb1];
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int tm = 0; tm < TMT; ++tm)
#pragma unroll
          for (int tn = 0; tn < TNT; ++tn) bt::dmma_884(acc[tm][tn][0], acc[tm][tn][1], af[h][tm], bf[h][tn]);
    }
  }
  double s = 0;
#pragma unroll
  for (int tm = 0; tm < TMT; ++tm)
#pragma unroll
    for (int tn = 0; tn < TNT; ++tn) s += acc[tm][tn][0] + acc[tm][tn][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  for (int ctas : {1, 2, 3, 4, 6}) {
    const int WARPS = 4;
    const size_t smem = WARPS * 6 * 3 * 64 * 8;
    auto k = inner<3, 3, 3, 4>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<148 * ctas, WARPS * 32, smem>>>(out, 10);
    cudaEventRecord(e0);
    k<<<148 * ctas, WARPS * 32, smem>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 24 * 24 * 24 * (double)iters * 148 * ctas * WARPS;
    printf("warps/SM %2d: %.2f TFLOP/s padded (%.1f%% of 37.1), useful-equiv %.2f\n", ctas * WARPS,
           fl / ms / 1e9, fl / ms / 1e9 / 37.1 * 100, fl / ms / 1e9 * (23.0 * 23 * 23) / (24 * 24 * 24));
  }
  return 0;
}
