// Microbenchmark: L2->SMEM bandwidth of per-warp cp.async.bulk rings (the
// k_smm_dmma staging pattern) vs plain LDG, on a working set like config 1's
// T8 operands (146 MB, random 4.6 KB block offsets).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1910_13555_b200/csrc/bt_ptx.cuh"

__global__ void bulk_ring(const double* __restrict__ src, const int* __restrict__ offs, int noffs,
                          int iters, int S, int bytes, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + wid * 8;
  unsigned char* buf = smem + nw * 64 + (size_t)wid * S * bytes;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) bt::mbar_init(&bars[s], 1);
    bt::fence_mbar_init();
  }
  __syncwarp();
  const int gw = blockIdx.x * nw + wid;
  unsigned long long acc = 0;
  int issued = 0;
  auto issue = [&](int q) {
    if (lane == 0) {
      const int s = q % S;
      bt::mbar_arrive_expect_tx(&bars[s], bytes);
      const int o = offs[(gw * 7919 + q * 104729) % noffs];
      bt::bulk_g2s(buf + s * bytes, src + (size_t)o * 64, bytes, &bars[s]);
    }
  };
  for (; issued < S; ++issued) issue(issued);
  for (int q = 0; q < iters; ++q) {
    const int s = q % S;
    bt::mbar_wait(&bars[s], (q / S) & 1);
    acc += buf[s * bytes + lane * 8];
    __syncwarp();
    if (issued < iters) issue(issued++);
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

int main() {
  const size_t bytes_total = 146ull << 20;
  const int block = 9216;  // one c1 product: A slab + B block (T8)
  double* src;
  cudaMalloc(&src, bytes_total);
  cudaMemset(src, 1, bytes_total);
  const int noffs = (int)(bytes_total / block) - 1;
  int* offs;
  cudaMalloc(&offs, noffs * 4);
  int* h = new int[noffs];
  for (int i = 0; i < noffs; ++i) h[i] = (int)(((long long)i * 2654435761u) % noffs) * (block / 512);
  cudaMemcpy(offs, h, noffs * 4, cudaMemcpyHostToDevice);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 24}) {
    for (int S : {1, 2, 3}) {
      const int wpc = 4;
      const int ctas = warps / wpc;
      const size_t smem = wpc * 64 + (size_t)wpc * S * block;
      if (smem * ctas > 227 * 1024) continue;
      cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int iters = 2000;
      bulk_ring<<<148 * ctas, wpc * 32, smem>>>(src, offs, noffs, 10, S, block, sink);
      cudaEventRecord(e0);
      bulk_ring<<<148 * ctas, wpc * 32, smem>>>(src, offs, noffs, iters, S, block, sink);
      cudaEventRecord(e1);
      cudaError_t err = cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double gb = (double)block * iters * 148 * ctas * wpc / 1e9;
      printf("warps/SM %2d S=%d: %.2f TB/s  (%s)\n", warps, S, gb / ms, cudaGetErrorString(err));
    }
  }
  return 0;
}
