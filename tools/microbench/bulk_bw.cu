// Microbenchmark: L2->SMEM bandwidth of per-warp cp.async.bulk rings (the
// k_smm_dmma staging pattern) vs plain LDG, on a working set like config 1's
// T8 operands (146 MB, random 4.6 KB block offsets).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1910_13555_b200/csrc/bt_ptx.cuh"

// mode 0: one `bytes` bulk copy per product; 1: two bulk copies of bytes/2
// from independent offsets (the A slab + B block of k_smm_dmma); 2: one bulk
// copy of bytes/2 + bytes/2 by the 32 lanes with cp.async (LDGSTS), both
// completing on the stage mbarrier (cp.async.mbarrier.arrive.noinc)
__device__ int g_mode = 0;
__global__ void bulk_ring(const double* __restrict__ src, const int* __restrict__ offs, int noffs,
                          int iters, int S, int bytes, unsigned long long* sink) {
  const int mode = g_mode;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + wid * 8;
  unsigned char* buf = smem + nw * 64 + (size_t)wid * S * bytes;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) bt::mbar_init(&bars[s], mode == 2 ? 33 : 1);
    bt::fence_mbar_init();
  }
  __syncwarp();
  const int gw = blockIdx.x * nw + wid;
  unsigned long long acc = 0;
  int issued = 0;
  auto issue = [&](int q) {
    const int s = q % S;
    const int o = offs[(gw * 7919 + q * 104729) % noffs];
    const int o2 = offs[(gw * 104729 + q * 7919 + 17) % noffs];
    if (mode == 0) {
      if (lane == 0) {
        bt::mbar_arrive_expect_tx(&bars[s], bytes);
        bt::bulk_g2s(buf + s * bytes, src + (size_t)o * 64, bytes, &bars[s]);
      }
    } else if (mode == 1) {
      if (lane == 0) {
        bt::mbar_arrive_expect_tx(&bars[s], bytes);
        bt::bulk_g2s(buf + s * bytes, src + (size_t)o * 64, bytes / 2, &bars[s]);
        bt::bulk_g2s(buf + s * bytes + bytes / 2, src + (size_t)o2 * 64, bytes / 2, &bars[s]);
      }
    } else {
      if (lane == 0) {
        bt::mbar_arrive_expect_tx(&bars[s], bytes / 2);
        bt::bulk_g2s(buf + s * bytes, src + (size_t)o * 64, bytes / 2, &bars[s]);
      }
      const char* g2 = reinterpret_cast<const char*>(src + (size_t)o2 * 64);
      unsigned char* d2 = buf + s * bytes + bytes / 2;
      for (int c = lane * 16; c < bytes / 2; c += 512) bt::cp_async16(d2 + c, g2 + c);
      asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(bt::smem_u32(&bars[s]))
                   : "memory");
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
  for (int mode = 0; mode < 3; ++mode) {
  cudaMemcpyToSymbol(g_mode, &mode, sizeof(int));
  printf("mode %d (%s)\n", mode, mode == 0 ? "one 9.2 KB bulk copy" : mode == 1 ? "two 4.6 KB bulk copies" : "4.6 KB bulk + 4.6 KB LDGSTS");
  for (int warps : {16, 20, 24}) {
    for (int S : {1}) {
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
  }
  return 0;
}
