// Microbenchmark: B200 FP64 throughput (DFMA vs DMMA shapes) and L2/HBM read bandwidth.
// Used to pick the small-GEMM instruction path and the roofline denominator.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters, double s) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, s, 1.0); a1 = fma(a1, s, 1.0); a2 = fma(a2, s, 1.0); a3 = fma(a3, s, 1.0);
      a4 = fma(a4, s, 1.0); a5 = fma(a5, s, 1.0); a6 = fma(a6, s, 1.0); a7 = fma(a7, s, 1.0);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

// 8 independent m8n8k4 accumulators per warp
__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int t = 0; t < 8; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// m16n8k16: A 8 regs, B 4 regs, C 4 regs
__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int t = 0; t < 8; ++t) a[t] = threadIdx.x * 1e-3 + t;
#pragma unroll
  for (int t = 0; t < 4; ++t) b[t] = 1.0 - threadIdx.x * 1e-4 - t;
  double c[4][4];
#pragma unroll
  for (int t = 0; t < 4; ++t) for (int q = 0; q < 4; ++q) c[t][q] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void read_kernel(const double2* __restrict__ p, size_t n, int reps, double* out) {
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(p + i);
      acc += v.x + v.y;
    }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d maxclk %d kHz L2 %d MB\n", prop.name, prop.multiProcessorCount, clk, prop.l2CacheSize >> 20);
  int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 64 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int occ : {4, 8, 16}) {
    int blocks = sms * occ, threads = 256, iters = 2000;
    dfma_kernel<<<blocks, threads>>>(out, 10, 0.999);
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 0.999); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * blocks * threads * (double)iters * 16 * 8;
    printf("DFMA  occ %2d: %.2f TFLOP/s\n", occ, flops / ms / 1e9);
  }
  for (int occ : {1, 2, 4, 8}) {
    int blocks = sms * occ, threads = 256, iters = 2000;
    dmma884_kernel<<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0); dmma884_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * (blocks * threads / 32) * (double)iters * 4 * 8 * 256;
    printf("DMMA m8n8k4 warps/SM %2d: %.2f TFLOP/s\n", occ * 8, flops / ms / 1e9);
  }
  for (int occ : {1, 2, 4, 8}) {
    int blocks = sms * occ, threads = 256, iters = 2000;
    dmma16816_kernel<<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0); dmma16816_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * (blocks * threads / 32) * (double)iters * 4 * 16 * 8 * 16;
    printf("DMMA m16n8k16 warps/SM %2d: %.2f TFLOP/s\n", occ * 8, flops / ms / 1e9);
  }
  for (size_t mb : {32, 64, 96, 4096}) {
    size_t bytes = mb << 20; double2* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes));
    size_t n = bytes / 16; int reps = mb < 1000 ? 50 : 3;
    read_kernel<<<sms * 8, 512>>>(buf, n, 1, out);
    cudaEventRecord(e0); read_kernel<<<sms * 8, 512>>>(buf, n, reps, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("read %5zu MB x%d: %.1f GB/s\n", mb, reps, (double)bytes * reps / ms / 1e6);
    cudaFree(buf);
  }
  return 0;
}
