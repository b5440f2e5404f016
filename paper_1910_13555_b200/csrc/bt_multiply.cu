// bt_multiply.cu -- the hot path: local block-sparse C += A*B on one B200.
//
// Device equivalent of detail::multiply_tiles_into (multiply_cannon.hpp:24-44):
//   reference                               here (all device-resident)
//   std::map b_by_k + BatchItem list   ->   B column index (CSC, radix sort) + per-C-row
//   (multiply_cannon.hpp:27-36)             k-map stack generation (k_stack<...>)
//   order_batches (block.hpp:112-118)  ->   stacks grouped per C block, k ascending
//   get_or_create (matrix.hpp:191-196) ->   symbolic bitmap union C_in U products
//                                           (k_sym_count / k_sym_fill)
//   block_gemm_acc (block.hpp:45-60)   ->   k_smm_dmma<TM,TN>: one warp per C tile,
//                                           bulk-async (TMA 1D) staged A/B blocks,
//                                           FP64 DMMA 8x8x4 from shared memory;
//                                           k_smm_generic for shapes outside the
//                                           DMMA classes.
// Accumulation per C element follows the reference order over k-blocks
// (ascending), each C block written exactly once (no atomics): results are
// deterministic run to run.
#include <cub/cub.cuh>

#include <algorithm>
#include <array>

#include "bt_internal.cuh"
#include "bt_ptx.cuh"

namespace bt {

// ------------------------------------------------------------ small kernels
__global__ void k_expand_rows(const int32_t* __restrict__ rp, int64_t nbr,
                              int32_t* __restrict__ rows) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nbr) return;
  for (int32_t e = rp[i]; e < rp[i + 1]; ++e) rows[e] = static_cast<int32_t>(i);
}

__global__ void k_csc_keys(const int32_t* __restrict__ rows, const int32_t* __restrict__ col,
                           int64_t n, uint64_t* __restrict__ keys, int32_t* __restrict__ idx,
                           int32_t* __restrict__ colcnt) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  keys[e] = (static_cast<uint64_t>(col[e]) << 32) | static_cast<uint32_t>(rows[e]);
  idx[e] = static_cast<int32_t>(e);
  atomicAdd(&colcnt[col[e]], 1);
}

__global__ void k_csc_split(const uint64_t* __restrict__ keys, int64_t n, int32_t* __restrict__ k) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  k[e] = static_cast<int32_t>(keys[e] & 0xffffffffu);
}

__device__ __forceinline__ bool keep_product(const double* na, const double* nb, int32_t e,
                                             int32_t f, double eps) {
  return !(eps > 0.0) || __dmul_rn(na[e], nb[f]) >= eps;
}

// Symbolic pass 1: per A block-row i, the bitmap of C block columns
// C_in(i,:) U {j : exists k, A_ik, B_kj stored and kept}; popcount -> row_cnt.
__global__ void k_sym_count(const int32_t* __restrict__ a_rp, const int32_t* __restrict__ a_col,
                            const int32_t* __restrict__ b_rp, const int32_t* __restrict__ b_col,
                            const int32_t* __restrict__ c_rp, const int32_t* __restrict__ c_col,
                            const double* __restrict__ na, const double* __restrict__ nb,
                            double eps, int nwords, uint32_t* __restrict__ g_bm,
                            int32_t* __restrict__ row_cnt) {
  extern __shared__ uint32_t bm[];
  const int64_t i = blockIdx.x;
  for (int w = threadIdx.x; w < nwords; w += blockDim.x) bm[w] = 0;
  __syncthreads();
  for (int32_t e = c_rp[i] + threadIdx.x; e < c_rp[i + 1]; e += blockDim.x) {
    const int32_t j = c_col[e];
    atomicOr(&bm[j >> 5], 1u << (j & 31));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int32_t e = a_rp[i] + wid; e < a_rp[i + 1]; e += nw) {
    const int32_t k = a_col[e];
    for (int32_t f = b_rp[k] + lane; f < b_rp[k + 1]; f += 32) {
      if (!keep_product(na, nb, e, f, eps)) continue;
      const int32_t j = b_col[f];
      atomicOr(&bm[j >> 5], 1u << (j & 31));
    }
  }
  __syncthreads();
  int cnt = 0;
  for (int w = threadIdx.x; w < nwords; w += blockDim.x) {
    const uint32_t v = bm[w];
    g_bm[i * nwords + w] = v;
    cnt += __popc(v);
  }
  using BR = cub::BlockReduce<int, 256>;
  __shared__ typename BR::TempStorage tmp;
  const int tot = BR(tmp).Sum(cnt);
  if (threadIdx.x == 0) row_cnt[i] = tot;
}

// Symbolic pass 2: emit sorted C columns of row i, their padded sizes, the row
// of each entry, and the C_in slot feeding it (or -1).
__global__ void k_sym_fill(const uint32_t* __restrict__ g_bm, int nwords,
                           const int32_t* __restrict__ out_rp, const int32_t* __restrict__ rsz,
                           const int32_t* __restrict__ csz, const int32_t* __restrict__ cin_rp,
                           const int32_t* __restrict__ cin_col,
                           const int64_t* __restrict__ cin_off, int32_t* __restrict__ out_col,
                           int32_t* __restrict__ out_row, int64_t* __restrict__ out_len,
                           int64_t* __restrict__ cin_map,
                           unsigned long long* __restrict__ elems_total) {
  extern __shared__ int32_t wpref[];
  const int64_t i = blockIdx.x;
  const int32_t base = out_rp[i];
  const int m = rsz[i];
  using BS = cub::BlockScan<int, 256>;
  __shared__ typename BS::TempStorage tmp;
  int running = 0;
  unsigned long long elems = 0;
  for (int w0 = 0; w0 < nwords; w0 += blockDim.x) {
    const int w = w0 + threadIdx.x;
    uint32_t word = w < nwords ? g_bm[i * nwords + w] : 0u;
    int excl, total;
    BS(tmp).ExclusiveSum(__popc(word), excl, total);
    if (w < nwords) wpref[w] = running + excl;
    int32_t pos = base + running + excl;
    while (word) {
      const int b = __ffs(word) - 1;
      const int32_t j = w * 32 + b;
      out_col[pos] = j;
      out_row[pos] = static_cast<int32_t>(i);
      const int64_t L = static_cast<int64_t>(m) * csz[j];
      out_len[pos] = pad2(L);
      elems += static_cast<unsigned long long>(L);
      cin_map[pos] = -1;
      ++pos;
      word &= word - 1;
    }
    running += total;
    __syncthreads();
  }
  {
    using BR = cub::BlockReduce<unsigned long long, 256>;
    __shared__ typename BR::TempStorage rt;
    const unsigned long long tot = BR(rt).Sum(elems);
    if (threadIdx.x == 0 && tot) atomicAdd(elems_total, tot);
  }
  __syncthreads();
  for (int32_t e = cin_rp[i] + threadIdx.x; e < cin_rp[i + 1]; e += blockDim.x) {
    const int32_t j = cin_col[e];
    const int w = j >> 5;
    const uint32_t below = g_bm[i * nwords + w] & ((1u << (j & 31)) - 1u);
    cin_map[base + wpref[w] + __popc(below)] = cin_off[e];
  }
}

// Stack generation.  One CTA per C block-row i; kmap[k] = A entry of (i,k)
// (shared memory) so each C block (i,j) walks only B's column j (k ascending):
// products come out grouped per C block in the reference's (row, col, k) order
// (order_batches, block.hpp:112-118).
template <bool FILL, bool KMAP>
__global__ void k_stack(const int32_t* __restrict__ a_rp, const int32_t* __restrict__ a_col,
                        int64_t a_nbc, const int32_t* __restrict__ bc_ptr,
                        const int32_t* __restrict__ bc_k, const int32_t* __restrict__ bc_e,
                        const int32_t* __restrict__ c_rp, const int32_t* __restrict__ c_col,
                        const double* __restrict__ na, const double* __restrict__ nb, double eps,
                        const int32_t* __restrict__ m_sz, const int32_t* __restrict__ n_sz,
                        const int32_t* __restrict__ k_sz, int32_t* __restrict__ cnt,
                        unsigned long long* __restrict__ totals,
                        const int64_t* __restrict__ stk_ptr, int32_t* __restrict__ stk_a,
                        int32_t* __restrict__ stk_b) {
  extern __shared__ int32_t kmap[];
  const int64_t i = blockIdx.x;
  const int32_t a0 = a_rp[i], a1 = a_rp[i + 1];
  if (KMAP) {
    for (int64_t k = threadIdx.x; k < a_nbc; k += blockDim.x) kmap[k] = -1;
    __syncthreads();
    for (int32_t e = a0 + threadIdx.x; e < a1; e += blockDim.x) kmap[a_col[e]] = e;
    __syncthreads();
  }
  unsigned long long cand = 0, mnk = 0;
  for (int32_t c = c_rp[i] + threadIdx.x; c < c_rp[i + 1]; c += blockDim.x) {
    const int32_t j = c_col[c];
    int32_t n = 0;
    unsigned long long ksum = 0;
    int64_t dst = FILL ? stk_ptr[c] : 0;
    for (int32_t f = bc_ptr[j]; f < bc_ptr[j + 1]; ++f) {
      const int32_t k = bc_k[f];
      int32_t e;
      if (KMAP) {
        e = kmap[k];
      } else {
        int32_t lo = a0, hi = a1;
        while (lo < hi) {
          const int32_t mid = (lo + hi) >> 1;
          if (a_col[mid] < k) lo = mid + 1; else hi = mid;
        }
        e = (lo < a1 && a_col[lo] == k) ? lo : -1;
      }
      if (e < 0) continue;
      ++cand;
      const int32_t bent = bc_e[f];
      if (!keep_product(na, nb, e, bent, eps)) continue;
      if (FILL) {
        stk_a[dst] = e;
        stk_b[dst] = bent;
        ++dst;
      }
      if (!FILL) ksum += static_cast<unsigned long long>(k_sz[k]);
      ++n;
    }
    if (!FILL) {
      cnt[c] = n;
      mnk += ksum * static_cast<unsigned long long>(m_sz[i]) * n_sz[j];
    }
  }
  if (!FILL) {
    using BR = cub::BlockReduce<unsigned long long, 128>;
    __shared__ typename BR::TempStorage tmp;
    const unsigned long long tot = BR(tmp).Sum(cand);
    __syncthreads();
    const unsigned long long tot2 = BR(tmp).Sum(mnk);
    if (threadIdx.x == 0) {
      if (tot) atomicAdd(&totals[0], tot);
      if (tot2) atomicAdd(&totals[1], tot2);
    }
  }
}

// ------------------------------------------------------------- work items
// A work item is one C tile: (C entry, block row, first row) -- C blocks taller
// than 32 rows are split into 32-row tiles (config 4's (ab|P) blocks).
enum { NCLASS = 17, GENERIC = 16 };

__host__ __device__ inline int shape_class(int m, int n, bool dmma_ok) {
  if (!dmma_ok || n > 32) return GENERIC;
  const int mc = m > 32 ? 4 : (m + 7) / 8;
  const int nc = (n + 7) / 8;
  return (mc - 1) * 4 + (nc - 1);
}

__global__ void k_classify(const int32_t* __restrict__ c_row, const int32_t* __restrict__ c_col,
                           const int32_t* __restrict__ rsz, const int32_t* __restrict__ csz,
                           int64_t n, bool dmma_ok, uint8_t* __restrict__ cls,
                           int32_t* __restrict__ order, int32_t* __restrict__ hist) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int k = shape_class(rsz[c_row[c]], csz[c_col[c]], dmma_ok);
  cls[c] = static_cast<uint8_t>(k);
  order[c] = static_cast<int32_t>(c);
  atomicAdd(&hist[k], 1);
}

__global__ void k_tiles(const int32_t* __restrict__ order, const uint8_t* __restrict__ cls_sorted,
                        const int32_t* __restrict__ c_row, const int32_t* __restrict__ rsz,
                        int64_t n, int32_t* __restrict__ ntiles) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int m = rsz[c_row[order[t]]];
  ntiles[t] = (cls_sorted[t] != GENERIC && m > 32) ? (m + 31) / 32 : 1;
}

__global__ void k_expand_items(const int32_t* __restrict__ order,
                               const int32_t* __restrict__ c_row,
                               const int32_t* __restrict__ ntiles,
                               const int64_t* __restrict__ tstart,
                               const int32_t* __restrict__ cnt, int64_t n,
                               int4* __restrict__ items, int64_t* __restrict__ weight) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int32_t c = order[t];
  const int64_t s = tstart[t];
  for (int q = 0; q < ntiles[t]; ++q) {
    items[s + q] = make_int4(c, c_row[c], 32 * q, 0);
    weight[s + q] = static_cast<int64_t>(cnt[c]) + 1;
  }
}

struct NumArgs {
  const int4* items;
  const int64_t* item_pp;
  int64_t item_lo, item_hi;
  const int64_t* stk_ptr;
  const int32_t* stk_a;
  const int32_t* stk_b;
  const double* a_vals;
  const int64_t* a_off;
  const int32_t* a_col;
  const int32_t* k_sz;  // A column block sizes
  const double* b_vals;
  const int64_t* b_off;
  const int32_t* m_sz;  // C row block sizes
  const int32_t* n_sz;  // C column block sizes
  const int32_t* c_col;
  double* c_vals;
  const int64_t* c_off;
  const int64_t* cin_map;
  const double* cin_vals;
  int stages;
  int stage_elems;
  int a_region;
};

__device__ __forceinline__ int64_t first_item_at(const int64_t* pp, int64_t lo, int64_t hi,
                                                 int64_t target) {
  // first it in [lo, hi] with pp[it] >= target
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (pp[mid] < target) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// FP64 DMMA small-GEMM: one warp owns one C tile of TM = 8*TMT rows by
// TN = 8*TNT columns (m <= TM, n <= TN); the tile's products stream through a
// per-warp ring of `stages` shared-memory buffers filled by bulk async copies
// (one A block slab + one B block per product) completing on mbarriers.
// Accumulators stay in registers for the whole product chain; the C tile is
// written once.  Warps take contiguous item ranges balanced by product count.
template <int TMT, int TNT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_smm_dmma(const NumArgs g) {
  constexpr int TM = 8 * TMT;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int S = g.stages;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + wid * 8;
  double* stages = reinterpret_cast<double*>(smem + WARPS * 64) +
                   static_cast<int64_t>(wid) * S * g.stage_elems;

  const int64_t W = static_cast<int64_t>(gridDim.x) * WARPS;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * WARPS + wid;
  const int64_t p0 = g.item_pp[g.item_lo], pt = g.item_pp[g.item_hi] - p0;
  const int64_t it0 = first_item_at(g.item_pp, g.item_lo, g.item_hi, p0 + pt * gw / W);
  const int64_t it1 = first_item_at(g.item_pp, g.item_lo, g.item_hi, p0 + pt * (gw + 1) / W);
  if (it0 >= it1) return;

  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();

  // producer cursor (uniform across the warp; lane 0 issues)
  int64_t p_it = it0, p_pos = 0, p_end = 0;
  {
    const int c = g.items[p_it].x;
    p_pos = g.stk_ptr[c];
    p_end = g.stk_ptr[c + 1];
  }
  auto p_skip = [&]() {
    while (p_it < it1 && p_pos >= p_end) {
      ++p_it;
      if (p_it < it1) {
        const int c = g.items[p_it].x;
        p_pos = g.stk_ptr[c];
        p_end = g.stk_ptr[c + 1];
      }
    }
  };
  auto issue = [&](int s) {
    if (p_it >= it1) return;
    if (lane == 0) {
      const int4 item = g.items[p_it];
      const int32_t ae = g.stk_a[p_pos], be = g.stk_b[p_pos];
      const int k = g.k_sz[g.a_col[ae]];
      const int m = g.m_sz[item.y];
      const int n = g.n_sz[g.c_col[item.x]];
      const int rows = min(TM, m - item.z);
      const uint32_t ba = static_cast<uint32_t>((rows * k * 8 + 15) & ~15);
      const uint32_t bb = static_cast<uint32_t>((k * n * 8 + 15) & ~15);
      double* st = stages + static_cast<int64_t>(s) * g.stage_elems;
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&bars[s], ba + bb);
      bulk_g2s(st, g.a_vals + g.a_off[ae] + static_cast<int64_t>(item.z) * k, ba, &bars[s]);
      bulk_g2s(st + g.a_region, g.b_vals + g.b_off[be], bb, &bars[s]);
    }
    ++p_pos;
    p_skip();
  };
  p_skip();
  for (int s = 0; s < S; ++s) issue(s);

  uint32_t seq = 0;
  for (int64_t it = it0; it < it1; ++it) {
    const int4 item = g.items[it];
    const int c = item.x, r0 = item.z;
    const int m = g.m_sz[item.y];
    const int n = g.n_sz[g.c_col[c]];
    const int rows = min(TM, m - r0);
    double acc[TMT][TNT][2];
    const int64_t cin = g.cin_map[c];
#pragma unroll
    for (int tm = 0; tm < TMT; ++tm)
#pragma unroll
      for (int tn = 0; tn < TNT; ++tn) {
        const int r = 8 * tm + gq, cc = 8 * tn + 2 * tq;
        acc[tm][tn][0] = 0.0;
        acc[tm][tn][1] = 0.0;
        if (cin >= 0 && r < rows) {
          const double* src = g.cin_vals + cin + static_cast<int64_t>(r0 + r) * n;
          if (cc < n) acc[tm][tn][0] = src[cc];
          if (cc + 1 < n) acc[tm][tn][1] = src[cc + 1];
        }
      }
    const int64_t pe = g.stk_ptr[c + 1];
    for (int64_t p = g.stk_ptr[c]; p < pe; ++p) {
      const int s = static_cast<int>(seq % static_cast<uint32_t>(S));
      const uint32_t par = (seq / static_cast<uint32_t>(S)) & 1u;
      const int k = g.k_sz[g.a_col[g.stk_a[p]]];
      mbar_wait(&bars[s], par);
      const double* sA = stages + static_cast<int64_t>(s) * g.stage_elems;
      const double* sB = sA + g.a_region;
      const int kfull = k >> 2;
#pragma unroll 2
      for (int kc = 0; kc < kfull; ++kc) {
        double af[TMT], bf[TNT];
#pragma unroll
        for (int tm = 0; tm < TMT; ++tm) af[tm] = sA[(8 * tm + gq) * k + 4 * kc + tq];
#pragma unroll
        for (int tn = 0; tn < TNT; ++tn) bf[tn] = sB[(4 * kc + tq) * n + 8 * tn + gq];
#pragma unroll
        for (int tm = 0; tm < TMT; ++tm)
#pragma unroll
          for (int tn = 0; tn < TNT; ++tn) dmma_884(acc[tm][tn][0], acc[tm][tn][1], af[tm], bf[tn]);
      }
      if (k & 3) {
        const int kk = 4 * kfull + tq;
        const bool ok = kk < k;
        double af[TMT], bf[TNT];
#pragma unroll
        for (int tm = 0; tm < TMT; ++tm) {
          af[tm] = 0.0;
          if (ok) af[tm] = sA[(8 * tm + gq) * k + kk];
        }
#pragma unroll
        for (int tn = 0; tn < TNT; ++tn) {
          bf[tn] = 0.0;
          if (ok) bf[tn] = sB[kk * n + 8 * tn + gq];
        }
#pragma unroll
        for (int tm = 0; tm < TMT; ++tm)
#pragma unroll
          for (int tn = 0; tn < TNT; ++tn) dmma_884(acc[tm][tn][0], acc[tm][tn][1], af[tm], bf[tn]);
      }
      __syncwarp();
      issue(s);
      ++seq;
    }
    double* dst = g.c_vals + g.c_off[c];
#pragma unroll
    for (int tm = 0; tm < TMT; ++tm)
#pragma unroll
      for (int tn = 0; tn < TNT; ++tn) {
        const int r = 8 * tm + gq, cc = 8 * tn + 2 * tq;
        if (r < rows) {
          double* d = dst + static_cast<int64_t>(r0 + r) * n;
          if (cc < n) d[cc] = acc[tm][tn][0];
          if (cc + 1 < n) d[cc + 1] = acc[tm][tn][1];
        }
      }
  }
}

// Generic small-GEMM for shapes outside the DMMA classes (n > 32 or k > 64):
// one CTA per C block, one thread per element, products in k order.
__global__ void k_smm_generic(const NumArgs g) {
  const int64_t it = g.item_lo + blockIdx.x;
  if (it >= g.item_hi) return;
  const int4 item = g.items[it];
  const int c = item.x;
  const int m = g.m_sz[item.y];
  const int n = g.n_sz[g.c_col[c]];
  const int64_t cin = g.cin_map[c];
  const int64_t p0 = g.stk_ptr[c], p1 = g.stk_ptr[c + 1];
  double* dst = g.c_vals + g.c_off[c];
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int r = e / n, q = e % n;
    double acc = cin >= 0 ? g.cin_vals[cin + e] : 0.0;
    for (int64_t p = p0; p < p1; ++p) {
      const int32_t ae = g.stk_a[p];
      const int k = g.k_sz[g.a_col[ae]];
      const double* a = g.a_vals + g.a_off[ae] + static_cast<int64_t>(r) * k;
      const double* b = g.b_vals + g.b_off[g.stk_b[p]] + q;
      for (int t = 0; t < k; ++t) acc = fma(a[t], b[static_cast<int64_t>(t) * n], acc);
    }
    dst[e] = acc;
  }
}

// ------------------------------------------------------------------- host
namespace {

template <class T>
T read_scalar(const T* dptr, cudaStream_t s) {
  T v;
  BT_CUDA(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, s));
  BT_CUDA(cudaStreamSynchronize(s));
  return v;
}

template <class TIn, class TOut>
void exclusive_scan(Ctx& x, const TIn* in, TOut* out, int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, x.stream);
  void* tmp = x.ensure_scratch(bytes);
  cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, n, x.stream);
  count_launch(&x, 2);
}

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

struct Launch {
  int warps = 4;
  int stages = 3;
  int stage_elems = 0;
  int a_region = 0;
  size_t smem = 0;
};

using KernelFn = void (*)(const NumArgs);

KernelFn dmma_kernel(int cls) {
  static const KernelFn table[16] = {
      k_smm_dmma<1, 1, 4>, k_smm_dmma<1, 2, 4>, k_smm_dmma<1, 3, 4>, k_smm_dmma<1, 4, 4>,
      k_smm_dmma<2, 1, 4>, k_smm_dmma<2, 2, 4>, k_smm_dmma<2, 3, 4>, k_smm_dmma<2, 4, 4>,
      k_smm_dmma<3, 1, 4>, k_smm_dmma<3, 2, 4>, k_smm_dmma<3, 3, 4>, k_smm_dmma<3, 4, 4>,
      k_smm_dmma<4, 1, 4>, k_smm_dmma<4, 2, 4>, k_smm_dmma<4, 3, 4>, k_smm_dmma<4, 4, 4>};
  return table[cls];
}

// Shared-memory plan for one DMMA class: per warp `stages` buffers of
// (TM x kmax) + (kmax x TN) doubles; aim for >= 8 resident warps per SM.
Launch plan_dmma(const Ctx& x, int cls, int kmax) {
  Launch L;
  const int TM = 8 * (cls / 4 + 1), TN = 8 * (cls % 4 + 1);
  L.a_region = static_cast<int>(pad2(static_cast<int64_t>(TM) * kmax));
  L.stage_elems = L.a_region + static_cast<int>(pad2(static_cast<int64_t>(kmax) * TN));
  const size_t per_stage = static_cast<size_t>(L.stage_elems) * 8;
  const size_t budget = 220 * 1024;  // per SM, leaves room for the CTA reservation
  // largest stage count (<= 4) that keeps 8 warps per SM, at least 2
  int s = 4;
  while (s > 2 && 8 * s * per_stage + 2 * L.warps * 64 > budget) --s;
  L.stages = s;
  L.smem = L.warps * 64 + static_cast<size_t>(L.warps) * s * per_stage;
  return L;
}

}  // namespace

}  // namespace bt

using namespace bt;

extern "C" int bt_multiply(bt_ctx* ctx, const bt_mat* ah, const bt_mat* bh, bt_mat* ch,
                           double eps, bt_stats* stats) {
  return guard([&] {
    BT_REQUIRE(ctx && ah && bh && ch, BT_ERR_INVALID_ARGUMENT, "null argument");
    Ctx& x = ctx->impl;
    const Mat& A = ah->impl;
    const Mat& B = bh->impl;
    Mat& Cm = ch->impl;
    BT_REQUIRE(A.ctx == &x && B.ctx == &x && Cm.ctx == &x, BT_ERR_INVALID_ARGUMENT,
               "bt_multiply: matrices belong to another context");
    // conformity (multiply_cannon.hpp:70-73, multiply_rect.hpp:106-112)
    BT_REQUIRE(A.h_csz == B.h_rsz, BT_ERR_INVALID_ARGUMENT,
               "multiply: inner blockings of A and B differ");
    BT_REQUIRE(Cm.h_rsz == A.h_rsz && Cm.h_csz == B.h_csz, BT_ERR_INVALID_ARGUMENT,
               "multiply: C blockings do not conform");
    BT_REQUIRE(&Cm != &A && &Cm != &B, BT_ERR_INVALID_ARGUMENT,
               "multiply: C must not alias A or B");
    BT_CUDA(cudaSetDevice(x.device));
    cudaStream_t st = x.stream;
    const int64_t k0 = x.kernels;
    bt_stats S{};
    S.c_blocks_in = Cm.nblk;
    if (x.timing) BT_CUDA(cudaEventRecord(x.ev[0], st));
    const int64_t M = Cm.nbr, N = Cm.nbc, K = A.nbc;

    // ---- norms for the eps filter
    DBuf<double> na, nb;
    if (eps > 0 && A.nblk && B.nblk) {
      na.alloc(A.nblk, st);
      nb.alloc(B.nblk, st);
      k_block_norms<<<blocks_for(A.nblk, 128), 128, 0, st>>>(A.vals.p, A.row_ptr.p, A.col.p,
                                                              A.off.p, A.rsz.p, A.csz.p, A.nbr,
                                                              na.p, A.nblk);
      k_block_norms<<<blocks_for(B.nblk, 128), 128, 0, st>>>(B.vals.p, B.row_ptr.p, B.col.p,
                                                              B.off.p, B.rsz.p, B.csz.p, B.nbr,
                                                              nb.p, B.nblk);
      check_launch("block_norms");
      count_launch(&x, 2);
    }

    // ---- B column index (CSC): bc_ptr[N+1], bc_k (row k), bc_e (B entry)
    DBuf<int32_t> bc_ptr(N + 1, st), bc_k(std::max<int64_t>(B.nblk, 1), st),
        bc_e(std::max<int64_t>(B.nblk, 1), st);
    {
      DBuf<int32_t> colcnt(N + 1, st);
      BT_CUDA(cudaMemsetAsync(colcnt.p, 0, sizeof(int32_t) * (N + 1), st));
      if (B.nblk) {
        DBuf<int32_t> rows(B.nblk, st), idx(B.nblk, st);
        DBuf<uint64_t> keys(B.nblk, st), keys_s(B.nblk, st);
        k_expand_rows<<<blocks_for(B.nbr, 128), 128, 0, st>>>(B.row_ptr.p, B.nbr, rows.p);
        k_csc_keys<<<blocks_for(B.nblk, 256), 256, 0, st>>>(rows.p, B.col.p, B.nblk, keys.p,
                                                             idx.p, colcnt.p);
        check_launch("csc_keys");
        count_launch(&x, 2);
        int end_bit = 32;
        while (end_bit < 64 && (int64_t(1) << (end_bit - 32)) <= N) ++end_bit;
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, keys_s.p, idx.p, bc_e.p,
                                        B.nblk, 0, end_bit, st);
        void* tmp = x.ensure_scratch(bytes);
        cub::DeviceRadixSort::SortPairs(tmp, bytes, keys.p, keys_s.p, idx.p, bc_e.p, B.nblk, 0,
                                        end_bit, st);
        count_launch(&x, 4);
        k_csc_split<<<blocks_for(B.nblk, 256), 256, 0, st>>>(keys_s.p, B.nblk, bc_k.p);
        count_launch(&x);
      }
      exclusive_scan(x, colcnt.p, bc_ptr.p, N + 1);
    }

    // ---- symbolic: C_out pattern = C_in U products (get_or_create semantics)
    const int nwords = static_cast<int>((N + 31) / 32);
    BT_REQUIRE(static_cast<size_t>(nwords) * 4 * 2 <= x.smem_optin, BT_ERR_INVALID_ARGUMENT,
               "multiply: too many block columns for the symbolic bitmap");
    DBuf<int32_t> out_rp(M + 1, st), row_cnt(M + 1, st);
    DBuf<uint32_t> bm(std::max<int64_t>(M * nwords, 1), st);
    int64_t nout = 0;
    if (M > 0) {
      const size_t sm1 = static_cast<size_t>(nwords) * 4;
      if (sm1 > 48 * 1024)
        BT_CUDA(cudaFuncSetAttribute(k_sym_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sm1)));
      k_sym_count<<<static_cast<unsigned>(M), 256, sm1, st>>>(
          A.row_ptr.p, A.col.p, B.row_ptr.p, B.col.p, Cm.row_ptr.p, Cm.col.p, na.p, nb.p, eps,
          nwords, bm.p, row_cnt.p);
      check_launch("sym_count");
      count_launch(&x);
      BT_CUDA(cudaMemsetAsync(row_cnt.p + M, 0, sizeof(int32_t), st));
      exclusive_scan(x, row_cnt.p, out_rp.p, M + 1);
      nout = read_scalar(out_rp.p + M, st);
    } else {
      BT_CUDA(cudaMemsetAsync(out_rp.p, 0, sizeof(int32_t), st));
    }
    BT_REQUIRE(nout < (int64_t(1) << 31), BT_ERR_INVALID_ARGUMENT, "C exceeds 2^31 blocks");
    DBuf<int32_t> out_col(std::max<int64_t>(nout, 1), st), out_row(std::max<int64_t>(nout, 1), st);
    DBuf<int64_t> out_len(nout + 1, st), out_off(nout + 1, st), cin_map(std::max<int64_t>(nout, 1), st);
    int64_t nvals = 0, nelems = 0;
    DBuf<unsigned long long> d_elems(1, st);
    BT_CUDA(cudaMemsetAsync(d_elems.p, 0, sizeof(unsigned long long), st));
    if (nout > 0) {
      const size_t sm2 = static_cast<size_t>(nwords) * 4;
      if (sm2 > 48 * 1024)
        BT_CUDA(cudaFuncSetAttribute(k_sym_fill, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sm2)));
      k_sym_fill<<<static_cast<unsigned>(M), 256, sm2, st>>>(
          bm.p, nwords, out_rp.p, Cm.rsz.p, Cm.csz.p, Cm.row_ptr.p, Cm.col.p, Cm.off.p, out_col.p,
          out_row.p, out_len.p, cin_map.p, d_elems.p);
      check_launch("sym_fill");
      count_launch(&x);
      BT_CUDA(cudaMemsetAsync(out_len.p + nout, 0, sizeof(int64_t), st));
      exclusive_scan(x, out_len.p, out_off.p, nout + 1);
      nvals = read_scalar(out_off.p + nout, st);
      nelems = static_cast<int64_t>(read_scalar(d_elems.p, st));
    }
    bm.release();

    // ---- stacks: products per C block, k ascending
    DBuf<int32_t> cnt(std::max<int64_t>(nout, 1) + 1, st);
    DBuf<int64_t> stk_ptr(nout + 1, st);
    DBuf<unsigned long long> cand(2, st);
    BT_CUDA(cudaMemsetAsync(cand.p, 0, 2 * sizeof(unsigned long long), st));
    const bool use_kmap = static_cast<size_t>(K) * 4 <= std::min<size_t>(x.smem_optin, 96 * 1024);
    const size_t sm3 = use_kmap ? static_cast<size_t>(K) * 4 : 0;
    int64_t nprod = 0;
    if (nout > 0) {
      auto kc = use_kmap ? k_stack<false, true> : k_stack<false, false>;
      if (sm3 > 48 * 1024)
        BT_CUDA(cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sm3)));
      kc<<<static_cast<unsigned>(M), 128, sm3, st>>>(A.row_ptr.p, A.col.p, K, bc_ptr.p, bc_k.p,
                                                     bc_e.p, out_rp.p, out_col.p, na.p, nb.p,
                                                     eps, Cm.rsz.p, Cm.csz.p, A.csz.p, cnt.p,
                                                     cand.p, nullptr, nullptr, nullptr);
      check_launch("stack_count");
      count_launch(&x);
      BT_CUDA(cudaMemsetAsync(cnt.p + nout, 0, sizeof(int32_t), st));
      exclusive_scan(x, cnt.p, stk_ptr.p, nout + 1);
      nprod = read_scalar(stk_ptr.p + nout, st);
      unsigned long long tot[2];
      BT_CUDA(cudaMemcpyAsync(tot, cand.p, sizeof(tot), cudaMemcpyDeviceToHost, st));
      BT_CUDA(cudaStreamSynchronize(st));
      S.candidates = static_cast<int64_t>(tot[0]);
      S.flops = 2.0 * static_cast<double>(tot[1]);
    }
    S.products = nprod;
    DBuf<int32_t> stk_a(std::max<int64_t>(nprod, 1), st), stk_b(std::max<int64_t>(nprod, 1), st);
    if (nprod > 0) {
      auto kf = use_kmap ? k_stack<true, true> : k_stack<true, false>;
      if (sm3 > 48 * 1024)
        BT_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sm3)));
      kf<<<static_cast<unsigned>(M), 128, sm3, st>>>(A.row_ptr.p, A.col.p, K, bc_ptr.p, bc_k.p,
                                                     bc_e.p, out_rp.p, out_col.p, na.p, nb.p,
                                                     eps, nullptr, nullptr, nullptr, nullptr,
                                                     nullptr, stk_ptr.p, stk_a.p, stk_b.p);
      check_launch("stack_fill");
      count_launch(&x);
    }

    // ---- numeric phase
    DBuf<double> new_vals(std::max<int64_t>(nvals, 2), st);
    if (nout > 0) {
      const int kmax = A.max_c;
      const bool dmma_ok = kmax <= 64;
      DBuf<uint8_t> cls(nout, st), cls_s(nout, st);
      DBuf<int32_t> order(nout, st), order_s(nout, st), hist(NCLASS, st);
      BT_CUDA(cudaMemsetAsync(hist.p, 0, sizeof(int32_t) * NCLASS, st));
      k_classify<<<blocks_for(nout, 256), 256, 0, st>>>(out_row.p, out_col.p, Cm.rsz.p, Cm.csz.p,
                                                        nout, dmma_ok, cls.p, order.p, hist.p);
      check_launch("classify");
      count_launch(&x);
      std::array<int32_t, NCLASS> h_hist{};
      BT_CUDA(cudaMemcpyAsync(h_hist.data(), hist.p, sizeof(int32_t) * NCLASS,
                              cudaMemcpyDeviceToHost, st));
      BT_CUDA(cudaStreamSynchronize(st));
      int nclasses = 0;
      for (int q = 0; q < NCLASS; ++q) nclasses += h_hist[q] > 0;
      const int32_t* ord = order.p;
      const uint8_t* cl = cls.p;
      if (nclasses > 1) {
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, cls.p, cls_s.p, order.p, order_s.p,
                                        nout, 0, 5, st);
        void* tmp = x.ensure_scratch(bytes);
        cub::DeviceRadixSort::SortPairs(tmp, bytes, cls.p, cls_s.p, order.p, order_s.p, nout, 0,
                                        5, st);
        count_launch(&x, 2);
        ord = order_s.p;
        cl = cls_s.p;
      }
      DBuf<int32_t> ntiles(nout + 1, st);
      DBuf<int64_t> tstart(nout + 1, st);
      k_tiles<<<blocks_for(nout, 256), 256, 0, st>>>(ord, cl, out_row.p, Cm.rsz.p, nout, ntiles.p);
      count_launch(&x);
      BT_CUDA(cudaMemsetAsync(ntiles.p + nout, 0, sizeof(int32_t), st));
      exclusive_scan(x, ntiles.p, tstart.p, nout + 1);
      // class boundaries in entry space -> item space
      std::array<int64_t, NCLASS + 1> ebound{};
      for (int q = 0; q < NCLASS; ++q) ebound[q + 1] = ebound[q] + h_hist[q];
      std::array<int64_t, NCLASS + 1> ibound{};
      for (int q = 0; q <= NCLASS; ++q) {
        BT_CUDA(cudaMemcpyAsync(&ibound[q], tstart.p + ebound[q], sizeof(int64_t),
                                cudaMemcpyDeviceToHost, st));
      }
      BT_CUDA(cudaStreamSynchronize(st));
      const int64_t nitems = ibound[NCLASS];
      DBuf<int4> items(nitems, st);
      DBuf<int64_t> weight(nitems + 1, st), item_pp(nitems + 1, st);
      k_expand_items<<<blocks_for(nout, 256), 256, 0, st>>>(ord, out_row.p, ntiles.p, tstart.p,
                                                            cnt.p, nout, items.p, weight.p);
      count_launch(&x);
      BT_CUDA(cudaMemsetAsync(weight.p + nitems, 0, sizeof(int64_t), st));
      exclusive_scan(x, weight.p, item_pp.p, nitems + 1);

      NumArgs g{};
      g.items = items.p;
      g.item_pp = item_pp.p;
      g.stk_ptr = stk_ptr.p;
      g.stk_a = stk_a.p;
      g.stk_b = stk_b.p;
      g.a_vals = A.vals.p;
      g.a_off = A.off.p;
      g.a_col = A.col.p;
      g.k_sz = A.csz.p;
      g.b_vals = B.vals.p;
      g.b_off = B.off.p;
      g.m_sz = Cm.rsz.p;
      g.n_sz = Cm.csz.p;
      g.c_col = out_col.p;
      g.c_vals = new_vals.p;
      g.c_off = out_off.p;
      g.cin_map = cin_map.p;
      g.cin_vals = Cm.vals.p;
      if (x.timing) BT_CUDA(cudaEventRecord(x.ev[1], st));
      for (int q = 0; q < NCLASS; ++q) {
        const int64_t lo = ibound[q], hi = ibound[q + 1];
        if (hi <= lo) continue;
        g.item_lo = lo;
        g.item_hi = hi;
        if (q == GENERIC) {
          k_smm_generic<<<static_cast<unsigned>(hi - lo), 128, 0, st>>>(g);
          check_launch("smm_generic");
          count_launch(&x);
          continue;
        }
        const Launch L = plan_dmma(x, q, std::max(kmax, 1));
        g.stages = L.stages;
        g.stage_elems = L.stage_elems;
        g.a_region = L.a_region;
        KernelFn fn = dmma_kernel(q);
        BT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(L.smem)));
        int per_sm = 0;
        BT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, L.warps * 32, L.smem));
        per_sm = std::max(per_sm, 1);
        const int64_t want_warps = std::min<int64_t>(static_cast<int64_t>(x.num_sms) * per_sm * L.warps,
                                                     hi - lo);
        const unsigned grid = static_cast<unsigned>((want_warps + L.warps - 1) / L.warps);
        fn<<<grid, L.warps * 32, L.smem, st>>>(g);
        check_launch("smm_dmma");
        count_launch(&x);
      }
      if (x.timing) BT_CUDA(cudaEventRecord(x.ev[2], st));
    }

    // ---- install C_out
    Cm.vals = std::move(new_vals);
    Cm.row_ptr = std::move(out_rp);
    Cm.col = std::move(out_col);
    Cm.off = std::move(out_off);
    Cm.nblk = nout;
    Cm.nvals = nvals;
    Cm.nelems = nelems;
    if (x.timing) BT_CUDA(cudaEventRecord(x.ev[3], st));
    BT_CUDA(cudaStreamSynchronize(st));
    if (x.timing) {
      float ms = 0;
      if (nout > 0) {
        BT_CUDA(cudaEventElapsedTime(&ms, x.ev[1], x.ev[2]));
        S.ms_numeric = ms;
      }
      BT_CUDA(cudaEventElapsedTime(&ms, x.ev[0], x.ev[3]));
      S.ms_total = ms;
    }
    S.c_blocks_out = nout;
    S.kernels = static_cast<int32_t>(x.kernels - k0);
    if (stats) *stats = S;
  });
}
