// bt_tensor.cu -- tensor <-> matrix index remap (no reference
// code exists for the tensor module: parity is pinned to the written spec and a
// nested-loop dense oracle, DESIGN.md 3/6).
//
// A rank-n block-sparse tensor (n <= 4) is stored as a matrix under a
// matricization map: a row group and a column group of dimensions.  Block
// indices are mixed radix over each group with later-listed dimensions fastest
// (SPEC.md:505-513, 533); inside a block, elements follow the same rule, i.e.
// the matrix block is transpose(tensor_block, rows + cols).reshape(R, C) of the
// C-ordered tensor block.  bt_tensor_remap moves a tensor from one map to
// another entirely on the device: one pass computes the destination block keys,
// a radix sort builds the destination CSR, one kernel permutes the elements of
// every block.  This is the "tensor->matrix index-remap kernel" of the
// north_star; contract() in the Python layer uses it to bring operands into
// contraction-compatible layouts and then calls the block-sparse multiply.
#include <cub/cub.cuh>

#include <algorithm>
#include <numeric>

#include "bt_internal.cuh"

namespace bt {

constexpr int kMaxRank = 4;
#ifndef BT_REMAP_U
#define BT_REMAP_U 4
#endif

struct TensorMap {
  int ndim;
  int nr;                   // dims in the row group
  int dims[kMaxRank];       // row-group dims then col-group dims
};

struct TensorShape {
  int ndim;
  int64_t nb[kMaxRank];          // blocks per dimension
  const int32_t* sz[kMaxRank];   // device: block sizes per dimension
};

// block coords of a matrix (row, col) index pair under `map`
__device__ __forceinline__ void decompose(const TensorShape& s, const TensorMap& m, int64_t row,
                                          int64_t col, int64_t* coord) {
  for (int q = m.ndim - 1; q >= m.nr; --q) {
    const int d = m.dims[q];
    coord[d] = col % s.nb[d];
    col /= s.nb[d];
  }
  for (int q = m.nr - 1; q >= 0; --q) {
    const int d = m.dims[q];
    coord[d] = row % s.nb[d];
    row /= s.nb[d];
  }
}

__device__ __forceinline__ void compose(const TensorShape& s, const TensorMap& m,
                                        const int64_t* coord, int64_t& row, int64_t& col) {
  row = 0;
  col = 0;
  for (int q = 0; q < m.nr; ++q) row = row * s.nb[m.dims[q]] + coord[m.dims[q]];
  for (int q = m.nr; q < m.ndim; ++q) col = col * s.nb[m.dims[q]] + coord[m.dims[q]];
}

// destination key (row * ncols + col) of every source entry: one thread per
// stored block (its row by a binary search of the row pointer)
__global__ void k_remap_keys(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                             int64_t nbr, int64_t nblk, TensorShape s, TensorMap from,
                             TensorMap to, int64_t dst_nbc, uint64_t* __restrict__ keys,
                             int32_t* __restrict__ idx) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= nblk) return;
  int64_t lo = 0, hi = nbr;  // last row with rp[row] <= e
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (rp[mid] <= e) lo = mid; else hi = mid;
  }
  int64_t c[kMaxRank];
  decompose(s, from, lo, col[e], c);
  int64_t r2, c2;
  compose(s, to, c, r2, c2);
  keys[e] = static_cast<uint64_t>(r2 * dst_nbc + c2);
  idx[e] = static_cast<int32_t>(e);
}

// column of every sorted entry, per-row counts, T8 slot length and element count
__global__ void k_remap_rows(const uint64_t* __restrict__ keys, int64_t n, int64_t dst_nbc,
                             const int32_t* __restrict__ rsz, const int32_t* __restrict__ csz,
                             int32_t* __restrict__ row_cnt, int32_t* __restrict__ out_col,
                             int64_t* __restrict__ len, int64_t* __restrict__ elems) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > n) return;
  if (t == n) {  // scan sentinels: the totals land in element n
    len[n] = 0;
    elems[n] = 0;
    return;
  }
  const int64_t r = static_cast<int64_t>(keys[t] / dst_nbc), c = static_cast<int64_t>(keys[t] % dst_nbc);
  atomicAdd(&row_cnt[r], 1);
  out_col[t] = static_cast<int32_t>(c);
  len[t] = t8_size(rsz[r], csz[c]);
  elems[t] = static_cast<int64_t>(rsz[r]) * csz[c];
}

// Element permutation of one block, written in destination T8 storage order
// (coalesced stores, padding written as zeros) and gathered from the source
// block (L1/L2 resident).  The source position is separable:
//   r1 = RA[r2] + RB[c2],  c1 = CA[r2] + CB[c2]
// because a mixed-radix index is a sum of per-dimension terms and every
// dimension's element offset comes either from the destination row r2 or from
// the destination column c2.  The four tables are built per block in shared
// memory (R2 + C2 entries each), so the inner loop is two lookups and adds.
// tab_n: entries per table (dynamic shared memory 16 * tab_n bytes), at least
// the largest R2 and C2 of the launch; 0 = no tables (per-element decomposition)
constexpr int kRemapTabMax = 3072;
__global__ void __launch_bounds__(128) k_remap_vals(
    const uint64_t* __restrict__ keys, const int32_t* __restrict__ src_e,
    const int64_t* __restrict__ src_off, const int64_t* __restrict__ dst_off, int64_t n,
    int64_t dst_nbc, TensorShape s, TensorMap from, TensorMap to, const double* __restrict__ src,
    double* __restrict__ dst, int tab_n) {
  extern __shared__ int32_t tab[];
  const int64_t t = blockIdx.x;
  if (t >= n) return;
  int64_t c[kMaxRank];
  decompose(s, to, static_cast<int64_t>(keys[t] / dst_nbc), static_cast<int64_t>(keys[t] % dst_nbc), c);
  int ext[kMaxRank];
  for (int d = 0; d < s.ndim; ++d) ext[d] = s.sz[d][c[d]];
  // block shapes under both maps; strides of every dim in the source map
  int C1 = 1, R2 = 1, C2 = 1;
  int sr[kMaxRank] = {0, 0, 0, 0}, sc[kMaxRank] = {0, 0, 0, 0};
  for (int q = from.ndim - 1, acc = 1; q >= from.nr; --q) {
    sc[from.dims[q]] = acc;
    acc *= ext[from.dims[q]];
    C1 = acc;
  }
  for (int q = from.nr - 1, acc = 1; q >= 0; --q) {
    sr[from.dims[q]] = acc;
    acc *= ext[from.dims[q]];
  }
  for (int q = 0; q < to.ndim; ++q) (q < to.nr ? R2 : C2) *= ext[to.dims[q]];
  const double* sb = src + src_off[src_e[t]];
  double* db = dst + dst_off[t];
  const int ntc1 = tiles8(C1), ntc2 = tiles8(C2);
  const int64_t slot = static_cast<int64_t>(tiles8(R2)) * ntc2 * 64;
  auto row_terms = [&](int r2, int& ra, int& ca) {  // dst row -> source row/col terms
    ra = 0;
    ca = 0;
    for (int q = to.nr - 1; q >= 0; --q) {
      const int d = to.dims[q];
      const int o = r2 % ext[d];
      r2 /= ext[d];
      ra += o * sr[d];
      ca += o * sc[d];
    }
  };
  auto col_terms = [&](int c2, int& rb, int& cb) {
    rb = 0;
    cb = 0;
    for (int q = to.ndim - 1; q >= to.nr; --q) {
      const int d = to.dims[q];
      const int o = c2 % ext[d];
      c2 /= ext[d];
      rb += o * sr[d];
      cb += o * sc[d];
    }
  };
  const bool tables = R2 <= tab_n && C2 <= tab_n;
  int32_t *RA = tab, *CA = tab + tab_n, *RB = tab + 2 * tab_n, *CB = tab + 3 * tab_n;
  if (tables) {
    for (int r = threadIdx.x; r < R2; r += blockDim.x) row_terms(r, RA[r], CA[r]);
    for (int q = threadIdx.x; q < C2; q += blockDim.x) col_terms(q, RB[q], CB[q]);
    __syncthreads();
  }
  // destination tiles in storage order, blockDim / 64 tiles per sweep: lane w
  // of a 64-thread group always handles element w of its tile (fixed row rr
  // and swizzled column cc), tile coordinates advance incrementally (32-bit,
  // no division in the loop)
  const int ntiles = tiles8(R2) * ntc2;
  const int w = threadIdx.x & 63;
  const int rr = w >> 3;
  const int cc = (w & 7) ^ (((rr >> 1) & 1) << 2);  // the T8 swizzle is an involution
  const int step = blockDim.x >> 6;
  // four tiles per thread and sweep: the four gathers are issued together
  // (the kernel is bound by gather latency, ncu: long-scoreboard stalls)
  constexpr int U = BT_REMAP_U;
  for (int t0 = threadIdx.x >> 6; t0 < ntiles; t0 += U * step) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int tl = t0 + u * step;
      v[u] = 0.0;
      if (tl < ntiles) {
        const int tr = tl / ntc2, tc = tl - tr * ntc2;
        const int r2 = tr * 8 + rr, c2 = tc * 8 + cc;
        if (r2 < R2 && c2 < C2) {
          int ra, ca, rb, cb;
          if (tables) {
            ra = RA[r2];
            ca = CA[r2];
            rb = RB[c2];
            cb = CB[c2];
          } else {
            row_terms(r2, ra, ca);
            col_terms(c2, rb, cb);
          }
          const int r1 = ra + rb, c1 = ca + cb;
          v[u] = __ldg(sb + (((r1 >> 3) * ntc1 + (c1 >> 3)) << 6) + ((r1 & 7) << 3) +
                       ((c1 & 7) ^ (((r1 >> 1) & 1) << 2)));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int tl = t0 + u * step;
      if (tl < ntiles) __stcs(db + (static_cast<int64_t>(tl) << 6) + w, v[u]);
    }
  }
  (void)slot;
}

}  // namespace bt

using namespace bt;

extern "C" int bt_tensor_remap(bt_ctx* ctx, int ndim, const int64_t* nblocks,
                               const int32_t* const* dim_sizes, int src_nrow,
                               const int* src_dims, const bt_mat* src, int dst_nrow,
                               const int* dst_dims, bt_mat* dst) {
  return guard([&] {
    BT_REQUIRE(ctx && src && dst && nblocks && dim_sizes && src_dims && dst_dims,
               BT_ERR_INVALID_ARGUMENT, "null argument");
    BT_REQUIRE(ndim >= 2 && ndim <= kMaxRank, BT_ERR_INVALID_ARGUMENT,
               "tensor: rank must be in [2, 4]");
    Ctx& x = ctx->impl;
    const Mat& S = src->impl;
    Mat& D = dst->impl;
    cudaStream_t st = x.stream;
    auto check_map = [&](int nrow, const int* dims, const char* who) {
      BT_REQUIRE(nrow >= 1 && nrow < ndim, BT_ERR_INVALID_ARGUMENT,
                 std::string(who) + ": row and column groups must both be non-empty");
      std::vector<int> seen(ndim, 0);
      for (int q = 0; q < ndim; ++q) {
        BT_REQUIRE(dims[q] >= 0 && dims[q] < ndim && !seen[dims[q]], BT_ERR_INVALID_ARGUMENT,
                   std::string(who) + ": map is not a partition of the dimensions");
        seen[dims[q]] = 1;
      }
    };
    check_map(src_nrow, src_dims, "tensor_remap(src)");
    check_map(dst_nrow, dst_dims, "tensor_remap(dst)");
    TensorShape s{};
    s.ndim = ndim;
    std::vector<DBuf<int32_t>> dsz(ndim);
    for (int d = 0; d < ndim; ++d) {
      s.nb[d] = nblocks[d];
      dsz[d].alloc(std::max<int64_t>(nblocks[d], 1), st);
      BT_CUDA(cudaMemcpyAsync(dsz[d].p, dim_sizes[d], 4 * nblocks[d], cudaMemcpyHostToDevice, st));
      s.sz[d] = dsz[d].p;
    }
    TensorMap from{ndim, src_nrow, {0, 0, 0, 0}}, to{ndim, dst_nrow, {0, 0, 0, 0}};
    for (int q = 0; q < ndim; ++q) {
      from.dims[q] = src_dims[q];
      to.dims[q] = dst_dims[q];
    }
    // blockings must be the ones the maps induce
    auto group_blocks = [&](const TensorMap& m, bool rows) {
      int64_t n = 1;
      for (int q = rows ? 0 : m.nr; q < (rows ? m.nr : m.ndim); ++q) n *= nblocks[m.dims[q]];
      return n;
    };
    BT_REQUIRE(S.nbr == group_blocks(from, true) && S.nbc == group_blocks(from, false),
               BT_ERR_INVALID_ARGUMENT, "tensor_remap: source blockings do not match its map");
    BT_REQUIRE(D.nbr == group_blocks(to, true) && D.nbc == group_blocks(to, false),
               BT_ERR_INVALID_ARGUMENT, "tensor_remap: target blockings do not match its map");
    BT_REQUIRE(D.nbr * D.nbc < (int64_t(1) << 62), BT_ERR_INVALID_ARGUMENT, "tensor too large");
    const int64_t n = S.nblk;
    if (n == 0) {
      D.init_empty();
      return;
    }
    DBuf<uint64_t> keys(n, st), keys_s(n, st);
    DBuf<int32_t> idx(n, st), idx_s(n, st);
    k_remap_keys<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(
        S.row_ptr.p, S.col.p, S.nbr, n, s, from, to, D.nbc, keys.p, idx.p);
    check_launch("remap_keys");
    int end_bit = 1;
    while (end_bit < 64 && (uint64_t(1) << end_bit) < static_cast<uint64_t>(D.nbr * D.nbc)) ++end_bit;
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, keys_s.p, idx.p, idx_s.p, n, 0, end_bit, st);
    void* tmp = x.ensure_scratch(bytes);
    cub::DeviceRadixSort::SortPairs(tmp, bytes, keys.p, keys_s.p, idx.p, idx_s.p, n, 0, end_bit, st);
    DBuf<int32_t> cnt(D.nbr + 1, st), rp(D.nbr + 1, st), col(n, st);
    DBuf<int64_t> len(n + 1, st), el(n + 1, st), d_off(n + 1, st), d_el(n + 1, st);
    BT_CUDA(cudaMemsetAsync(cnt.p, 0, 4 * (D.nbr + 1), st));
    k_remap_rows<<<static_cast<unsigned>((n + 256) / 256), 256, 0, st>>>(
        keys_s.p, n, D.nbc, D.rsz.p, D.csz.p, cnt.p, col.p, len.p, el.p);
    check_launch("remap_rows");
    auto scan = [&](auto* in, auto* out, int64_t m) {
      size_t b2 = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, b2, in, out, m, st);
      void* t2 = x.ensure_scratch(b2);
      cub::DeviceScan::ExclusiveSum(t2, b2, in, out, m, st);
    };
    scan(cnt.p, rp.p, D.nbr + 1);
    scan(len.p, d_off.p, n + 1);   // destination T8 offsets; [n] = slab length
    scan(el.p, d_el.p, n + 1);     // [n] = stored elements
    int64_t tot[2];
    BT_CUDA(cudaMemcpyAsync(&tot[0], d_off.p + n, 8, cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaMemcpyAsync(&tot[1], d_el.p + n, 8, cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaStreamSynchronize(st));
    const int64_t nv = tot[0], ne = tot[1];
    DBuf<double> vals(std::max<int64_t>(nv, 64), st);
    // every destination slot is written in full (padding as zeros): no memset
    // per-block lookup tables sized for the largest destination block of the
    // launch (from the per-dimension maximum block sizes)
    int64_t max_r = 1, max_c = 1;
    for (int q = 0; q < ndim; ++q) {
      const int d = dst_dims[q];
      const int32_t mx = nblocks[d] ? *std::max_element(dim_sizes[d], dim_sizes[d] + nblocks[d]) : 1;
      (q < dst_nrow ? max_r : max_c) *= mx;
    }
    const int64_t tab_want = std::max(max_r, max_c);
    const int tab_n = tab_want <= kRemapTabMax ? static_cast<int>(tab_want) : 0;
    k_remap_vals<<<static_cast<unsigned>(n), 128, 16 * static_cast<size_t>(tab_n), st>>>(
        keys_s.p, idx_s.p, S.off.p, d_off.p, n, D.nbc, s, from, to, S.vals.p, vals.p, tab_n);
    check_launch("remap_vals");
    count_launch(&x, 8);
    D.vals = std::move(vals);
    D.row_ptr = std::move(rp);
    D.col = std::move(col);
    D.off = std::move(d_off);
    D.nblk = n;
    D.norms_ok = false;
    D.nvals = nv;
    D.nelems = ne;
    BT_CUDA(cudaStreamSynchronize(st));
  });
}
