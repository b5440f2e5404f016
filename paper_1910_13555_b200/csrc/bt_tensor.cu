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

// destination key (row * ncols + col) of every source entry
__global__ void k_remap_keys(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                             int64_t nbr, TensorShape s, TensorMap from, TensorMap to,
                             int64_t dst_nbc, uint64_t* __restrict__ keys,
                             int32_t* __restrict__ idx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nbr) return;
  for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
    int64_t c[kMaxRank];
    decompose(s, from, i, col[e], c);
    int64_t r2, c2;
    compose(s, to, c, r2, c2);
    keys[e] = static_cast<uint64_t>(r2 * dst_nbc + c2);
    idx[e] = static_cast<int32_t>(e);
  }
}

__global__ void k_remap_rows(const uint64_t* __restrict__ keys, int64_t n, int64_t dst_nbc,
                             int32_t* __restrict__ row_cnt, int32_t* __restrict__ out_col) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  atomicAdd(&row_cnt[keys[t] / dst_nbc], 1);
  out_col[t] = static_cast<int32_t>(keys[t] % dst_nbc);
}

// element permutation of one block: destination (r2, c2) <- source (r, c)
__global__ void k_remap_vals(const uint64_t* __restrict__ keys, const int32_t* __restrict__ src_e,
                             const int64_t* __restrict__ src_off, const int64_t* __restrict__ dst_off,
                             int64_t n, int64_t dst_nbc, TensorShape s, TensorMap from,
                             TensorMap to, const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t t = blockIdx.x;
  if (t >= n) return;
  int64_t c[kMaxRank];
  decompose(s, to, static_cast<int64_t>(keys[t] / dst_nbc), static_cast<int64_t>(keys[t] % dst_nbc), c);
  int ext[kMaxRank];
  int total = 1;
  for (int d = 0; d < s.ndim; ++d) {
    ext[d] = s.sz[d][c[d]];
    total *= ext[d];
  }
  // block shapes under both maps
  int R1 = 1, C1 = 1, R2 = 1, C2 = 1;
  for (int q = 0; q < from.ndim; ++q) (q < from.nr ? R1 : C1) *= ext[from.dims[q]];
  for (int q = 0; q < to.ndim; ++q) (q < to.nr ? R2 : C2) *= ext[to.dims[q]];
  const double* sb = src + src_off[src_e[t]];
  double* db = dst + dst_off[t];
  const int ntc1 = tiles8(C1), ntc2 = tiles8(C2);
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    // element offsets per dim from the destination (row, col) of e
    const int r2 = e / C2, c2 = e - r2 * C2;
    int o[kMaxRank];
    int rr = r2, cc = c2;
    for (int q = to.ndim - 1; q >= to.nr; --q) {
      const int d = to.dims[q];
      o[d] = cc % ext[d];
      cc /= ext[d];
    }
    for (int q = to.nr - 1; q >= 0; --q) {
      const int d = to.dims[q];
      o[d] = rr % ext[d];
      rr /= ext[d];
    }
    int r1 = 0, c1 = 0;
    for (int q = 0; q < from.nr; ++q) r1 = r1 * ext[from.dims[q]] + o[from.dims[q]];
    for (int q = from.nr; q < from.ndim; ++q) c1 = c1 * ext[from.dims[q]] + o[from.dims[q]];
    db[t8_pos(r2, c2, ntc2)] = sb[t8_pos(r1, c1, ntc1)];
  }
  (void)R1;
  (void)R2;
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
    k_remap_keys<<<static_cast<unsigned>((S.nbr + 127) / 128), 128, 0, st>>>(
        S.row_ptr.p, S.col.p, S.nbr, s, from, to, D.nbc, keys.p, idx.p);
    check_launch("remap_keys");
    int end_bit = 1;
    while (end_bit < 64 && (uint64_t(1) << end_bit) < static_cast<uint64_t>(D.nbr * D.nbc)) ++end_bit;
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, keys_s.p, idx.p, idx_s.p, n, 0, end_bit, st);
    void* tmp = x.ensure_scratch(bytes);
    cub::DeviceRadixSort::SortPairs(tmp, bytes, keys.p, keys_s.p, idx.p, idx_s.p, n, 0, end_bit, st);
    DBuf<int32_t> cnt(D.nbr + 1, st), rp(D.nbr + 1, st), col(n, st);
    BT_CUDA(cudaMemsetAsync(cnt.p, 0, 4 * (D.nbr + 1), st));
    k_remap_rows<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(keys_s.p, n, D.nbc, cnt.p,
                                                                         col.p);
    {
      size_t b2 = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, b2, cnt.p, rp.p, D.nbr + 1, st);
      void* t2 = x.ensure_scratch(b2);
      cub::DeviceScan::ExclusiveSum(t2, b2, cnt.p, rp.p, D.nbr + 1, st);
    }
    // destination offsets: host pass over the sorted keys (index-sized work)
    std::vector<uint64_t> hk(n);
    BT_CUDA(cudaMemcpyAsync(hk.data(), keys_s.p, 8 * n, cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaStreamSynchronize(st));
    std::vector<int64_t> off(n);
    int64_t nv = 0, ne = 0;
    for (int64_t t = 0; t < n; ++t) {
      const int64_t r = static_cast<int64_t>(hk[t] / D.nbc), c = static_cast<int64_t>(hk[t] % D.nbc);
      off[t] = nv;
      nv += t8_size(D.h_rsz[r], D.h_csz[c]);
      ne += int64_t(D.h_rsz[r]) * D.h_csz[c];
    }
    DBuf<int64_t> d_off(n, st);
    BT_CUDA(cudaMemcpyAsync(d_off.p, off.data(), 8 * n, cudaMemcpyHostToDevice, st));
    DBuf<double> vals(std::max<int64_t>(nv, 64), st);
    BT_CUDA(cudaMemsetAsync(vals.p, 0, 8 * std::max<int64_t>(nv, 64), st));
    k_remap_vals<<<static_cast<unsigned>(n), 128, 0, st>>>(keys_s.p, idx_s.p, S.off.p, d_off.p, n,
                                                           D.nbc, s, from, to, S.vals.p, vals.p);
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
