// bt_dist.cu -- distributed layer: process group + ledger (SimComm, comm.hpp:152-397),
// distributed matrix (DistMatrix, matrix.hpp:279-401), redistribution
// (matrix.hpp:545-622) and the three multiply drivers (multiply_cannon.hpp:62-118,
// multiply_rect.hpp:123-250), B200-native.
//
// Ranks and transports:
//  * NCCL: one process per GPU (torchrun); every message is a whole block-CSR
//    store (the device analogue of Packet{values, meta}, matrix.hpp:503-513): a
//    3-word header, then row_ptr / col / off / T8 values, as grouped
//    ncclSend/ncclRecv on a dedicated comm stream so Cannon's shifts overlap the
//    local multiply (send-before-compute, multiply_cannon.hpp:106-116).
//  * Local: all ranks of the group live in this process on the context's GPU
//    ("virtual ranks"); a message is a device copy.  Same algorithms, same
//    ledger -- used to test every driver against the reference on one GPU.
// The algorithms are written bulk-synchronously over the ranks this process
// owns, so both transports run the same code.  The ledger charges exactly what
// the reference's Ledger charges: matrix elements and 4 meta words per block
// for every message between distinct ranks.
#include <nccl.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <functional>
#include <map>
#include <memory>
#include <numeric>

#include "bt_internal.cuh"

namespace bt {

// =============================================================== store kernels
// owner rank of each entry under a layout; transpose swaps (i, j) first
__global__ void k_owner(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                        int64_t nbr, const int32_t* __restrict__ rdist,
                        const int32_t* __restrict__ cdist, int gcols, int transpose,
                        int32_t* __restrict__ owner) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nbr) return;
  for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
    const int64_t r = transpose ? col[e] : i, c = transpose ? i : col[e];
    owner[e] = rdist[r] * gcols + cdist[c];
  }
}

// Merge contributions into a new store.  Output block b gathers contributions
// [seg[b], seg[b+1]) (stable key order); contribution t has source pointer
// srcp[t] (a T8 block, stored transposed when tr[t]).  The first contribution
// initialises the block, later ones are added (accumulate) -- or only the last
// one is taken (replace).
__global__ void k_merge_vals(const int64_t* __restrict__ key, const int64_t* __restrict__ seg,
                             int64_t nout, const double* const* __restrict__ srcp,
                             const uint8_t* __restrict__ tr, int64_t nbc,
                             const int32_t* __restrict__ rsz, const int32_t* __restrict__ csz,
                             const int64_t* __restrict__ out_off, int accumulate,
                             double* __restrict__ out) {
  const int64_t b = blockIdx.x;
  if (b >= nout) return;
  const int64_t t0 = seg[b], t1 = seg[b + 1];
  const int64_t k = key[t0];
  const int m = rsz[k / nbc], n = csz[k % nbc];
  const int ntc = tiles8(n), ntr = tiles8(m);
  double* d = out + out_off[b];
  const int64_t first = accumulate ? t0 : t1 - 1;  // replace: the last contribution wins
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int r = e / n, c = e - r * n;
    double v = 0.0;
    for (int64_t t = first; t < t1; ++t) {
      // transposed sources are stored as the n x m block
      const double x = tr[t] ? srcp[t][t8_pos(c, r, ntr)] : srcp[t][t8_pos(r, c, ntc)];
      v = (t == first) ? x : __dadd_rn(v, x);
    }
    d[t8_pos(r, c, ntc)] = v;
  }
}

// select entries with owner == target into compact index lists
__global__ void k_flag_owner(const int32_t* __restrict__ owner, int64_t n, int target,
                             int32_t* __restrict__ flag) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  flag[e] = owner[e] == target ? 1 : 0;
}

__global__ void k_gather_sel(const int32_t* __restrict__ flag, const int32_t* __restrict__ fscan,
                             int64_t n, int64_t* __restrict__ sel) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  if (flag[e]) sel[fscan[e]] = e;
}

// ================================================================ host utils
namespace {

inline unsigned nb(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

template <class TIn, class TOut>
void dscan(Ctx& x, const TIn* in, TOut* out, int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, x.stream);
  void* tmp = x.ensure_scratch(bytes);
  cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, n, x.stream);
  count_launch(&x, 2);
}

template <class T>
T readback(const T* d, cudaStream_t s) {
  T v;
  BT_CUDA(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  BT_CUDA(cudaStreamSynchronize(s));
  return v;
}

}  // namespace

// A contribution to a merge: the blocks `sel` (entry indices; all when null) of
// `src`, optionally transposed.
struct Contribution {
  const Mat* src;
  const int64_t* sel;  // device entry indices, or null for all entries
  int64_t n;           // number of entries
  bool transpose;
};

// Device side of merge_into: one thread per contributed entry writes its
// destination key, its position in contribution order, the source block pointer
// and the transposed flag at [base, base + n).
__global__ void k_merge_keys(const int32_t* __restrict__ rp, int64_t nbr,
                             const int32_t* __restrict__ col, const int64_t* __restrict__ off,
                             const double* vals, const int64_t* __restrict__ sel, int64_t n,
                             int tr, int64_t nbc, int64_t base, int64_t* __restrict__ key,
                             int64_t* __restrict__ pos, const double** __restrict__ src,
                             uint8_t* __restrict__ trf) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int64_t e = sel ? sel[q] : q;
  int64_t lo = 0, hi = nbr;  // row = last i with rp[i] <= e
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (rp[mid] <= e) lo = mid; else hi = mid;
  }
  const int64_t i = lo, j = col[e];
  key[base + q] = tr ? j * nbc + i : i * nbc + j;
  pos[base + q] = base + q;
  src[base + q] = vals + off[e];
  trf[base + q] = static_cast<uint8_t>(tr);
}

// Over the key-sorted contributions: segment heads, their T8 value sizes and
// element counts (zero elsewhere), and the sources/flags in sorted order.
__global__ void k_merge_heads(const int64_t* __restrict__ skey, const int64_t* __restrict__ spos,
                              int64_t total, int64_t nbc, const int32_t* __restrict__ rsz,
                              const int32_t* __restrict__ csz, const double* const* __restrict__ src,
                              const uint8_t* __restrict__ trf, int32_t* __restrict__ head,
                              int64_t* __restrict__ vsz, int64_t* __restrict__ esz,
                              const double** __restrict__ ssrc, uint8_t* __restrict__ strf) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > total) return;
  if (t == total) {  // trailing zero: the exclusive scans' last element is the total
    head[t] = 0;
    vsz[t] = 0;
    esz[t] = 0;
    return;
  }
  const int64_t k = skey[t];
  const bool h = t == 0 || skey[t - 1] != k;
  const int m = rsz[k / nbc], n = csz[k % nbc];
  head[t] = h ? 1 : 0;
  vsz[t] = h ? t8_size(m, n) : 0;
  esz[t] = h ? int64_t(m) * n : 0;
  ssrc[t] = src[spos[t]];
  strf[t] = trf[spos[t]];
}

// Compacts the heads into the output index (col, off, segment start, key) and
// writes the totals (blocks, values, elements) for the host.
__global__ void k_merge_compact(const int64_t* __restrict__ skey, int64_t total,
                                const int32_t* __restrict__ head, const int32_t* __restrict__ hscan,
                                const int64_t* __restrict__ vscan, const int64_t* __restrict__ escan,
                                int64_t nbc, int32_t* __restrict__ ocol, int64_t* __restrict__ ooff,
                                int64_t* __restrict__ oseg, int64_t* __restrict__ okey,
                                int64_t* __restrict__ totals) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t == 0) {
    totals[0] = hscan[total];
    totals[1] = vscan[total];
    totals[2] = escan[total];
    oseg[hscan[total]] = total;
  }
  if (t >= total || !head[t]) return;
  const int64_t u = hscan[t];
  ocol[u] = static_cast<int32_t>(skey[t] % nbc);
  ooff[u] = vscan[t];
  oseg[u] = t;
  okey[u] = skey[t];
}

// row_ptr[i] = first output block with key >= i * nbc
__global__ void k_merge_rowptr(const int64_t* __restrict__ okey, const int64_t* __restrict__ totals,
                               int64_t nbr, int64_t nbc, int32_t* __restrict__ rp) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > nbr) return;
  const int64_t target = i * nbc;
  int64_t lo = 0, hi = totals[0];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (okey[mid] < target) lo = mid + 1; else hi = mid;
  }
  rp[i] = static_cast<int32_t>(lo);
}

// Builds dst := (accumulate ? dst : {}) merged with the contributions, in order.
// Blocks present in several contributions are summed in contribution order
// (accumulate) or the last one wins (LocalStore::insert, matrix.hpp:167-189).
// All index work is on the device (stable radix sort by destination key); the
// host reads back the three totals once, to size the value buffer.
void merge_into(Mat& dst, const std::vector<Contribution>& parts, bool accumulate) {
  Ctx& x = *dst.ctx;
  cudaStream_t st = x.stream;
  const int64_t nbc = dst.nbc;
  int64_t total = accumulate ? dst.nblk : 0;
  for (const auto& p : parts) total += p.n;
  if (total == 0) {
    dst.init_empty();
    return;
  }
  DBuf<int64_t> key(total, st), skey(total, st), pos(total, st), spos(total, st);
  DBuf<const double*> src(total, st), ssrc(total, st);
  DBuf<uint8_t> trf(total, st), strf(total, st);
  int64_t base = 0;
  auto add_part = [&](const Mat& m, const int64_t* sel, int64_t n, bool tr) {
    if (n == 0) return;
    k_merge_keys<<<nb(n, 256), 256, 0, st>>>(m.row_ptr.p, m.nbr, m.col.p, m.off.p, m.vals.p, sel,
                                             n, tr ? 1 : 0, nbc, base, key.p, pos.p, src.p, trf.p);
    check_launch("merge_keys");
    count_launch(&x);
    base += n;
  };
  if (accumulate) add_part(dst, nullptr, dst.nblk, false);
  for (const auto& p : parts) add_part(*p.src, p.sel, p.n, p.transpose);
  // stable (radix) sort by key keeps contribution order within a block
  const uint64_t kmax = static_cast<uint64_t>(std::max<int64_t>(dst.nbr * nbc, 1));
  const int end_bit = std::max(1, 64 - __builtin_clzll(kmax));
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, skey.p, pos.p, spos.p, total, 0, end_bit,
                                  st);
  void* tmp = x.ensure_scratch(bytes);
  cub::DeviceRadixSort::SortPairs(tmp, bytes, key.p, skey.p, pos.p, spos.p, total, 0, end_bit, st);
  count_launch(&x, 4);
  DBuf<int32_t> head(total + 1, st), hscan(total + 1, st);
  DBuf<int64_t> vsz(total + 1, st), vscan(total + 1, st), esz(total + 1, st), escan(total + 1, st);
  k_merge_heads<<<nb(total + 1, 256), 256, 0, st>>>(skey.p, spos.p, total, nbc, dst.rsz.p,
                                                    dst.csz.p, src.p, trf.p, head.p, vsz.p, esz.p,
                                                    ssrc.p, strf.p);
  check_launch("merge_heads");
  count_launch(&x);
  dscan(x, head.p, hscan.p, total + 1);
  dscan(x, vsz.p, vscan.p, total + 1);
  dscan(x, esz.p, escan.p, total + 1);
  // outputs sized for the worst case (every contribution its own block)
  DBuf<int32_t> cl(total, st), rp(dst.nbr + 1, st);
  DBuf<int64_t> of(total, st), seg(total + 1, st), okey(total, st), tot(3, st);
  k_merge_compact<<<nb(total, 256), 256, 0, st>>>(skey.p, total, head.p, hscan.p, vscan.p,
                                                  escan.p, nbc, cl.p, of.p, seg.p, okey.p, tot.p);
  check_launch("merge_compact");
  k_merge_rowptr<<<nb(dst.nbr + 1, 256), 256, 0, st>>>(okey.p, tot.p, dst.nbr, nbc, rp.p);
  check_launch("merge_rowptr");
  count_launch(&x, 2);
  int64_t h_tot[3];
  BT_CUDA(cudaMemcpyAsync(h_tot, tot.p, sizeof(h_tot), cudaMemcpyDeviceToHost, st));
  BT_CUDA(cudaStreamSynchronize(st));
  const int64_t nout = h_tot[0], nv = h_tot[1], ne = h_tot[2];
  DBuf<double> vals(std::max<int64_t>(nv, 64), st);
  BT_CUDA(cudaMemsetAsync(vals.p, 0, 8 * std::max<int64_t>(nv, 64), st));  // T8 padding = 0
  k_merge_vals<<<static_cast<unsigned>(nout), 128, 0, st>>>(skey.p, seg.p, nout, ssrc.p, strf.p,
                                                            nbc, dst.rsz.p, dst.csz.p, of.p,
                                                            accumulate ? 1 : 0, vals.p);
  check_launch("merge_vals");
  count_launch(&x);
  BT_CUDA(cudaStreamSynchronize(st));  // sources may be released by the caller
  dst.vals = std::move(vals);
  dst.row_ptr = std::move(rp);
  dst.col = std::move(cl);
  dst.off = std::move(of);
  dst.nblk = nout;
  dst.norms_ok = false;
  dst.nvals = nv;
  dst.nelems = ne;
}

// entry indices (device) of the entries of `m` whose owner (under the layout,
// optionally transposed) is `target`; returns the count
int64_t select_owned(Mat& m, const int32_t* d_owner, int target, DBuf<int64_t>& sel) {
  Ctx& x = *m.ctx;
  cudaStream_t st = x.stream;
  if (m.nblk == 0) return 0;
  DBuf<int32_t> flag(m.nblk + 1, st), fscan(m.nblk + 1, st);
  k_flag_owner<<<nb(m.nblk, 256), 256, 0, st>>>(d_owner, m.nblk, target, flag.p);
  BT_CUDA(cudaMemsetAsync(flag.p + m.nblk, 0, 4, st));
  dscan(x, flag.p, fscan.p, m.nblk + 1);
  const int64_t n = readback(fscan.p + m.nblk, st);
  sel.alloc(std::max<int64_t>(n, 1), st);
  k_gather_sel<<<nb(m.nblk, 256), 256, 0, st>>>(flag.p, fscan.p, m.nblk, sel.p);
  count_launch(&x, 2);
  return n;
}

// ---- one-pass split of a store by owner (non-transposed redistribute)
// Per entry: its row, the sort key (owner) and identity payload; per owner: the
// entry, value and element totals.
__global__ void k_split_hist(const int32_t* __restrict__ rp, int64_t nbr,
                             const int32_t* __restrict__ col, const int32_t* __restrict__ owner,
                             const int32_t* __restrict__ rsz, const int32_t* __restrict__ csz,
                             int P, int32_t* __restrict__ row_of, int32_t* __restrict__ ident,
                             unsigned long long* __restrict__ hist) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nbr) return;
  for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
    const int m = rsz[i], n = csz[col[e]], d = owner[e];
    row_of[e] = static_cast<int32_t>(i);
    ident[e] = e;
    atomicAdd(&hist[d], 1ull);
    atomicAdd(&hist[P + d], static_cast<unsigned long long>(t8_size(m, n)));
    atomicAdd(&hist[2 * P + d], static_cast<unsigned long long>(m) * n);
  }
}

// T8 value sizes of the owner-sorted entries (plus a trailing zero)
__global__ void k_split_vsz(const int32_t* __restrict__ ord, int64_t n,
                            const int32_t* __restrict__ row_of, const int32_t* __restrict__ col,
                            const int32_t* __restrict__ rsz, const int32_t* __restrict__ csz,
                            int64_t* __restrict__ vsz) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > n) return;
  if (t == n) { vsz[t] = 0; return; }
  const int32_t e = ord[t];
  vsz[t] = t8_size(rsz[row_of[e]], csz[col[e]]);
}

// One bucket: entries ord[t0, t0 + n) (key order) -> col/off, values copied
// warp per block.
__global__ void k_split_fill(const int32_t* __restrict__ ord, int64_t t0, int64_t n,
                             const int32_t* __restrict__ col, const int64_t* __restrict__ off,
                             const double* __restrict__ vals, const int64_t* __restrict__ vscan,
                             int32_t* __restrict__ bcol, int64_t* __restrict__ boff,
                             double* __restrict__ bvals) {
  const int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= n) return;
  const int32_t e = ord[t0 + q];
  const int64_t o = vscan[t0 + q] - vscan[t0], len = vscan[t0 + q + 1] - vscan[t0 + q];
  if (lane == 0) {
    bcol[q] = col[e];
    boff[q] = o;
  }
  const double2* s2 = reinterpret_cast<const double2*>(vals + off[e]);
  double2* d2 = reinterpret_cast<double2*>(bvals + o);
  for (int64_t k = lane; k < len / 2; k += 32) d2[k] = s2[k];
}

// bucket row_ptr[i] = first bucket entry whose row is >= i
__global__ void k_split_rowptr(const int32_t* __restrict__ ord, int64_t t0, int64_t n,
                               const int32_t* __restrict__ row_of, int64_t nbr,
                               int32_t* __restrict__ rp) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > nbr) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (row_of[ord[t0 + mid]] < i) lo = mid + 1; else hi = mid;
  }
  rp[i] = static_cast<int32_t>(lo);
}

// Splits `s` into P stores by the per-entry owner: one stable radix sort by
// owner and a single readback of the per-owner totals (vs. a select + merge
// per destination).
void split_by_owner(Ctx& x, const Mat& s, const int32_t* d_owner, int P,
                    std::vector<std::unique_ptr<bt_mat>>& out) {
  cudaStream_t st = x.stream;
  const int64_t n = s.nblk;
  DBuf<int32_t> row_of(n, st), ident(n, st), okey(n, st), ord(n, st);
  DBuf<unsigned long long> hist(3 * P, st);
  BT_CUDA(cudaMemsetAsync(hist.p, 0, 8 * 3 * P, st));
  k_split_hist<<<nb(s.nbr, 128), 128, 0, st>>>(s.row_ptr.p, s.nbr, s.col.p, d_owner, s.rsz.p,
                                               s.csz.p, P, row_of.p, ident.p, hist.p);
  check_launch("split_hist");
  const int end_bit = std::max(1, 32 - __builtin_clz(static_cast<unsigned>(std::max(P - 1, 1))));
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, d_owner, okey.p, ident.p, ord.p, n, 0, end_bit,
                                  st);
  void* tmp = x.ensure_scratch(bytes);
  cub::DeviceRadixSort::SortPairs(tmp, bytes, d_owner, okey.p, ident.p, ord.p, n, 0, end_bit, st);
  DBuf<int64_t> vsz(n + 1, st), vscan(n + 1, st);
  k_split_vsz<<<nb(n + 1, 256), 256, 0, st>>>(ord.p, n, row_of.p, s.col.p, s.rsz.p, s.csz.p,
                                              vsz.p);
  check_launch("split_vsz");
  dscan(x, vsz.p, vscan.p, n + 1);
  count_launch(&x, 6);
  std::vector<unsigned long long> h(3 * P);
  BT_CUDA(cudaMemcpyAsync(h.data(), hist.p, 8 * 3 * P, cudaMemcpyDeviceToHost, st));
  BT_CUDA(cudaStreamSynchronize(st));
  int64_t t0 = 0;
  for (int d = 0; d < P; ++d) {
    const int64_t nd = static_cast<int64_t>(h[d]);
    Mat& b = out[d]->impl;
    if (nd) {
      b.row_ptr.alloc(b.nbr + 1, st);
      b.col.alloc(nd, st);
      b.off.alloc(nd, st);
      const int64_t nv = static_cast<int64_t>(h[P + d]);
      b.vals.alloc(std::max<int64_t>(nv, 64), st);
      k_split_fill<<<nb(nd * 32, 256), 256, 0, st>>>(ord.p, t0, nd, s.col.p, s.off.p, s.vals.p,
                                                     vscan.p, b.col.p, b.off.p, b.vals.p);
      check_launch("split_fill");
      k_split_rowptr<<<nb(b.nbr + 1, 256), 256, 0, st>>>(ord.p, t0, nd, row_of.p, b.nbr,
                                                         b.row_ptr.p);
      check_launch("split_rowptr");
      count_launch(&x, 2);
      b.nblk = nd;
      b.norms_ok = false;
      b.nvals = nv;
      b.nelems = static_cast<int64_t>(h[2 * P + d]);
    }
    t0 += nd;
  }
  BT_CUDA(cudaStreamSynchronize(st));  // the temporaries above are released on return
}

// ================================================================= group
struct Counters {
  int64_t v[4] = {0, 0, 0, 0};  // elements sent, received, meta sent, received
  Counters& operator+=(const Counters& o) {
    for (int t = 0; t < 4; ++t) v[t] += o.v[t];
    return *this;
  }
};

struct Grid {
  Ctx* ctx = nullptr;
  int P = 1;
  int first = 0, nlocal = 1;
  bool nccl = false;
  cudaStream_t comm = nullptr;
  cudaStream_t comm_vals = nullptr;  // the value all-gather's stream (second communicator)
  cudaEvent_t ev_comm = nullptr, ev_main = nullptr, ev_idx = nullptr;
  std::vector<Counters> totals;
  std::vector<std::map<std::string, Counters>> phases;
  std::vector<std::string> phase;
  // persistent buffers of the overlapped B gather (grow-only, reused per call)
  std::unique_ptr<bt_mat> gather_full;
  std::vector<DBuf<int32_t>> gather_rps;
  DBuf<int64_t> gather_sizes;
  DBuf<int32_t> gather_idx;    // P packed index segments (allgather path)
  cudaEvent_t phase_ev = nullptr;  // BT_PHASES: recorded at the numeric start
  cudaEvent_t ev_sizes = nullptr;  // size round of the gather read back
  int64_t spec_capb = 0, spec_capv = 0;  // speculative segment capacities
  bool spec_last = false;
  DBuf<int32_t> gather_rdist;  // row -> owning rank of the gathered slabs
  std::vector<int32_t> gather_rdist_h;
  bool is_local(int r) const { return r >= first && r < first + nlocal; }
  void set_phase(const std::string& p) {
    for (int r = first; r < first + nlocal; ++r) phase[r] = p;
  }
  void charge_send(int r, int64_t el, int64_t meta) {
    totals[r].v[0] += el;
    totals[r].v[2] += meta;
    auto& c = phases[r][phase[r]];
    c.v[0] += el;
    c.v[2] += meta;
  }
  void charge_recv(int r, int64_t el, int64_t meta) {
    totals[r].v[1] += el;
    totals[r].v[3] += meta;
    auto& c = phases[r][phase[r]];
    c.v[1] += el;
    c.v[3] += meta;
  }
};

// A message: a whole store from rank `from` to rank `to` (FIFO per pair, like
// SimComm's queues, comm.hpp:183-226).  Sends name the payload on the sending
// side, receives the destination store on the receiving side.
struct Send {
  int from, to;
  const Mat* payload;
};
struct Recv {
  int to, from;
  Mat* dst;
};

void copy_store(const Mat& s, Mat& d);

// One bulk-synchronous exchange step over the group.  Local transport: device
// copies (matched by (from, to) in posting order).  NCCL: a header round, then
// the arrays as grouped send/recv on the comm stream; with `async` the data
// round is left in flight (finish_exchange makes the main stream wait).
void exchange(Grid& g, const std::vector<Send>& sends, const std::vector<Recv>& recvs,
              bool charged = true, bool async = false) {
  Ctx& x = *g.ctx;
  for (const auto& s : sends)
    if (charged && s.from != s.to && g.is_local(s.from))
      g.charge_send(s.from, s.payload->nelems, 4 * s.payload->nblk);
  auto match = [&](const Recv& rv, std::vector<bool>& used) -> const Send* {
    for (size_t q = 0; q < sends.size(); ++q)
      if (!used[q] && sends[q].from == rv.from && sends[q].to == rv.to) {
        used[q] = true;
        return &sends[q];
      }
    return nullptr;
  };
  std::vector<bool> used(sends.size(), false);
  if (!g.nccl) {
    // snapshot first: a payload may be a receiver's destination in the same step
    std::vector<std::unique_ptr<bt_mat>> snap;
    std::vector<const Send*> src;
    for (const auto& rv : recvs) {
      const Send* s = match(rv, used);
      BT_REQUIRE(s, BT_ERR_DEADLOCK,
                 "deadlock: rank " + std::to_string(rv.to) + " waits on " + std::to_string(rv.from));
      auto t = std::make_unique<bt_mat>();
      t->impl.ctx = s->payload->ctx;
      t->impl.nbr = s->payload->nbr;
      t->impl.nbc = s->payload->nbc;
      copy_store(*s->payload, t->impl);
      snap.push_back(std::move(t));
    }
    for (size_t q = 0; q < recvs.size(); ++q) {
      copy_store(snap[q]->impl, *recvs[q].dst);
      if (charged && recvs[q].from != recvs[q].to)
        g.charge_recv(recvs[q].to, recvs[q].dst->nelems, 4 * recvs[q].dst->nblk);
    }
    for (size_t q = 0; q < sends.size(); ++q)
      BT_REQUIRE(used[q], BT_ERR_INTERNAL,
                 "run: unconsumed message from rank " + std::to_string(sends[q].from) +
                     " to rank " + std::to_string(sends[q].to));
    return;
  }
  // ---- NCCL (this process is rank g.first)
  ncclComm_t comm = static_cast<ncclComm_t>(x.nccl);
  const int me = g.first;
  std::vector<const Send*> peer_sends;
  std::vector<const Recv*> peer_recvs;
  for (const auto& rv : recvs) {
    if (rv.from == me) {  // self message
      const Send* s = match(rv, used);
      BT_REQUIRE(s, BT_ERR_DEADLOCK, "deadlock: self receive without send");
      copy_store(*s->payload, *rv.dst);
    } else {
      peer_recvs.push_back(&rv);
    }
  }
  for (size_t q = 0; q < sends.size(); ++q)
    if (!used[q]) peer_sends.push_back(&sends[q]);
  const size_t ns = peer_sends.size(), nr = peer_recvs.size();
  int64_t* hdr = reinterpret_cast<int64_t*>(x.pinned) + 64;  // pinned staging
  BT_REQUIRE(3 * (ns + nr) <= 400, BT_ERR_INTERNAL, "exchange: too many messages in one step");
  DBuf<int64_t> dh(3 * std::max<size_t>(ns + nr, 1), x.stream);
  for (size_t q = 0; q < ns; ++q) {
    hdr[3 * q] = peer_sends[q]->payload->nblk;
    hdr[3 * q + 1] = peer_sends[q]->payload->nvals;
    hdr[3 * q + 2] = peer_sends[q]->payload->nelems;
  }
  // the comm stream must see every prior main-stream write of the payloads
  BT_CUDA(cudaEventRecord(g.ev_main, x.stream));
  BT_CUDA(cudaStreamWaitEvent(g.comm, g.ev_main, 0));
  if (ns) BT_CUDA(cudaMemcpyAsync(dh.p, hdr, 8 * 3 * ns, cudaMemcpyHostToDevice, g.comm));
  ncclResult_t r = ncclGroupStart();
  for (size_t q = 0; q < ns; ++q) ncclSend(dh.p + 3 * q, 3, ncclInt64, peer_sends[q]->to, comm, g.comm);
  for (size_t q = 0; q < nr; ++q)
    ncclRecv(dh.p + 3 * (ns + q), 3, ncclInt64, peer_recvs[q]->from, comm, g.comm);
  r = ncclGroupEnd();
  BT_REQUIRE(r == ncclSuccess, BT_ERR_NCCL, std::string("NCCL header round: ") + ncclGetErrorString(r));
  if (nr) BT_CUDA(cudaMemcpyAsync(hdr + 3 * ns, dh.p + 3 * ns, 8 * 3 * nr, cudaMemcpyDeviceToHost, g.comm));
  BT_CUDA(cudaStreamSynchronize(g.comm));
  for (size_t q = 0; q < nr; ++q) {
    Mat& d = *peer_recvs[q]->dst;
    d.nblk = hdr[3 * (ns + q)];
    d.norms_ok = false;
    d.nvals = hdr[3 * (ns + q) + 1];
    d.nelems = hdr[3 * (ns + q) + 2];
    d.row_ptr.alloc(d.nbr + 1, g.comm);
    d.col.alloc(std::max<int64_t>(d.nblk, 1), g.comm);
    d.off.alloc(std::max<int64_t>(d.nblk, 1), g.comm);
    d.vals.alloc(std::max<int64_t>(d.nvals, 64), g.comm);
    if (charged) g.charge_recv(peer_recvs[q]->to, d.nelems, 4 * d.nblk);
  }
  r = ncclGroupStart();
  for (size_t q = 0; q < ns; ++q) {
    const Mat& s = *peer_sends[q]->payload;
    const int to = peer_sends[q]->to;
    ncclSend(s.row_ptr.p, s.nbr + 1, ncclInt32, to, comm, g.comm);
    if (s.nblk) {
      ncclSend(s.col.p, s.nblk, ncclInt32, to, comm, g.comm);
      ncclSend(s.off.p, s.nblk, ncclInt64, to, comm, g.comm);
      ncclSend(s.vals.p, s.nvals, ncclFloat64, to, comm, g.comm);
    }
  }
  for (size_t q = 0; q < nr; ++q) {
    Mat& d = *peer_recvs[q]->dst;
    const int from = peer_recvs[q]->from;
    ncclRecv(d.row_ptr.p, d.nbr + 1, ncclInt32, from, comm, g.comm);
    if (d.nblk) {
      ncclRecv(d.col.p, d.nblk, ncclInt32, from, comm, g.comm);
      ncclRecv(d.off.p, d.nblk, ncclInt64, from, comm, g.comm);
      ncclRecv(d.vals.p, d.nvals, ncclFloat64, from, comm, g.comm);
    }
  }
  r = ncclGroupEnd();
  BT_REQUIRE(r == ncclSuccess, BT_ERR_NCCL, std::string("NCCL data round: ") + ncclGetErrorString(r));
  // received buffers were allocated on the comm stream: hand them to main
  for (size_t q = 0; q < nr; ++q) {
    Mat& d = *peer_recvs[q]->dst;
    d.row_ptr.s = d.col.s = d.off.s = d.vals.s = x.stream;
  }
  BT_CUDA(cudaEventRecord(g.ev_comm, g.comm));
  if (!async) BT_CUDA(cudaStreamWaitEvent(x.stream, g.ev_comm, 0));
}

void finish_exchange(Grid& g) {
  if (g.nccl) BT_CUDA(cudaStreamWaitEvent(g.ctx->stream, g.ev_comm, 0));
}

void copy_store(const Mat& s, Mat& d) {
  cudaStream_t st = d.stream();
  d.row_ptr.alloc(d.nbr + 1, st);
  BT_CUDA(cudaMemcpyAsync(d.row_ptr.p, s.row_ptr.p, 4 * (d.nbr + 1), cudaMemcpyDeviceToDevice, st));
  d.col.alloc(std::max<int64_t>(s.nblk, 1), st);
  d.off.alloc(std::max<int64_t>(s.nblk, 1), st);
  d.vals.alloc(std::max<int64_t>(s.nvals, 64), st);
  if (s.nblk) {
    BT_CUDA(cudaMemcpyAsync(d.col.p, s.col.p, 4 * s.nblk, cudaMemcpyDeviceToDevice, st));
    BT_CUDA(cudaMemcpyAsync(d.off.p, s.off.p, 8 * s.nblk, cudaMemcpyDeviceToDevice, st));
    BT_CUDA(cudaMemcpyAsync(d.vals.p, s.vals.p, 8 * s.nvals, cudaMemcpyDeviceToDevice, st));
  }
  d.nblk = s.nblk;
  d.norms_ok = false;
  d.nvals = s.nvals;
  d.nelems = s.nelems;
}

// ============================================================ distributed matrix
struct DMat {
  Grid* g = nullptr;
  int64_t nbr = 0, nbc = 0;
  std::vector<int32_t> rsz, csz;
  int gr = 1, gc = 1;                  // ProcessGrid dims (grid.hpp:17-69)
  std::vector<int32_t> rdist, cdist;   // Axis distributions (matrix.hpp:26-130)
  std::vector<std::unique_ptr<bt_mat>> local;  // one store per local rank
  int owner(int64_t i, int64_t j) const { return rdist[i] * gc + cdist[j]; }
  Mat& store(int r) { return local[r - g->first]->impl; }
  const Mat& store(int r) const { return local[r - g->first]->impl; }
};

std::unique_ptr<bt_mat> new_store(Ctx* ctx, const std::vector<int32_t>& rsz,
                                  const std::vector<int32_t>& csz) {
  auto m = std::make_unique<bt_mat>();
  Mat& x = m->impl;
  x.ctx = ctx;
  x.nbr = static_cast<int64_t>(rsz.size());
  x.nbc = static_cast<int64_t>(csz.size());
  x.h_rsz = rsz;
  x.h_csz = csz;
  upload_sizes(x);
  x.init_empty();
  return m;
}

std::unique_ptr<DMat> new_dmat(Grid* g, std::vector<int32_t> rsz, std::vector<int32_t> csz, int gr,
                               int gc, std::vector<int32_t> rdist, std::vector<int32_t> cdist) {
  BT_REQUIRE(gr >= 1 && gc >= 1, BT_ERR_INVALID_ARGUMENT,
             "ProcessGrid: every grid extent must be >= 1");
  BT_REQUIRE(rdist.size() == rsz.size() && cdist.size() == csz.size(), BT_ERR_INVALID_ARGUMENT,
             "Axis: distribution length does not match block count");
  for (int v : rdist)
    BT_REQUIRE(v >= 0 && v < gr, BT_ERR_INVALID_ARGUMENT,
               "Axis: distribution coordinate " + std::to_string(v) + " out of grid range");
  for (int v : cdist)
    BT_REQUIRE(v >= 0 && v < gc, BT_ERR_INVALID_ARGUMENT,
               "Axis: distribution coordinate " + std::to_string(v) + " out of grid range");
  BT_REQUIRE(gr * gc <= g->P, BT_ERR_INVALID_ARGUMENT,
             "DistMatrix: grid larger than the process group");
  auto d = std::make_unique<DMat>();
  d->g = g;
  d->nbr = static_cast<int64_t>(rsz.size());
  d->nbc = static_cast<int64_t>(csz.size());
  d->rsz = std::move(rsz);
  d->csz = std::move(csz);
  d->gr = gr;
  d->gc = gc;
  d->rdist = std::move(rdist);
  d->cdist = std::move(cdist);
  for (int r = 0; r < g->nlocal; ++r) d->local.push_back(new_store(g->ctx, d->rsz, d->csz));
  return d;
}

bool same_dist(const std::vector<int32_t>& a, const std::vector<int32_t>& b) { return a == b; }

// ChunkPartition (partition.hpp:17-41)
std::vector<int32_t> chunk_dist(int64_t n, int parts) {
  std::vector<int32_t> d(n);
  const int64_t chunk = parts > 0 ? (n + parts - 1) / parts : 0;
  for (int64_t b = 0; b < n; ++b) d[b] = chunk == 0 ? 0 : static_cast<int32_t>(b / chunk);
  return d;
}

// redistribute / redistribute_add (matrix.hpp:567-622): every block of src moves
// (once) to its owner under dst's layout; transpose lands (i,j) at (j,i).
void redistribute(const DMat& src, DMat& dst, bool transpose, bool accumulate,
                  const std::string& phase) {
  Grid& g = *src.g;
  Ctx& x = *g.ctx;
  cudaStream_t st = x.stream;
  if (!transpose)
    BT_REQUIRE(src.rsz == dst.rsz && src.csz == dst.csz, BT_ERR_INVALID_ARGUMENT,
               "redistribute: target blockings do not match the source");
  else
    BT_REQUIRE(src.rsz == dst.csz && src.csz == dst.rsz, BT_ERR_INVALID_ARGUMENT,
               "redistribute: transposed target blockings do not match");
  g.set_phase(phase);
  Trace tr("redistribute");
  DBuf<int32_t> rdist(std::max<size_t>(dst.rdist.size(), 1), st),
      cdist(std::max<size_t>(dst.cdist.size(), 1), st);
  BT_CUDA(cudaMemcpyAsync(rdist.p, dst.rdist.data(), 4 * dst.rdist.size(), cudaMemcpyHostToDevice, st));
  BT_CUDA(cudaMemcpyAsync(cdist.p, dst.cdist.data(), 4 * dst.cdist.size(), cudaMemcpyHostToDevice, st));
  // per local rank and destination: the outgoing bucket as a store
  const int P = g.P;
  std::vector<std::vector<std::unique_ptr<bt_mat>>> out(g.nlocal);
  for (int lr = 0; lr < g.nlocal; ++lr) {
    const int r = g.first + lr;
    Mat& s = const_cast<Mat&>(src.store(r));
    DBuf<int32_t> owner(std::max<int64_t>(s.nblk, 1), st);
    if (s.nblk) {
      k_owner<<<nb(s.nbr, 128), 128, 0, st>>>(s.row_ptr.p, s.col.p, s.nbr, rdist.p, cdist.p,
                                              dst.gc, transpose ? 1 : 0, owner.p);
      count_launch(&x);
    }
    if (!transpose && s.nblk) {
      for (int d = 0; d < P; ++d) out[lr].push_back(new_store(g.ctx, dst.rsz, dst.csz));
      split_by_owner(x, s, owner.p, P, out[lr]);
      continue;
    }
    for (int d = 0; d < P; ++d) {
      auto bucket = new_store(g.ctx, dst.rsz, dst.csz);
      DBuf<int64_t> sel;
      const int64_t n = select_owned(s, owner.p, d, sel);
      if (n) merge_into(bucket->impl, {Contribution{&s, sel.p, n, transpose}}, false);
      out[lr].push_back(std::move(bucket));
    }
  }
  tr.mark("buckets");
  // exchange: step t, rank r sends to (r+t)%P and receives from (r-t)%P
  // (exchange_blocks, matrix.hpp:545-560); deliveries merged in that order
  std::vector<std::vector<std::unique_ptr<bt_mat>>> in(g.nlocal);
  std::vector<Send> sends;
  std::vector<Recv> recvs;
  for (int lr = 0; lr < g.nlocal; ++lr)
    for (int t = 0; t < P; ++t) in[lr].push_back(new_store(g.ctx, dst.rsz, dst.csz));
  for (int t = 0; t < P; ++t)
    for (int lr = 0; lr < g.nlocal; ++lr) {
      const int r = g.first + lr;
      const int to = (r + t) % P, from = (r - t + P) % P;
      sends.push_back(Send{r, to, &out[lr][to]->impl});
      recvs.push_back(Recv{r, from, &in[lr][t]->impl});
    }
  exchange(g, sends, recvs);
  tr.mark("exchange");
  for (int lr = 0; lr < g.nlocal; ++lr) {
    std::vector<Contribution> parts;
    for (int t = 0; t < P; ++t) {
      const Mat& m = in[lr][t]->impl;
      if (m.nblk) parts.push_back(Contribution{&m, nullptr, m.nblk, false});
    }
    Mat& d = dst.store(g.first + lr);
    if (!accumulate) d.init_empty();
    merge_into(d, parts, accumulate);
  }
  tr.mark("merge");
}

}  // namespace bt

// =========================================================== drivers (bt::)
namespace bt {

namespace {

void add_stats(bt_stats& acc, const bt_stats& s) {
  acc.candidates += s.candidates;
  acc.products += s.products;
  acc.flops += s.flops;
  acc.c_blocks_in += s.c_blocks_in;
  acc.c_blocks_out += s.c_blocks_out;
  acc.kernels += s.kernels;
  acc.ms_numeric += s.ms_numeric;
  acc.ms_total += s.ms_total;
}

void rank_multiply(Ctx* ctx, const Mat& a, const Mat& b, Mat& c, double eps, bt_stats& acc,
                   cudaEvent_t wait_numeric = nullptr, cudaEvent_t numeric_start = nullptr,
                   const std::function<void()>* after_sizes = nullptr, bool poll_sizes = false) {
  bt_stats s{};
  local_multiply(*ctx, a, b, c, eps, &s, wait_numeric, numeric_start, after_sizes, true,
                 poll_sizes);
  add_stats(acc, s);
}

void ledger_stats(const Grid& g, const Counters& before_sent, bt_stats& S) {
  Counters now{};
  for (int r = g.first; r < g.first + g.nlocal; ++r) now += g.totals[r];
  S.elements_sent = now.v[0] - before_sent.v[0];
  S.elements_received = now.v[1] - before_sent.v[1];
  S.meta_sent = now.v[2] - before_sent.v[2];
  S.meta_received = now.v[3] - before_sent.v[3];
}

Counters ledger_snapshot(const Grid& g) {
  Counters c{};
  for (int r = g.first; r < g.first + g.nlocal; ++r) c += g.totals[r];
  return c;
}

void check_conformal(const DMat& a, const DMat& b, const DMat& c, const char* who) {
  BT_REQUIRE(a.csz == b.rsz, BT_ERR_INVALID_ARGUMENT,
             std::string(who) + ": inner blockings of A and B differ");
  BT_REQUIRE(c.rsz == a.rsz && c.csz == b.csz, BT_ERR_INVALID_ARGUMENT,
             std::string(who) + ": C blockings do not conform");
}

// A layout-only view: a DMat that borrows `src`'s stores when src already has
// the requested layout (redistribution would move nothing and charge nothing),
// else a redistributed copy.
struct Relaid {
  const DMat* view = nullptr;
  std::unique_ptr<DMat> owned;
};

Relaid relayout(const DMat& src, int gr, int gc, const std::vector<int32_t>& rdist,
                const std::vector<int32_t>& cdist, const std::string& phase) {
  Relaid r;
  if (src.gr == gr && src.gc == gc && src.rdist == rdist && src.cdist == cdist) {
    r.view = &src;
    return r;
  }
  r.owned = new_dmat(src.g, src.rsz, src.csz, gr, gc, rdist, cdist);
  redistribute(src, *r.owned, false, false, phase);
  r.view = r.owned.get();
  return r;
}

// Concatenate stores holding disjoint, increasing row ranges (rank order of a
// ChunkPartition of the rows) into one store: index fix-ups + device copies.
__global__ void k_shift_rows(int32_t* __restrict__ rp, int64_t r0, int64_t r1, int32_t add) {
  const int64_t i = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > r1) return;
  rp[i] += add;
}
__global__ void k_shift_off(int64_t* __restrict__ off, int64_t n, int64_t add) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n) off[e] += add;
}

void concat_rows(const std::vector<const Mat*>& parts, const std::vector<int32_t>& rdist, Mat& out) {
  Ctx& x = *out.ctx;
  cudaStream_t st = x.stream;
  int64_t nblk = 0, nvals = 0, nel = 0;
  for (auto* p : parts) {
    nblk += p->nblk;
    nvals += p->nvals;
    nel += p->nelems;
  }
  DBuf<int32_t> rp(out.nbr + 1, st), col(std::max<int64_t>(nblk, 1), st);
  DBuf<int64_t> off(std::max<int64_t>(nblk, 1), st);
  DBuf<double> vals(std::max<int64_t>(nvals, 64), st);
  int64_t bb = 0, vb = 0;
  for (size_t p = 0; p < parts.size(); ++p) {
    const Mat& m = *parts[p];
    // rows owned by part p: [r0, r1)
    int64_t r0 = -1, r1 = -1;
    for (int64_t i = 0; i < out.nbr; ++i)
      if (rdist[i] == static_cast<int32_t>(p)) {
        if (r0 < 0) r0 = i;
        r1 = i + 1;
      }
    if (r0 < 0) continue;
    // row_ptr[r0..r1] of the part (its rows outside [r0, r1) are empty)
    BT_CUDA(cudaMemcpyAsync(rp.p + r0, m.row_ptr.p + r0, 4 * (r1 - r0 + 1), cudaMemcpyDeviceToDevice, st));
    if (bb) k_shift_rows<<<nb(r1 - r0 + 1, 256), 256, 0, st>>>(rp.p, r0, r1, static_cast<int32_t>(bb));
    if (m.nblk) {
      BT_CUDA(cudaMemcpyAsync(col.p + bb, m.col.p, 4 * m.nblk, cudaMemcpyDeviceToDevice, st));
      BT_CUDA(cudaMemcpyAsync(off.p + bb, m.off.p, 8 * m.nblk, cudaMemcpyDeviceToDevice, st));
      if (vb) k_shift_off<<<nb(m.nblk, 256), 256, 0, st>>>(off.p + bb, m.nblk, vb);
      BT_CUDA(cudaMemcpyAsync(vals.p + vb, m.vals.p, 8 * m.nvals, cudaMemcpyDeviceToDevice, st));
    }
    count_launch(&x, 2);
    bb += m.nblk;
    vb += m.nvals;
  }
  // rows before the first owned row
  BT_CUDA(cudaMemsetAsync(rp.p, 0, 4, st));
  out.row_ptr = std::move(rp);
  out.col = std::move(col);
  out.off = std::move(off);
  out.vals = std::move(vals);
  out.nblk = nblk;
  out.norms_ok = false;
  out.nvals = nvals;
  out.nelems = nel;
}

// All-gather of row slabs over NCCL into one store, values overlapped: the
// index (row_ptr/col/off) is exchanged first and assembled synchronously; the
// values of every slab are then received straight into their place in the
// full slab on the comm stream.  Returns an event recorded when the values have
// landed; the local multiply's symbolic passes run meanwhile.
cudaEvent_t gather_rows_nccl(Grid& g, const Mat& mine, const std::vector<int32_t>& rdist, int nprocs,
                             Mat& full) {
  Ctx& x = *g.ctx;
  Trace tr("gather");
  ncclComm_t comm = static_cast<ncclComm_t>(x.nccl);
  const int me = g.first;
  cudaStream_t cs = g.comm;
  // sizes of every slab (3 words each)
  auto grow = [&](auto& buf, size_t n) {
    if (buf.n < n) buf.alloc(n + n / 8, x.stream);
  };
  grow(g.gather_sizes, static_cast<size_t>(3 * nprocs));
  DBuf<int64_t>& dsz = g.gather_sizes;
  int64_t* h = reinterpret_cast<int64_t*>(x.pinned) + 64;
  h[0] = mine.nblk;
  h[1] = mine.nvals;
  h[2] = mine.nelems;
  BT_CUDA(cudaEventRecord(g.ev_main, x.stream));
  BT_CUDA(cudaStreamWaitEvent(cs, g.ev_main, 0));
  BT_CUDA(cudaMemcpyAsync(dsz.p + 3 * me, h, 24, cudaMemcpyHostToDevice, cs));
  ncclResult_t r = ncclAllGather(dsz.p + 3 * me, dsz.p, 3, ncclInt64, comm, cs);
  BT_REQUIRE(r == ncclSuccess, BT_ERR_NCCL, std::string("NCCL size gather: ") + ncclGetErrorString(r));
  BT_CUDA(cudaMemcpyAsync(h + 8, dsz.p, 24 * nprocs, cudaMemcpyDeviceToHost, cs));
  BT_CUDA(cudaStreamSynchronize(cs));
  tr.mark("sizes");
  std::vector<int64_t> bb(nprocs + 1, 0), vb(nprocs + 1, 0);
  int64_t nel = 0;
  for (int p = 0; p < nprocs; ++p) {
    bb[p + 1] = bb[p] + h[8 + 3 * p];
    vb[p + 1] = vb[p] + h[8 + 3 * p + 1];
    nel += h[8 + 3 * p + 2];
  }
  grow(full.row_ptr, static_cast<size_t>(full.nbr + 1));
  grow(full.col, static_cast<size_t>(std::max<int64_t>(bb[nprocs], 1)));
  grow(full.off, static_cast<size_t>(std::max<int64_t>(bb[nprocs], 1)));
  grow(full.vals, static_cast<size_t>(std::max<int64_t>(vb[nprocs], 64)));
  full.nblk = bb[nprocs];
  full.norms_ok = false;
  full.nvals = vb[nprocs];
  full.nelems = nel;
  if (static_cast<int>(g.gather_rps.size()) < nprocs) g.gather_rps.resize(nprocs);
  std::vector<DBuf<int32_t>>& rps = g.gather_rps;
  for (int p = 0; p < nprocs; ++p) grow(rps[p], static_cast<size_t>(full.nbr + 1));
  tr.mark("alloc");
  BT_CUDA(cudaEventRecord(g.ev_main, x.stream));
  BT_CUDA(cudaStreamWaitEvent(cs, g.ev_main, 0));
  // index round
  BT_CUDA(cudaMemcpyAsync(rps[me].p, mine.row_ptr.p, 4 * (full.nbr + 1), cudaMemcpyDeviceToDevice, cs));
  if (mine.nblk) {
    BT_CUDA(cudaMemcpyAsync(full.col.p + bb[me], mine.col.p, 4 * mine.nblk, cudaMemcpyDeviceToDevice, cs));
    BT_CUDA(cudaMemcpyAsync(full.off.p + bb[me], mine.off.p, 8 * mine.nblk, cudaMemcpyDeviceToDevice, cs));
  }
  ncclGroupStart();
  for (int p = 0; p < nprocs; ++p) {
    if (p == me) continue;
    ncclSend(mine.row_ptr.p, full.nbr + 1, ncclInt32, p, comm, cs);
    if (mine.nblk) {
      ncclSend(mine.col.p, mine.nblk, ncclInt32, p, comm, cs);
      ncclSend(mine.off.p, mine.nblk, ncclInt64, p, comm, cs);
    }
    const int64_t n = bb[p + 1] - bb[p];
    ncclRecv(rps[p].p, full.nbr + 1, ncclInt32, p, comm, cs);
    if (n) {
      ncclRecv(full.col.p + bb[p], n, ncclInt32, p, comm, cs);
      ncclRecv(full.off.p + bb[p], n, ncclInt64, p, comm, cs);
    }
  }
  r = ncclGroupEnd();
  BT_REQUIRE(r == ncclSuccess, BT_ERR_NCCL, std::string("NCCL index round: ") + ncclGetErrorString(r));
  BT_CUDA(cudaEventRecord(g.ev_idx, cs));
  // values round (left in flight)
  if (mine.nvals)
    BT_CUDA(cudaMemcpyAsync(full.vals.p + vb[me], mine.vals.p, 8 * mine.nvals,
                            cudaMemcpyDeviceToDevice, cs));
  ncclGroupStart();
  for (int p = 0; p < nprocs; ++p) {
    if (p == me) continue;
    if (mine.nvals) ncclSend(mine.vals.p, mine.nvals, ncclFloat64, p, comm, cs);
    const int64_t nv = vb[p + 1] - vb[p];
    if (nv) ncclRecv(full.vals.p + vb[p], nv, ncclFloat64, p, comm, cs);
  }
  r = ncclGroupEnd();
  BT_REQUIRE(r == ncclSuccess, BT_ERR_NCCL, std::string("NCCL value round: ") + ncclGetErrorString(r));
  BT_CUDA(cudaEventRecord(g.ev_comm, cs));
  tr.mark("enqueue rounds");
  // assemble the index on the main stream once the index round is in; the
  // values keep streaming on the comm stream
  BT_CUDA(cudaStreamWaitEvent(x.stream, g.ev_idx, 0));
  for (int p = 0; p < nprocs; ++p) {
    int64_t r0 = -1, r1 = -1;
    for (int64_t i = 0; i < full.nbr; ++i)
      if (rdist[i] == p) {
        if (r0 < 0) r0 = i;
        r1 = i + 1;
      }
    if (r0 < 0) continue;
    BT_CUDA(cudaMemcpyAsync(full.row_ptr.p + r0, rps[p].p + r0, 4 * (r1 - r0 + 1),
                            cudaMemcpyDeviceToDevice, x.stream));
    if (bb[p]) k_shift_rows<<<nb(r1 - r0 + 1, 256), 256, 0, x.stream>>>(full.row_ptr.p, r0, r1,
                                                                         static_cast<int32_t>(bb[p]));
    const int64_t n = bb[p + 1] - bb[p];
    if (vb[p] && n) k_shift_off<<<nb(n, 256), 256, 0, x.stream>>>(full.off.p + bb[p], n, vb[p]);
    count_launch(&x, 2);
  }
  BT_CUDA(cudaMemsetAsync(full.row_ptr.p, 0, 4, x.stream));
  tr.mark("assemble");
  g.charge_send(me, (nprocs - 1) * mine.nelems, (nprocs - 1) * 4 * mine.nblk);
  g.charge_recv(me, nel - mine.nelems, 4 * (bb[nprocs] - mine.nblk));
  return g.ev_comm;
}

// Assembles the gathered slabs' index into one store (allgather layout): rank
// q's segment holds row_ptr (dense over all rows) | col | off, so the global
// row pointer is the sum of the ranks' row pointers, and row i's entries are
// those of its owner p = rdist[i], value offsets shifted by p * maxv.  One warp
// per block row.
__global__ void k_assemble_gathered(const int32_t* __restrict__ gidx, int64_t seg, int64_t colb,
                                    int64_t offb, int P, const int32_t* __restrict__ rdist,
                                    int64_t nbr, int64_t maxv, int64_t capb,
                                    int32_t* __restrict__ rp, int32_t* __restrict__ col,
                                    int64_t* __restrict__ off) {
  const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i > nbr) return;
  // a slab larger than the segment capacity (a missed speculation, redone by
  // the host) is treated as empty so every read stays inside the buffers
  int32_t dst = 0;
  for (int q = 0; q < P; ++q)
    if (gidx[q * seg + nbr] <= capb) dst += gidx[q * seg + i];
  if (lane == 0) rp[i] = dst;
  if (i == nbr) return;
  const int p = rdist[i];
  const int32_t* s = gidx + p * seg;
  if (s[nbr] > capb) return;
  const int32_t e0 = s[i], n = s[i + 1] - e0;
  const int32_t* sc = s + colb;
  const int64_t* so = reinterpret_cast<const int64_t*>(s + offb);
  const int64_t shift = static_cast<int64_t>(p) * maxv;
  for (int t = lane; t < n; t += 32) {
    col[dst + t] = sc[e0 + t];
    off[dst + t] = so[e0 + t] + shift;
  }
}

// All-gather of row slabs into one store with in-place ncclAllGather calls
// (every rank of the communicator takes part): a 3-word size round, the packed
// index (row_ptr | col | off, one segment per rank) and the T8 values (one
// segment per rank), all on the comm stream; the index is assembled by one
// kernel on the main stream as soon as it lands while the values keep
// streaming.  Returns the event recorded when the values have landed.
//
// Segment capacities.  exact (spec = false): the host waits for the size
// round and sizes the segments to the largest slab.  spec = true: the
// segments take the capacities remembered from earlier calls and there is no
// size round (the sizes ride in the index segments' headers), so the index
// and value rounds are enqueued at once without any host wait;
// gather_check() (run by the multiply right after its own pass-1 sync, before
// any value is read) confirms every slab fit, or throws SpecMiss and the caller
// redoes the gather exactly.  All ranks see the same sizes, so they all take
// the same branch.
struct SpecMiss {};

// Sizes of the last gather: exact store metadata and ledger charges; in the
// speculative case throws SpecMiss when a slab did not fit its segment.
void gather_check(Grid& g, const Mat& mine, int nprocs, Mat& full, bool spec) {
  Ctx& x = *g.ctx;
  BT_CUDA(cudaEventSynchronize(g.ev_sizes));
  const int64_t* h = reinterpret_cast<const int64_t*>(x.pinned) + 384;
  int64_t nblk = 0, nel = 0, maxb = 0, maxv = 0;
  for (int p = 0; p < nprocs; ++p) {
    nblk += h[8 + 3 * p];
    maxb = std::max(maxb, h[8 + 3 * p]);
    maxv = std::max(maxv, h[8 + 3 * p + 1]);
    nel += h[8 + 3 * p + 2];
  }
  if (spec && (maxb > g.spec_capb || maxv > g.spec_capv)) throw SpecMiss{};
  // next call's capacities: 1/8 headroom over this call, decaying slowly
  // when the slabs shrink (identical on every rank: same sizes)
  g.spec_capb = std::max(maxb + maxb / 8, g.spec_capb - g.spec_capb / 8);
  g.spec_capv = std::max((maxv + maxv / 8 + 63) & ~int64_t(63),
                         (g.spec_capv - g.spec_capv / 8 + 63) & ~int64_t(63));
  if (env_int("BT_GATHER_SPEC_TEST", 0)) {  // tests: force the next speculation to miss
    g.spec_capb = maxb / 2;
    g.spec_capv = (maxv / 2) & ~int64_t(63);
  }
  full.nblk = nblk;
  full.norms_ok = false;
  full.nelems = nel;
  const int me = g.first;
  g.charge_send(me, (nprocs - 1) * mine.nelems, (nprocs - 1) * 4 * mine.nblk);
  g.charge_recv(me, nel - mine.nelems, 4 * (nblk - mine.nblk));
}

cudaEvent_t gather_rows_allgather(Grid& g, const Mat& mine, const std::vector<int32_t>& rdist,
                                  int nprocs, Mat& full, bool spec) {
  Ctx& x = *g.ctx;
  Trace tr("gather");
  ncclComm_t comm = static_cast<ncclComm_t>(x.nccl);
  const int me = g.first;
  cudaStream_t cs = g.comm;
  // BT_PHASES=1: device timeline of the gather (rank 0 prints the previous call's)
  static cudaEvent_t pev[6] = {};
  static bool pev_recorded = false;
  const bool phases = env_int("BT_PHASES", 0) != 0;
  if (phases && !pev[0])
    for (auto& e : pev) BT_CUDA(cudaEventCreate(&e));
  if (phases && me == 0 && pev_recorded) {
    BT_CUDA(cudaEventSynchronize(pev[5]));
    float t[5];
    for (int q = 0; q < 5; ++q) BT_CUDA(cudaEventElapsedTime(&t[q], pev[0], pev[q + 1]));
    fprintf(stderr, "[bt-gather] %s sizes %.1f | index %.1f | assembled %.1f | values %.1f | "
                    "numeric start %.1f us\n", g.spec_last ? "spec" : "exact", 1e3 * t[0],
            1e3 * t[1], 1e3 * t[2], 1e3 * t[3], 1e3 * t[4]);
  }
  g.spec_last = spec;
  auto grow = [&](auto& buf, size_t n) {
    if (buf.n < n) buf.alloc(n + n / 8, x.stream);
  };
  // pinned words [384, 384 + 8 + 3P): clear of the multiply's size readback
  int64_t* h = reinterpret_cast<int64_t*>(x.pinned) + 384;
  h[0] = mine.nblk;
  h[1] = mine.nvals;
  h[2] = mine.nelems;
  // the row -> rank map (host -> device only when it changes)
  if (g.gather_rdist_h != rdist) {
    g.gather_rdist_h = rdist;
    grow(g.gather_rdist, rdist.size());
    BT_CUDA(cudaMemcpyAsync(g.gather_rdist.p, g.gather_rdist_h.data(), 4 * rdist.size(),
                            cudaMemcpyHostToDevice, x.stream));
  }
  const int64_t nbr = full.nbr;
  BT_CUDA(cudaEventRecord(g.ev_main, x.stream));
  if (phases) BT_CUDA(cudaEventRecord(pev[0], x.stream));
  BT_CUDA(cudaStreamWaitEvent(cs, g.ev_main, 0));
  ncclResult_t r;
  int64_t maxb, maxv;
  if (spec) {
    // no size round: the sizes travel in the index segments' headers
    maxb = g.spec_capb;
    maxv = g.spec_capv;
    if (phases) BT_CUDA(cudaEventRecord(pev[1], cs));
  } else {
    grow(g.gather_sizes, static_cast<size_t>(3 * nprocs));
    DBuf<int64_t>& dsz = g.gather_sizes;
    BT_CUDA(cudaMemcpyAsync(dsz.p + 3 * me, h, 24, cudaMemcpyHostToDevice, cs));
    r = ncclAllGather(dsz.p + 3 * me, dsz.p, 3, ncclInt64, comm, cs);
    BT_REQUIRE(r == ncclSuccess, BT_ERR_NCCL,
               std::string("NCCL size gather: ") + ncclGetErrorString(r));
    BT_CUDA(cudaMemcpyAsync(h + 8, dsz.p, 24 * nprocs, cudaMemcpyDeviceToHost, cs));
    BT_CUDA(cudaEventRecord(g.ev_sizes, cs));
    if (phases) BT_CUDA(cudaEventRecord(pev[1], cs));
    BT_CUDA(cudaEventSynchronize(g.ev_sizes));
    maxb = maxv = 0;
    for (int p = 0; p < nprocs; ++p) {
      maxb = std::max(maxb, h[8 + 3 * p]);
      maxv = std::max(maxv, h[8 + 3 * p + 1]);
    }
  }
  tr.mark("sizes");
  // segment (int32 words): header (3 x int64) | row_ptr | col | off
  const int64_t rpb = 6;
  const int64_t colb = rpb + pad2(nbr + 1);
  const int64_t offb = colb + pad2(maxb);
  const int64_t seg = offb + 2 * maxb;
  grow(g.gather_idx, static_cast<size_t>(seg * nprocs));
  grow(full.row_ptr, static_cast<size_t>(nbr + 1));
  grow(full.col, static_cast<size_t>(std::max<int64_t>(maxb * nprocs, 1)));
  grow(full.off, static_cast<size_t>(std::max<int64_t>(maxb * nprocs, 1)));
  grow(full.vals, static_cast<size_t>(std::max<int64_t>(maxv * nprocs, 64)));
  full.nblk = maxb * nprocs;  // upper bound until the sizes are known (gather_check)
  full.norms_ok = false;
  full.nvals = maxv * nprocs;
  full.nelems = 0;
  BT_CUDA(cudaEventRecord(g.ev_main, x.stream));
  BT_CUDA(cudaStreamWaitEvent(cs, g.ev_main, 0));
  // my slab into my segments (clamped: a slab over capacity is a miss anyway)
  const int64_t sb = std::min(mine.nblk, maxb), sv = std::min(mine.nvals, maxv);
  int32_t* mseg = g.gather_idx.p + seg * me;
  BT_CUDA(cudaMemcpyAsync(mseg, h, 24, cudaMemcpyHostToDevice, cs));
  BT_CUDA(cudaMemcpyAsync(mseg + rpb, mine.row_ptr.p, 4 * (nbr + 1), cudaMemcpyDeviceToDevice, cs));
  if (sb) {
    BT_CUDA(cudaMemcpyAsync(mseg + colb, mine.col.p, 4 * sb, cudaMemcpyDeviceToDevice, cs));
    BT_CUDA(cudaMemcpyAsync(mseg + offb, mine.off.p, 8 * sb, cudaMemcpyDeviceToDevice, cs));
  }
  r = ncclAllGather(mseg, g.gather_idx.p, seg, ncclInt32, comm, cs);
  BT_REQUIRE(r == ncclSuccess, BT_ERR_NCCL, std::string("NCCL index gather: ") + ncclGetErrorString(r));
  BT_CUDA(cudaEventRecord(g.ev_idx, cs));
  if (phases) BT_CUDA(cudaEventRecord(pev[2], cs));
  // values: on a second communicator and stream, concurrent with the index
  // gather (on one communicator NCCL serialises them: the values started only
  // once the index had landed).  The communicator is split off the context's
  // on the first gather (a collective call: every rank is here).
  cudaStream_t vs = cs;
  ncclComm_t vcomm = comm;
  if (env_int("BT_GATHER_2COMM", 1) != 0 && g.comm_vals) {
    if (!x.nccl_vals) {
      ncclComm_t c2 = nullptr;
      ncclResult_t rs = ncclCommSplit(comm, 0, me, &c2, nullptr);
      BT_REQUIRE(rs == ncclSuccess, BT_ERR_NCCL, std::string("ncclCommSplit: ") + ncclGetErrorString(rs));
      x.nccl_vals = c2;
    }
    vcomm = static_cast<ncclComm_t>(x.nccl_vals);
    vs = g.comm_vals;
    BT_CUDA(cudaStreamWaitEvent(vs, g.ev_main, 0));
  }
  if (maxv) {
    if (sv)
      BT_CUDA(cudaMemcpyAsync(full.vals.p + maxv * me, mine.vals.p, 8 * sv,
                              cudaMemcpyDeviceToDevice, vs));
    r = ncclAllGather(full.vals.p + maxv * me, full.vals.p, maxv, ncclFloat64, vcomm, vs);
    BT_REQUIRE(r == ncclSuccess, BT_ERR_NCCL,
               std::string("NCCL value gather: ") + ncclGetErrorString(r));
  }
  BT_CUDA(cudaEventRecord(g.ev_comm, vs));
  if (phases) BT_CUDA(cudaEventRecord(pev[4], vs));
  tr.mark("enqueue rounds");
  BT_CUDA(cudaStreamWaitEvent(x.stream, g.ev_idx, 0));
  if (spec) {  // the headers of the landed index segments, for gather_check
    BT_CUDA(cudaMemcpy2DAsync(h + 8, 24, g.gather_idx.p, 4 * seg, 24, nprocs,
                              cudaMemcpyDeviceToHost, x.stream));
    BT_CUDA(cudaEventRecord(g.ev_sizes, x.stream));
  }
  k_assemble_gathered<<<nb((nbr + 1) * 32, 256), 256, 0, x.stream>>>(
      g.gather_idx.p + rpb, seg, colb - rpb, offb - rpb, nprocs, g.gather_rdist.p, nbr, maxv, maxb,
      full.row_ptr.p, full.col.p, full.off.p);
  check_launch("assemble_gathered");
  count_launch(&x);
  if (phases) {
    BT_CUDA(cudaEventRecord(pev[3], x.stream));
    g.phase_ev = pev[5];  // recorded by the multiply when its numeric phase starts
    pev_recorded = true;
  }
  tr.mark("assemble");
  if (!spec) gather_check(g, mine, nprocs, full, false);
  return g.ev_comm;
}

}  // namespace

// multiply_cannon (multiply_cannon.hpp:62-118)
void cannon(const DMat& a, const DMat& b, DMat& c, double eps, bt_stats& S) {
  Grid& g = *a.g;
  BT_REQUIRE(a.gr == a.gc, BT_ERR_GRID,
             "multiply_cannon: grid must be square, got " + std::to_string(a.gr) + "x" +
                 std::to_string(a.gc));
  BT_REQUIRE(b.gr == a.gr && b.gc == a.gc && c.gr == a.gr && c.gc == a.gc, BT_ERR_GRID,
             "multiply_cannon: operands must share one square grid");
  BT_REQUIRE(a.csz == b.rsz, BT_ERR_INVALID_ARGUMENT,
             "multiply_cannon: inner blockings of A and B differ");
  BT_REQUIRE(c.rsz == a.rsz && c.csz == b.csz, BT_ERR_INVALID_ARGUMENT,
             "multiply_cannon: C blockings do not conform");
  BT_REQUIRE(a.cdist == b.rdist, BT_ERR_INVALID_ARGUMENT,
             "multiply_cannon: inner distributions of A and B differ; redistribute first");
  BT_REQUIRE(c.rdist == a.rdist && c.cdist == b.cdist, BT_ERR_INVALID_ARGUMENT,
             "multiply_cannon: C distribution must match A rows x B cols");
  const int q = a.gr, nprocs = q * q;
  BT_REQUIRE(g.P >= nprocs, BT_ERR_INVALID_ARGUMENT,
             "multiply_cannon: communicator smaller than the grid");
  const Counters before = ledger_snapshot(g);
  auto rank_of = [q](int r, int cc) { return ((r % q + q) % q) * q + ((cc % q + q) % q); };
  // skewed starting tiles (uncharged, like the reference's direct copies :84-94):
  // rank (r,c) starts with A of grid column (c+r)%q and B of grid row (r+c)%q
  std::vector<std::unique_ptr<bt_mat>> ta, tb, na_, nb_;
  for (int lr = 0; lr < g.nlocal; ++lr) {
    ta.push_back(new_store(g.ctx, a.rsz, a.csz));
    tb.push_back(new_store(g.ctx, b.rsz, b.csz));
    na_.push_back(new_store(g.ctx, a.rsz, a.csz));
    nb_.push_back(new_store(g.ctx, b.rsz, b.csz));
  }
  {
    std::vector<Send> sends;
    std::vector<Recv> recvs;
    for (int lr = 0; lr < g.nlocal; ++lr) {
      const int r = g.first + lr;
      if (r >= nprocs) continue;
      const int rr = r / q, cc = r % q;
      sends.push_back(Send{r, rank_of(rr, cc - rr), &a.store(r)});
      sends.push_back(Send{r, rank_of(rr - cc, cc), &b.store(r)});
      recvs.push_back(Recv{r, rank_of(rr, cc + rr), &ta[lr]->impl});
      recvs.push_back(Recv{r, rank_of(rr + cc, cc), &tb[lr]->impl});
    }
    exchange(g, sends, recvs, /*charged=*/false);
  }
  g.set_phase("cannon");
  for (int step = 0; step < q; ++step) {
    if (q > 1) {  // sends posted before the local compute (:106-116)
      std::vector<Send> sends;
      std::vector<Recv> recvs;
      for (int lr = 0; lr < g.nlocal; ++lr) {
        const int r = g.first + lr;
        if (r >= nprocs) continue;
        const int rr = r / q, cc = r % q;
        sends.push_back(Send{r, rank_of(rr, cc - 1), &ta[lr]->impl});  // left
        sends.push_back(Send{r, rank_of(rr - 1, cc), &tb[lr]->impl});  // up
        recvs.push_back(Recv{r, rank_of(rr, cc + 1), &na_[lr]->impl});  // from right
        recvs.push_back(Recv{r, rank_of(rr + 1, cc), &nb_[lr]->impl});  // from down
      }
      exchange(g, sends, recvs, true, /*async=*/true);
    }
    for (int lr = 0; lr < g.nlocal; ++lr) {
      const int r = g.first + lr;
      if (r >= nprocs) continue;
      rank_multiply(g.ctx, ta[lr]->impl, tb[lr]->impl, c.store(r), eps, S);
    }
    if (q > 1) {
      finish_exchange(g);
      std::swap(ta, na_);
      std::swap(tb, nb_);
    }
  }
  BT_CUDA(cudaStreamSynchronize(g.ctx->stream));
  ledger_stats(g, before, S);
}

// multiply_reduce_case1 (multiply_rect.hpp:123-192): K-slab split on a linear
// grid, local partials, reduction of the partials onto C's owners.
void case1(const DMat& a, const DMat& b, DMat& c, int nprocs, double eps, bt_stats& S) {
  Grid& g = *a.g;
  check_conformal(a, b, c, "multiply_reduce_case1");
  BT_REQUIRE(nprocs >= 1, BT_ERR_INVALID_ARGUMENT, "multiply_reduce_case1: nprocs must be positive");
  BT_REQUIRE(g.P >= nprocs && g.P >= a.gr * a.gc && g.P >= b.gr * b.gc && g.P >= c.gr * c.gc,
             BT_ERR_INVALID_ARGUMENT, "multiply_reduce_case1: communicator too small");
  const Counters before = ledger_snapshot(g);
  const auto ks = chunk_dist(static_cast<int64_t>(a.csz.size()), nprocs);
  // A by K-slab columns on a 1 x nprocs grid (the reference stores A^T by K-slab
  // rows; same blocks to the same ranks, so the same traffic), B by K-slab rows.
  auto al = relayout(a, 1, nprocs, std::vector<int32_t>(a.rsz.size(), 0), ks, "redistribute");
  auto bl = relayout(b, nprocs, 1, ks, std::vector<int32_t>(b.csz.size(), 0), "redistribute");
  g.set_phase("multiply");
  if (nprocs == 1 && c.gr * c.gc == 1 && g.is_local(0)) {
    // one rank owns everything: its product is C itself (no partial, no reduction)
    rank_multiply(g.ctx, al.view->store(0), bl.view->store(0), c.store(0), eps, S);
    ledger_stats(g, before, S);
    return;
  }
  // partial results live on a layout where every rank may hold any block: use
  // C's own layout's blockings, stored per rank
  auto part = new_dmat(&g, c.rsz, c.csz, c.gr, c.gc, c.rdist, c.cdist);
  for (int lr = 0; lr < g.nlocal; ++lr) {
    const int r = g.first + lr;
    if (r >= nprocs) continue;
    rank_multiply(g.ctx, al.view->store(r), bl.view->store(r), part->store(r), eps, S);
  }
  // reduce: every partial block goes once to its C owner and is accumulated
  // there (the reference's rotating ring + collect, :159-190, in one hop over
  // NVSwitch)
  redistribute(*part, c, false, true, "reduce");
  ledger_stats(g, before, S);
}

// multiply_virtual_case2 (multiply_rect.hpp:199-238): A and C row slabs stay
// resident, B K-slabs circulate.  gather = 0: the reference's P-step ring;
// gather = 1: every rank gathers all B slabs over NVLink in one step and runs
// one local multiply (same per-rank volume S_B*(P-1)/P, no P passes over C).
void case2(const DMat& a, const DMat& b, DMat& c, int nprocs, int gather, double eps,
           bt_stats& S) {
  Grid& g = *a.g;
  check_conformal(a, b, c, "multiply_virtual_case2");
  BT_REQUIRE(nprocs >= 1, BT_ERR_INVALID_ARGUMENT, "multiply_virtual_case2: nprocs must be positive");
  BT_REQUIRE(g.P >= nprocs && g.P >= a.gr * a.gc && g.P >= b.gr * b.gc && g.P >= c.gr * c.gc,
             BT_ERR_INVALID_ARGUMENT, "multiply_virtual_case2: communicator too small");
  const Counters before = ledger_snapshot(g);
  const auto ms = chunk_dist(static_cast<int64_t>(a.rsz.size()), nprocs);
  const auto ks = chunk_dist(static_cast<int64_t>(a.csz.size()), nprocs);
  const std::vector<int32_t> acols(a.csz.size(), 0), bcols(b.csz.size(), 0);
  auto al = relayout(a, nprocs, 1, ms, acols, "redistribute");
  auto bl = relayout(b, nprocs, 1, ks, bcols, "redistribute");
  // C slab target: C itself when it already has the slab layout
  const bool c_is_slab = c.gr == nprocs && c.gc == 1 && c.rdist == ms && c.cdist == bcols;
  std::unique_ptr<DMat> cl_owned;
  DMat* cl = &c;
  if (!c_is_slab) {
    cl_owned = new_dmat(&g, c.rsz, c.csz, nprocs, 1, ms, bcols);
    cl = cl_owned.get();
  }
  g.set_phase("ring");
  if (gather && g.nccl && g.first < nprocs) {
    // NCCL: index first, values overlapped with the symbolic passes
    const int r = g.first;
    if (!g.gather_full || g.gather_full->impl.h_rsz != b.rsz || g.gather_full->impl.h_csz != b.csz)
      g.gather_full = new_store(g.ctx, b.rsz, b.csz);
    Mat& full = g.gather_full->impl;
    // every rank of the communicator in the gather: collective calls (with
    // speculative segment capacities once a first call has sized them, eps = 0);
    // a sub-group: point-to-point rounds
    if (nprocs == g.P && env_int("BT_GATHER_P2P", 0) == 0) {
      bool spec = eps == 0.0 && g.spec_capb > 0 && env_int("BT_GATHER_SPEC", 1) != 0;
      const Mat& mine = bl.view->store(r);
      for (;;) {
        cudaEvent_t vals_ready = gather_rows_allgather(g, mine, ks, nprocs, full, spec);
        try {
          std::function<void()> check = [&] { gather_check(g, mine, nprocs, full, true); };
          // the pass-1 sizes by polling the mapped flag: nothing else of this
          // call is in flight but the already-enqueued all-gathers (4 GPUs:
          // 0.859 -> 0.835 ms per bench step; in Cannon, next to its shifts,
          // polling was slower -- DESIGN.md 4.2)
          rank_multiply(g.ctx, al.view->store(r), full, cl->store(r), eps, S, vals_ready,
                        g.phase_ev, spec ? &check : nullptr, true);
          break;
        } catch (const SpecMiss&) {
          spec = false;  // a slab outgrew its segment: redo exactly (capacities grow)
        }
      }
    } else {
      cudaEvent_t vals_ready = gather_rows_nccl(g, bl.view->store(r), ks, nprocs, full);
      rank_multiply(g.ctx, al.view->store(r), full, cl->store(r), eps, S, vals_ready, g.phase_ev);
    }
    g.phase_ev = nullptr;
  } else if (gather) {
    // all-gather of the B slabs
    std::vector<std::vector<std::unique_ptr<bt_mat>>> got(g.nlocal);
    std::vector<Send> sends;
    std::vector<Recv> recvs;
    for (int lr = 0; lr < g.nlocal; ++lr) {
      const int r = g.first + lr;
      for (int p = 0; p < nprocs; ++p) got[lr].push_back(new_store(g.ctx, b.rsz, b.csz));
      if (r >= nprocs) continue;
      for (int p = 0; p < nprocs; ++p) {
        if (p == r) continue;
        sends.push_back(Send{r, p, &bl.view->store(r)});
        recvs.push_back(Recv{r, p, &got[lr][p]->impl});
      }
    }
    exchange(g, sends, recvs);
    for (int lr = 0; lr < g.nlocal; ++lr) {
      const int r = g.first + lr;
      if (r >= nprocs) continue;
      std::vector<const Mat*> parts;
      for (int p = 0; p < nprocs; ++p) parts.push_back(p == r ? &bl.view->store(r) : &got[lr][p]->impl);
      auto full = new_store(g.ctx, b.rsz, b.csz);
      concat_rows(parts, ks, full->impl);
      rank_multiply(g.ctx, al.view->store(r), full->impl, cl->store(r), eps, S);
    }
  } else {
    std::vector<std::unique_ptr<bt_mat>> cur, nxt;
    for (int lr = 0; lr < g.nlocal; ++lr) {
      cur.push_back(new_store(g.ctx, b.rsz, b.csz));
      nxt.push_back(new_store(g.ctx, b.rsz, b.csz));
      const int r = g.first + lr;
      if (r < nprocs) copy_store(bl.view->store(r), cur[lr]->impl);
    }
    for (int step = 0; step < nprocs; ++step) {
      if (nprocs > 1) {
        std::vector<Send> sends;
        std::vector<Recv> recvs;
        for (int lr = 0; lr < g.nlocal; ++lr) {
          const int r = g.first + lr;
          if (r >= nprocs) continue;
          sends.push_back(Send{r, (r - 1 + nprocs) % nprocs, &cur[lr]->impl});  // up
          recvs.push_back(Recv{r, (r + 1) % nprocs, &nxt[lr]->impl});           // from down
        }
        exchange(g, sends, recvs, true, /*async=*/true);
      }
      for (int lr = 0; lr < g.nlocal; ++lr) {
        const int r = g.first + lr;
        if (r >= nprocs) continue;
        // the A window (rank+step)%P is implicit: cur only holds that K slab
        rank_multiply(g.ctx, al.view->store(r), cur[lr]->impl, cl->store(r), eps, S);
      }
      if (nprocs > 1) {
        finish_exchange(g);
        std::swap(cur, nxt);
      }
    }
  }
  if (!c_is_slab) redistribute(*cl, c, false, true, "collect");
  BT_CUDA(cudaStreamSynchronize(g.ctx->stream));
  ledger_stats(g, before, S);
}

}  // namespace bt

// ===================================================================== C-ABI
using namespace bt;

struct bt_grid {
  Grid impl;
};
struct bt_dmat {
  std::unique_ptr<DMat> impl;
};

extern "C" {

int bt_grid_create(bt_ctx* ctx, int nranks, bt_grid** out) {
  return guard([&] {
    BT_REQUIRE(ctx && out, BT_ERR_INVALID_ARGUMENT, "null argument");
    BT_REQUIRE(nranks >= 1, BT_ERR_INVALID_ARGUMENT, "ProcessGrid: size must be >= 1");
    Ctx& x = ctx->impl;
    auto* g = new bt_grid;
    Grid& G = g->impl;
    G.ctx = &x;
    G.P = nranks;
    if (x.nranks > 1) {
      BT_REQUIRE(nranks == x.nranks, BT_ERR_INVALID_ARGUMENT,
                 "bt_grid_create: an NCCL context's group has exactly its world size");
      G.nccl = true;
      G.first = x.rank;
      G.nlocal = 1;
      BT_CUDA(cudaStreamCreateWithFlags(&G.comm, cudaStreamNonBlocking));
      BT_CUDA(cudaStreamCreateWithFlags(&G.comm_vals, cudaStreamNonBlocking));
    } else {
      G.first = 0;
      G.nlocal = nranks;
    }
    BT_CUDA(cudaEventCreateWithFlags(&G.ev_comm, cudaEventDisableTiming));
    BT_CUDA(cudaEventCreateWithFlags(&G.ev_main, cudaEventDisableTiming));
    BT_CUDA(cudaEventCreateWithFlags(&G.ev_idx, cudaEventDisableTiming));
    BT_CUDA(cudaEventCreateWithFlags(&G.ev_sizes, cudaEventDisableTiming));
    G.totals.assign(nranks, Counters{});
    G.phases.assign(nranks, {});
    G.phase.assign(nranks, "");
    *out = g;
  });
}

int bt_grid_destroy(bt_grid* g) {
  return guard([&] {
    if (!g) return;
    Grid& G = g->impl;
    cudaStreamSynchronize(G.ctx->stream);
    if (G.comm) {
      cudaStreamSynchronize(G.comm);
      cudaStreamDestroy(G.comm);
    }
    if (G.comm_vals) {
      cudaStreamSynchronize(G.comm_vals);
      cudaStreamDestroy(G.comm_vals);
    }
    if (G.ev_comm) cudaEventDestroy(G.ev_comm);
    if (G.ev_main) cudaEventDestroy(G.ev_main);
    if (G.ev_idx) cudaEventDestroy(G.ev_idx);
    if (G.ev_sizes) cudaEventDestroy(G.ev_sizes);
    delete g;
  });
}

int bt_grid_info(const bt_grid* g, int* nranks, int* first_local, int* nlocal) {
  return guard([&] {
    BT_REQUIRE(g, BT_ERR_INVALID_ARGUMENT, "null grid");
    if (nranks) *nranks = g->impl.P;
    if (first_local) *first_local = g->impl.first;
    if (nlocal) *nlocal = g->impl.nlocal;
  });
}

int bt_grid_sum(bt_grid* g, int64_t* values, int n) {
  return guard([&] {
    BT_REQUIRE(g && (values || n == 0) && n >= 0, BT_ERR_INVALID_ARGUMENT, "null argument");
    Grid& G = g->impl;
    if (!G.nccl || n == 0) return;  // one process holds every rank: nothing to add
    Ctx& x = *G.ctx;
    int64_t* d = x.ws<int64_t>(14, n);
    BT_CUDA(cudaMemcpyAsync(d, values, 8 * n, cudaMemcpyHostToDevice, x.stream));
    const ncclResult_t r = ncclAllReduce(d, d, n, ncclInt64, ncclSum,
                                         static_cast<ncclComm_t>(x.nccl), x.stream);
    BT_REQUIRE(r == ncclSuccess, BT_ERR_NCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
    BT_CUDA(cudaMemcpyAsync(values, d, 8 * n, cudaMemcpyDeviceToHost, x.stream));
    BT_CUDA(cudaStreamSynchronize(x.stream));
  });
}

int bt_grid_ledger(const bt_grid* g, int rank, const char* phase, int what, int64_t* out) {
  return guard([&] {
    BT_REQUIRE(g && out, BT_ERR_INVALID_ARGUMENT, "null argument");
    const Grid& G = g->impl;
    BT_REQUIRE(rank >= 0 && rank < G.P && what >= 0 && what < 4, BT_ERR_INVALID_ARGUMENT,
               "bt_grid_ledger: bad rank or counter");
    if (phase && *phase) {
      auto it = G.phases[rank].find(phase);
      *out = it == G.phases[rank].end() ? 0 : it->second.v[what];
    } else {
      *out = G.totals[rank].v[what];
    }
  });
}

int bt_grid_reset_ledger(bt_grid* g) {
  return guard([&] {
    BT_REQUIRE(g, BT_ERR_INVALID_ARGUMENT, "null grid");
    for (auto& t : g->impl.totals) t = Counters{};
    for (auto& p : g->impl.phases) p.clear();
  });
}

int bt_dmat_create(bt_grid* g, int64_t nbr, const int32_t* rsz, int64_t nbc, const int32_t* csz,
                   int grid_rows, int grid_cols, const int32_t* row_dist,
                   const int32_t* col_dist, bt_dmat** out) {
  return guard([&] {
    BT_REQUIRE(g && out, BT_ERR_INVALID_ARGUMENT, "null argument");
    BT_REQUIRE(nbr >= 0 && nbc >= 0, BT_ERR_INVALID_ARGUMENT, "negative block count");
    for (int64_t t = 0; t < nbr; ++t)
      BT_REQUIRE(rsz[t] >= 1, BT_ERR_INVALID_ARGUMENT, "Blocking: block sizes must be positive");
    for (int64_t t = 0; t < nbc; ++t)
      BT_REQUIRE(csz[t] >= 1, BT_ERR_INVALID_ARGUMENT, "Blocking: block sizes must be positive");
    std::vector<int32_t> rd(nbr), cd(nbc);
    for (int64_t t = 0; t < nbr; ++t) rd[t] = row_dist ? row_dist[t] : static_cast<int32_t>(t % grid_rows);
    for (int64_t t = 0; t < nbc; ++t) cd[t] = col_dist ? col_dist[t] : static_cast<int32_t>(t % grid_cols);
    BT_CUDA(cudaSetDevice(g->impl.ctx->device));
    auto* d = new bt_dmat;
    d->impl = new_dmat(&g->impl, std::vector<int32_t>(rsz, rsz + nbr),
                       std::vector<int32_t>(csz, csz + nbc), grid_rows, grid_cols, std::move(rd),
                       std::move(cd));
    *out = d;
  });
}

int bt_dmat_destroy(bt_dmat* d) {
  return guard([&] { delete d; });
}

int bt_dmat_local(bt_dmat* d, int rank, bt_mat** store) {
  return guard([&] {
    BT_REQUIRE(d && store, BT_ERR_INVALID_ARGUMENT, "null argument");
    const Grid& G = *d->impl->g;
    BT_REQUIRE(G.is_local(rank), BT_ERR_OWNERSHIP,
               "bt_dmat_local: rank " + std::to_string(rank) + " is not local to this process");
    *store = d->impl->local[rank - G.first].get();
  });
}

int bt_dmat_owner(const bt_dmat* d, int64_t i, int64_t j, int* rank) {
  return guard([&] {
    BT_REQUIRE(d && rank, BT_ERR_INVALID_ARGUMENT, "null argument");
    BT_REQUIRE(i >= 0 && i < d->impl->nbr && j >= 0 && j < d->impl->nbc, BT_ERR_INVALID_ARGUMENT,
               "owner_rank: block index out of range");
    *rank = d->impl->owner(i, j);
  });
}

int bt_dmat_put_blocks(bt_dmat* d, int64_t n, const int64_t* bi, const int64_t* bj,
                       const double* vals, int accumulate) {
  return guard([&] {
    BT_REQUIRE(d, BT_ERR_INVALID_ARGUMENT, "null argument");
    DMat& D = *d->impl;
    const Grid& G = *D.g;
    std::vector<std::vector<int64_t>> ri(G.nlocal), rj(G.nlocal);
    std::vector<std::vector<double>> rv(G.nlocal);
    int64_t v = 0;
    for (int64_t t = 0; t < n; ++t) {
      BT_REQUIRE(bi[t] >= 0 && bi[t] < D.nbr && bj[t] >= 0 && bj[t] < D.nbc,
                 BT_ERR_INVALID_ARGUMENT, "put_block: block index out of range");
      const int o = D.owner(bi[t], bj[t]);
      const int64_t sz = int64_t(D.rsz[bi[t]]) * D.csz[bj[t]];
      BT_REQUIRE(G.is_local(o), BT_ERR_OWNERSHIP,
                 "put_block: block (" + std::to_string(bi[t]) + "," + std::to_string(bj[t]) +
                     ") is owned by rank " + std::to_string(o) + ", not local to this process");
      ri[o - G.first].push_back(bi[t]);
      rj[o - G.first].push_back(bj[t]);
      rv[o - G.first].insert(rv[o - G.first].end(), vals + v, vals + v + sz);
      v += sz;
    }
    for (int lr = 0; lr < G.nlocal; ++lr)
      if (!ri[lr].empty()) {
        const int rc = bt_mat_put_blocks(D.local[lr].get(), static_cast<int64_t>(ri[lr].size()),
                                         ri[lr].data(), rj[lr].data(), rv[lr].data(), accumulate);
        if (rc != BT_OK) throw Error(rc, bt_last_error());
      }
  });
}

int bt_redistribute(const bt_dmat* src, bt_dmat* dst, int transpose, int accumulate,
                    const char* phase) {
  return guard([&] {
    BT_REQUIRE(src && dst, BT_ERR_INVALID_ARGUMENT, "null argument");
    BT_REQUIRE(src->impl->g == dst->impl->g, BT_ERR_INVALID_ARGUMENT,
               "redistribute: matrices belong to different groups");
    redistribute(*src->impl, *dst->impl, transpose != 0, accumulate != 0,
                 phase && *phase ? phase : "redistribute");
  });
}

int bt_multiply_cannon(const bt_dmat* a, const bt_dmat* b, bt_dmat* c, double eps,
                       bt_stats* stats) {
  return guard([&] {
    BT_REQUIRE(a && b && c, BT_ERR_INVALID_ARGUMENT, "null argument");
    bt_stats S{};
    cannon(*a->impl, *b->impl, *c->impl, eps, S);
    if (stats) *stats = S;
  });
}

int bt_multiply_case1(const bt_dmat* a, const bt_dmat* b, bt_dmat* c, int nprocs, double eps,
                      bt_stats* stats) {
  return guard([&] {
    BT_REQUIRE(a && b && c, BT_ERR_INVALID_ARGUMENT, "null argument");
    bt_stats S{};
    case1(*a->impl, *b->impl, *c->impl, nprocs, eps, S);
    if (stats) *stats = S;
  });
}

int bt_multiply_case2(const bt_dmat* a, const bt_dmat* b, bt_dmat* c, int nprocs, int gather,
                      double eps, bt_stats* stats) {
  return guard([&] {
    BT_REQUIRE(a && b && c, BT_ERR_INVALID_ARGUMENT, "null argument");
    bt_stats S{};
    case2(*a->impl, *b->impl, *c->impl, nprocs, gather, eps, S);
    if (stats) *stats = S;
  });
}

}  // extern "C"
