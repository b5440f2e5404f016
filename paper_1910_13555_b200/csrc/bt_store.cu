// bt_store.cu -- context and device block-CSR store (LocalStore equivalent).
//
// Reference: matrix.hpp:137-275 (LocalStore), :279-401 (DistMatrix put/get),
// :404-418 (new_matrix).  The store is device resident; host buffers only
// cross the boundary inside put/export/get calls.
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <numeric>

#include "bt_internal.cuh"

namespace bt {

static thread_local std::string g_last_error;

double Trace::now() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}
// Every traced API call is also an NVTX range (marks for its phases), so an
// ncu / Nsight timeline shows put / multiply / export / redistribute by name;
// without an attached tool NVTX calls are a pointer test.
Trace::Trace(const char* w) : what(w) {
  static const bool enabled = [] {
    const char* v = getenv("BT_TRACE");
    return v && *v == '1';
  }();
  on = enabled;
  t0 = last = on ? now() : 0.0;
  nvtxRangePushA(w);
}
void Trace::mark(const char* phase) {
  nvtxMarkA(phase);
  if (!on) return;
  const double t = now();
  fprintf(stderr, "[bt-trace] %s %-18s %8.3f ms\n", what, phase, t - last);
  last = t;
}
Trace::~Trace() {
  nvtxRangePop();
  if (on) fprintf(stderr, "[bt-trace] %s %-18s %8.3f ms\n", what, "TOTAL", now() - t0);
}
void set_last_error(const std::string& msg) { g_last_error = msg; }

void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    throw Error(BT_ERR_CUDA, std::string("kernel launch failed (") + what + "): " +
                                 cudaGetErrorString(e));
}

void* Ctx::ensure_scratch(size_t bytes) {
  if (scratch.n < bytes) scratch.alloc(std::max(bytes, size_t(1) << 20), stream);
  return scratch.p;
}

void Ctx::sync_all() {
  BT_CUDA(cudaStreamSynchronize(stream));
  for (auto& a : aux)
    if (a) BT_CUDA(cudaStreamSynchronize(a));
  if (xfer) BT_CUDA(cudaStreamSynchronize(xfer));
}

unsigned char* Ctx::host_stage(size_t bytes) {
  BT_CUDA(cudaEventSynchronize(stage_ev));  // the previous upload has read it
  if (hstage_cap < bytes) {
    if (hstage) BT_CUDA(cudaFreeHost(hstage));
    hstage = nullptr;
    const size_t cap = std::max(bytes + bytes / 4, size_t(1) << 20);
    BT_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&hstage), cap, cudaHostAllocMapped));
    BT_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hstage_dev), hstage, 0));
    hstage_cap = cap;
  }
  return hstage;
}

// BT_ZEROCOPY=1 lets kernels access page-locked host buffers in place (PCIe
// loads/stores from the SMs) instead of copy-engine transfers.  Off by
// default: measured on B200 (c1, 68 MB puts / 667 MB export) the copy engine
// is faster (put 1.29 vs 1.52 ms, export 12.9 vs 15.2 ms).
static bool zero_copy_enabled() {
  static const bool on = [] {
    const char* v = getenv("BT_ZEROCOPY");
    return v && *v == '1';
  }();
  return on;
}

void* mapped_host_alias(const void* p) {
  if (!p) return nullptr;
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, p) != cudaSuccess) {
    cudaGetLastError();  // unregistered host memory
    return nullptr;
  }
  if (pa.type != cudaMemoryTypeHost) return nullptr;
  return pa.devicePointer;  // the device address of p itself (UVA: p)
}

void upload_parts(Ctx& x, const HostPart* parts, int n, void* const* dst) {
  size_t total = 0;
  std::vector<size_t> at(n);
  for (int t = 0; t < n; ++t) {
    at[t] = total;
    total += (parts[t].bytes + 255) & ~size_t(255);
  }
  unsigned char* h = x.host_stage(std::max<size_t>(total, 256));
  for (int t = 0; t < n; ++t)
    if (parts[t].bytes) std::memcpy(h + at[t], parts[t].src, parts[t].bytes);
  for (int t = 0; t < n; ++t)
    if (parts[t].bytes)
      BT_CUDA(cudaMemcpyAsync(dst[t], h + at[t], parts[t].bytes, cudaMemcpyHostToDevice, x.stream));
  BT_CUDA(cudaEventRecord(x.stage_ev, x.stream));
}

void upload_sizes(Mat& m) {
  m.rsz.alloc(std::max<int64_t>(m.nbr, 1), m.stream());
  m.csz.alloc(std::max<int64_t>(m.nbc, 1), m.stream());
  if (m.nbr)
    BT_CUDA(cudaMemcpyAsync(m.rsz.p, m.h_rsz.data(), sizeof(int32_t) * m.nbr,
                            cudaMemcpyHostToDevice, m.stream()));
  if (m.nbc)
    BT_CUDA(cudaMemcpyAsync(m.csz.p, m.h_csz.data(), sizeof(int32_t) * m.nbc,
                            cudaMemcpyHostToDevice, m.stream()));
  m.max_r = m.nbr ? *std::max_element(m.h_rsz.begin(), m.h_rsz.end()) : 0;
  m.max_c = m.nbc ? *std::max_element(m.h_csz.begin(), m.h_csz.end()) : 0;
  m.uniform_r = m.nbr == 0 || std::all_of(m.h_rsz.begin(), m.h_rsz.end(),
                                          [&](int32_t s) { return s == m.h_rsz[0]; });
  m.uniform_c = m.nbc == 0 || std::all_of(m.h_csz.begin(), m.h_csz.end(),
                                          [&](int32_t s) { return s == m.h_csz[0]; });
}

void Mat::clear_keep_capacity() {
  nblk = 0;
  norms_ok = false;
  nelems = 0;
  nvals = 0;
  if (row_ptr.n < static_cast<size_t>(nbr + 1)) row_ptr.alloc(nbr + 1, stream());
  BT_CUDA(cudaMemsetAsync(row_ptr.p, 0, sizeof(int32_t) * (nbr + 1), stream()));
}

void Mat::init_empty() {
  nblk = 0;
  norms_ok = false;
  nelems = 0;
  nvals = 0;
  col.release();
  off.release();
  vals.release();
  row_ptr.alloc(nbr + 1, stream());
  BT_CUDA(cudaMemsetAsync(row_ptr.p, 0, sizeof(int32_t) * (nbr + 1), stream()));
}

// ----------------------------------------------------------------- kernels
// One warp per block: copy a padded slot (even length, 16-byte aligned on both
// sides) with 16-byte vector accesses.
__global__ void k_gather_blocks(double* __restrict__ dst, const int64_t* __restrict__ dst_off,
                                const double* __restrict__ src,
                                const int64_t* __restrict__ src_off,
                                const int64_t* __restrict__ len, int64_t n) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const int64_t so = src_off[w];
  if (so < 0) return;
  const double2* s = reinterpret_cast<const double2*>(src + so);
  double2* d = reinterpret_cast<double2*>(dst + dst_off[w]);
  const int64_t n2 = len[w] >> 1;  // T8 slots: multiples of 64 doubles
  for (int64_t t = lane; t < n2; t += 32) d[t] = s[t];
}

// Put plan application: output block w = base (old slot or first input) +
// remaining inputs in batch order (LocalStore::insert accumulate semantics,
// matrix.hpp:176-179).  Inputs are compact row-major, old/new slots are T8;
// the new slab is zeroed beforehand so T8 padding stays zero.
__global__ void k_apply_put(double* __restrict__ dst, const int64_t* __restrict__ dst_off,
                            const int2* __restrict__ dims, const double* __restrict__ old,
                            const int64_t* __restrict__ old_off,
                            const double* __restrict__ inp, const int64_t* __restrict__ inp_ptr,
                            const int64_t* __restrict__ inp_src, int64_t n) {
  const int64_t w = blockIdx.x;
  if (w >= n) return;
  const int m = dims[w].x, nn = dims[w].y, ntc = tiles8(nn);
  double* d = dst + dst_off[w];
  const int64_t oo = old_off[w];
  const int64_t i0 = inp_ptr[w], i1 = inp_ptr[w + 1];
  for (int e = threadIdx.x; e < m * nn; e += blockDim.x) {
    const int r = e / nn, c = e - r * nn;
    const int64_t tp = t8_pos(r, c, ntc);
    double v;
    int64_t t = i0;
    if (oo >= 0) {
      v = old[oo + tp];
    } else {
      v = inp[inp_src[t] + e];
      ++t;
    }
    for (; t < i1; ++t) v = __dadd_rn(v, inp[inp_src[t] + e]);
    d[tp] = v;
  }
}

// Export plan: per stored entry its block row, block column and element count
// (the count is scanned into compact offsets afterwards).
__global__ void k_export_plan(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                              const int32_t* __restrict__ rsz, const int32_t* __restrict__ csz,
                              int64_t nbr, int64_t* __restrict__ bi, int64_t* __restrict__ bj,
                              int64_t* __restrict__ len, int64_t n) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e > n) return;
  if (e == n) {
    len[n] = 0;
    return;
  }
  int64_t lo = 0, hi = nbr;  // row of entry e: last r with row_ptr[r] <= e
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (row_ptr[mid] <= e) lo = mid; else hi = mid;
  }
  const int32_t j = col[e];
  bi[e] = lo;
  bj[e] = j;
  len[e] = static_cast<int64_t>(rsz[lo]) * csz[j];
}

// Export metadata straight into mapped page-locked host memory (no copy-engine
// D2H, which would queue behind a pending asynchronous value transfer): the
// block index (bi, bj) of every entry, and the compact offsets of the chunk
// boundaries the host needs to enqueue the per-chunk value copies.
__global__ void k_export_meta(const int64_t* __restrict__ d_bi, const int64_t* __restrict__ d_bj,
                              const int64_t* __restrict__ coff, int64_t n,
                              int64_t* __restrict__ h_bi, int64_t* __restrict__ h_bj,
                              const int64_t* __restrict__ cb, int ncb, int64_t* __restrict__ h_co) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (h_bi && e < n) {
    h_bi[e] = d_bi[e];
    h_bj[e] = d_bj[e];
  }
  if (e < ncb) h_co[e] = coff[cb[e]];
}

// T8 slot -> compact row-major (host order).  dst may be mapped host memory:
// consecutive threads write consecutive doubles, so the PCIe writes coalesce.
__global__ void k_compact(double* __restrict__ dst, const int64_t* __restrict__ dst_off,
                          const double* __restrict__ src, const int64_t* __restrict__ src_off,
                          const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                          const int32_t* __restrict__ rsz, const int32_t* __restrict__ csz,
                          int64_t w0, int64_t w1) {
  const int64_t w = w0 + blockIdx.x;
  if (w >= w1) return;
  const int m = rsz[row[w]], nn = csz[col[w]], ntc = tiles8(nn);
  const double* s = src + src_off[w];
  double* d = dst + dst_off[w];
  for (int e = threadIdx.x; e < m * nn; e += blockDim.x) {
    const int r = e / nn, c = e - r * nn;
    d[e] = s[t8_pos(r, c, ntc)];
  }
}

// Frobenius norm per block: squares summed along each row, then
// the row sums added in row order; unfused, so the oracle's identical loop
// gives identical bits.  One warp per block, one lane per row (32 rows at a
// time): the dependent chain is n + m additions, not m * n.
// Launch with kNormThreads threads per CTA.
__device__ __forceinline__ void block_norm(const double* __restrict__ vals,
                                           const int32_t* __restrict__ row_ptr,
                                           const int32_t* __restrict__ col,
                                           const int64_t* __restrict__ off,
                                           const int32_t* __restrict__ rsz,
                                           const int32_t* __restrict__ csz, int64_t nbr,
                                           double* __restrict__ out, int64_t b, int lane) {
  // row of entry b (last r with row_ptr[r] <= b): 32-way search, one probe
  // per lane per step, so ~log32(nbr) dependent loads instead of log2(nbr)
  int64_t lo = 0, hi = nbr;  // row_ptr[lo] <= b < row_ptr[hi]
  while (hi - lo > 1) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t probe = lo + static_cast<int64_t>(lane) * step;
    const bool le = probe < hi && row_ptr[probe] <= b;
    const unsigned ok = __ballot_sync(0xffffffffu, le);
    const int last = 31 - __clz(ok);  // probe 0 (= lo) always qualifies
    const int64_t nlo = lo + static_cast<int64_t>(last) * step;
    hi = min(hi, nlo + step);
    lo = nlo;
  }
  const int m = rsz[lo], n = csz[col[b]], ntc = tiles8(n);
  const double* p = vals + off[b];
  double s = 0.0;
  for (int r0 = 0; r0 < m; r0 += 32) {
    const int r = r0 + lane;
    double rs = 0.0;
    if (r < m) {
      // row r, 8 columns per T8 tile: one contiguous 64-byte tile row, stored
      // with the swizzle (column u at u ^ sw); the zero padding past column n
      // adds +0.0, which leaves the (non-negative) sum bit-identical
      const int sw = ((r >> 1) & 1) << 2;
      const double2* tr = reinterpret_cast<const double2*>(p + (((r >> 3) * ntc) << 6) +
                                                           ((r & 7) << 3));
      for (int tc = 0; tc < ntc; ++tc) {
        double w[8];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const double2 d = tr[(tc << 5) + h];  // tile tc: 64 doubles = 32 double2
          w[2 * h] = d.x;
          w[2 * h + 1] = d.y;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double v = sw ? w[u ^ 4] : w[u];
          rs = __dadd_rn(rs, __dmul_rn(v, v));
        }
      }
    }
    const int cnt = min(32, m - r0);
    for (int k = 0; k < cnt; ++k) s = __dadd_rn(s, __shfl_sync(0xffffffffu, rs, k));
  }
  if (lane == 0) out[b] = __dsqrt_rn(s);
}

__global__ void k_block_norms(const double* __restrict__ vals, const int32_t* __restrict__ row_ptr,
                              const int32_t* __restrict__ col, const int64_t* __restrict__ off,
                              const int32_t* __restrict__ rsz, const int32_t* __restrict__ csz,
                              int64_t nbr, double* __restrict__ out, int64_t nblk) {
  const int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (b >= nblk) return;
  block_norm(vals, row_ptr, col, off, rsz, csz, nbr, out, b, threadIdx.x & 31);
}

// latency-bound (a few dependent loads per warp): occupancy hides it best, so
// 8 CTAs of 256 threads per SM (32 registers; a per-warp preload variant with
// 72 registers was 40 % slower, profiles/r01d/norms_preload_ab.txt)
__global__ void __launch_bounds__(256, 8) k_block_norms_pair(NormSrc a, NormSrc b) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w < a.nblk) {
    block_norm(a.vals, a.row_ptr, a.col, a.off, a.rsz, a.csz, a.nbr, a.out, w, lane);
  } else if (w - a.nblk < b.nblk) {
    block_norm(b.vals, b.row_ptr, b.col, b.off, b.rsz, b.csz, b.nbr, b.out, w - a.nblk, lane);
  }
}

const double* Mat::norms(cudaStream_t st) const {
  if (nblk == 0) return nullptr;
  if (!norms_ok || norm_cache.n < static_cast<size_t>(nblk)) {
    if (norm_cache.n < static_cast<size_t>(nblk)) norm_cache.alloc(nblk, st);
    k_block_norms<<<static_cast<unsigned>((nblk * 32 + kNormThreads - 1) / kNormThreads),
                    kNormThreads, 0, st>>>(vals.p, row_ptr.p, col.p, off.p, rsz.p, csz.p, nbr,
                                           norm_cache.p, nblk);
    check_launch("block_norms");
    count_launch(ctx);
    norms_ok = true;
  }
  return norm_cache.p;
}

// ------------------------------------------------------------- host helpers
struct HostIndex {
  std::vector<int32_t> row_ptr, col;
  std::vector<int64_t> off;
};

// Index readback through the pinned stage (pageable D2H copies are slow).
static HostIndex download_index(const Mat& m) {
  HostIndex h;
  h.row_ptr.resize(m.nbr + 1);
  h.col.resize(m.nblk);
  h.off.resize(m.nblk);
  const size_t brp = sizeof(int32_t) * (m.nbr + 1);
  const size_t bcol = (sizeof(int32_t) * m.nblk + 255) & ~size_t(255);
  const size_t boff = sizeof(int64_t) * m.nblk;
  unsigned char* st = m.ctx->host_stage(((brp + 255) & ~size_t(255)) + bcol + boff);
  unsigned char* s_col = st + ((brp + 255) & ~size_t(255));
  unsigned char* s_off = s_col + bcol;
  BT_CUDA(cudaMemcpyAsync(st, m.row_ptr.p, brp, cudaMemcpyDeviceToHost, m.stream()));
  if (m.nblk) {
    BT_CUDA(cudaMemcpyAsync(s_col, m.col.p, sizeof(int32_t) * m.nblk, cudaMemcpyDeviceToHost,
                            m.stream()));
    BT_CUDA(cudaMemcpyAsync(s_off, m.off.p, boff, cudaMemcpyDeviceToHost, m.stream()));
  }
  BT_CUDA(cudaStreamSynchronize(m.stream()));
  std::memcpy(h.row_ptr.data(), st, brp);
  if (m.nblk) {
    std::memcpy(h.col.data(), s_col, sizeof(int32_t) * m.nblk);
    std::memcpy(h.off.data(), s_off, boff);
  }
  return h;
}

template <class T>
static HostPart part(const std::vector<T>& v) {
  return HostPart{v.data(), sizeof(T) * v.size()};
}

template <class T>
static DBuf<T> upload(const std::vector<T>& v, cudaStream_t s) {
  DBuf<T> d(std::max<size_t>(v.size(), 1), s);
  if (!v.empty())
    BT_CUDA(cudaMemcpyAsync(d.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, s));
  return d;
}

// Installs a new pattern (index arrays through the pinned stage); the caller
// provides the value slab.
static void install_pattern(Mat& m, const std::vector<int32_t>& row_ptr,
                            const std::vector<int32_t>& col, const std::vector<int64_t>& off,
                            int64_t nvals, int64_t nelems) {
  m.row_ptr.alloc(std::max<size_t>(row_ptr.size(), 1), m.stream());
  m.col.alloc(std::max<size_t>(col.size(), 1), m.stream());
  m.off.alloc(std::max<size_t>(off.size(), 1), m.stream());
  const HostPart parts[3] = {part(row_ptr), part(col), part(off)};
  void* const dst[3] = {m.row_ptr.p, m.col.p, m.off.p};
  upload_parts(*m.ctx, parts, 3, dst);
  m.nblk = static_cast<int64_t>(col.size());
  m.norms_ok = false;
  m.nvals = nvals;
  m.nelems = nelems;
}

static void check_mat(const bt_mat* m) {
  BT_REQUIRE(m != nullptr, BT_ERR_INVALID_ARGUMENT, "null matrix handle");
}

}  // namespace bt

using namespace bt;

extern "C" {

const char* bt_last_error(void) { return g_last_error.c_str(); }
int bt_version(void) { return 1; }

int bt_get_unique_id(void* id128) {
  return guard([&] {
    BT_REQUIRE(id128, BT_ERR_INVALID_ARGUMENT, "null id buffer");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    BT_REQUIRE(r == ncclSuccess, BT_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(id) == 128, "nccl id size");
    std::memcpy(id128, &id, 128);
  });
}

// device, streams, pool, pinned staging and events of a new context
static bt_ctx* new_ctx(int device) {
  int ndev = 0;
  BT_CUDA(cudaGetDeviceCount(&ndev));
  BT_REQUIRE(device >= 0 && device < ndev, BT_ERR_INVALID_ARGUMENT,
             "bt_ctx_create: device " + std::to_string(device) + " not present (" +
                 std::to_string(ndev) + " visible)");
  BT_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  BT_CUDA(cudaGetDeviceProperties(&prop, device));
  BT_REQUIRE(prop.major == 10, BT_ERR_CUDA,
             std::string("libbtcuda is built for sm_100a (B200); device is ") + prop.name);
  auto* c = new bt_ctx;
  Ctx& x = c->impl;
  x.device = device;
  x.num_sms = prop.multiProcessorCount;
  x.smem_optin = prop.sharedMemPerBlockOptin;
  BT_CUDA(cudaStreamCreateWithFlags(&x.stream, cudaStreamNonBlocking));
  cudaMemPool_t pool;
  BT_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = UINT64_MAX;
  BT_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  BT_CUDA(cudaHostAlloc(&x.pinned, Ctx::kPinnedBytes, cudaHostAllocMapped));
  BT_CUDA(cudaHostGetDevicePointer(&x.pinned_dev, x.pinned, 0));
  BT_CUDA(cudaEventCreateWithFlags(&x.stage_ev, cudaEventDisableTiming));
  for (auto& e : x.ev) BT_CUDA(cudaEventCreate(&e));
  for (auto& a : x.aux) BT_CUDA(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
  BT_CUDA(cudaStreamCreateWithFlags(&x.xfer, cudaStreamNonBlocking));
  BT_CUDA(cudaEventCreateWithFlags(&x.ev_fork, cudaEventDisableTiming));
  for (auto& e : x.xfer_done) BT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : x.ev_join) BT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return c;
}

int bt_ctx_create(int device, int nranks, int rank, const void* nccl_id, bt_ctx** out) {
  return guard([&] {
    BT_REQUIRE(out, BT_ERR_INVALID_ARGUMENT, "null output handle");
    BT_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, BT_ERR_INVALID_ARGUMENT,
               "bt_ctx_create: bad rank/nranks");
    BT_REQUIRE(nranks == 1 || nccl_id, BT_ERR_INVALID_ARGUMENT,
               "bt_ctx_create: nranks > 1 needs an NCCL unique id");
    bt_ctx* c = new_ctx(device);
    Ctx& x = c->impl;
    x.nranks = nranks;
    x.rank = rank;
    if (nranks > 1) {
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, 128);
      ncclComm_t comm;
      ncclResult_t r = ncclCommInitRank(&comm, nranks, id, rank);
      if (r != ncclSuccess) {
        bt_ctx_destroy(c);
        throw Error(BT_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
      }
      x.nccl = comm;
    }
    *out = c;
  });
}

int bt_ctx_split(bt_ctx* parent, int color, int key, bt_ctx** out) {
  return guard([&] {
    BT_REQUIRE(parent && out, BT_ERR_INVALID_ARGUMENT, "null argument");
    BT_REQUIRE(parent->impl.nccl, BT_ERR_INVALID_ARGUMENT,
               "bt_ctx_split: the parent context has no NCCL communicator (one process holds "
               "every rank: use one context per subgroup instead)");
    BT_REQUIRE(color >= 0, BT_ERR_INVALID_ARGUMENT, "bt_ctx_split: color must be >= 0");
    ncclComm_t sub = nullptr;
    ncclResult_t r = ncclCommSplit(static_cast<ncclComm_t>(parent->impl.nccl), color, key, &sub,
                                   nullptr);
    BT_REQUIRE(r == ncclSuccess, BT_ERR_NCCL, std::string("ncclCommSplit: ") + ncclGetErrorString(r));
    int n = 1, me = 0;
    ncclCommCount(sub, &n);
    ncclCommUserRank(sub, &me);
    bt_ctx* c = new_ctx(parent->impl.device);
    c->impl.nranks = n;
    c->impl.rank = me;
    if (n > 1) {
      c->impl.nccl = sub;
    } else {
      ncclCommDestroy(sub);  // a one-rank subgroup is a plain single-GPU context
    }
    *out = c;
  });
}

int bt_ctx_destroy(bt_ctx* c) {
  return guard([&] {
    if (!c) return;
    Ctx& x = c->impl;
    cudaSetDevice(x.device);
    cudaStreamSynchronize(x.stream);
    for (auto& a : x.aux)
      if (a) cudaStreamSynchronize(a);
    if (x.xfer) cudaStreamSynchronize(x.xfer);  // asynchronous exports still in flight
    for (auto& b : x.xstage) b.release();
    for (auto& e : x.xfer_done)
      if (e) cudaEventDestroy(e);
    x.scratch.release();
    for (auto& w : x.ws_slots) w.release();
    cudaStreamSynchronize(x.stream);
    if (x.nccl_vals) ncclCommDestroy(static_cast<ncclComm_t>(x.nccl_vals));
    if (x.nccl) ncclCommDestroy(static_cast<ncclComm_t>(x.nccl));
    if (x.pinned) cudaFreeHost(x.pinned);
    if (x.hstage) cudaFreeHost(x.hstage);
    if (x.stage_ev) cudaEventDestroy(x.stage_ev);
    for (auto& e : x.ev)
      if (e) cudaEventDestroy(e);
    for (auto& a : x.aux)
      if (a) cudaStreamDestroy(a);
    if (x.xfer) cudaStreamDestroy(x.xfer);
    if (x.ev_fork) cudaEventDestroy(x.ev_fork);
    for (auto& e : x.ev_join)
      if (e) cudaEventDestroy(e);
    cudaStreamDestroy(x.stream);
    delete c;
  });
}

int bt_ctx_sync(bt_ctx* c) {
  return guard([&] {
    BT_REQUIRE(c, BT_ERR_INVALID_ARGUMENT, "null context");
    c->impl.sync_all();
  });
}

int bt_ctx_rank(const bt_ctx* c, int* rank, int* nranks) {
  return guard([&] {
    BT_REQUIRE(c, BT_ERR_INVALID_ARGUMENT, "null context");
    if (rank) *rank = c->impl.rank;
    if (nranks) *nranks = c->impl.nranks;
  });
}

int bt_ctx_stream(bt_ctx* c, void** stream) {
  return guard([&] {
    BT_REQUIRE(c && stream, BT_ERR_INVALID_ARGUMENT, "null argument");
    *stream = c->impl.stream;
  });
}

int bt_ctx_kernel_count(const bt_ctx* c, int64_t* count) {
  return guard([&] {
    BT_REQUIRE(c && count, BT_ERR_INVALID_ARGUMENT, "null argument");
    *count = c->impl.kernels;
  });
}

int bt_ctx_set_timing(bt_ctx* c, int on) {
  return guard([&] {
    BT_REQUIRE(c, BT_ERR_INVALID_ARGUMENT, "null context");
    BT_REQUIRE(on >= 0 && on <= 2, BT_ERR_INVALID_ARGUMENT, "bt_ctx_set_timing: mode 0, 1 or 2");
    c->impl.timing = on;
  });
}

int bt_mat_create(bt_ctx* ctx, int64_t nbr, const int32_t* row_sizes, int64_t nbc,
                  const int32_t* col_sizes, bt_mat** out) {
  return guard([&] {
    BT_REQUIRE(ctx && out, BT_ERR_INVALID_ARGUMENT, "null argument");
    BT_REQUIRE(nbr >= 0 && nbc >= 0, BT_ERR_INVALID_ARGUMENT, "negative block count");
    BT_REQUIRE(nbr < (int64_t(1) << 31) - 1 && nbc < (int64_t(1) << 31) - 1,
               BT_ERR_INVALID_ARGUMENT, "block counts must fit int32");
    BT_REQUIRE((nbr == 0 || row_sizes) && (nbc == 0 || col_sizes), BT_ERR_INVALID_ARGUMENT,
               "null blocking");
    for (int64_t t = 0; t < nbr; ++t)
      BT_REQUIRE(row_sizes[t] >= 1, BT_ERR_INVALID_ARGUMENT,
                 "Blocking: block sizes must be positive");
    for (int64_t t = 0; t < nbc; ++t)
      BT_REQUIRE(col_sizes[t] >= 1, BT_ERR_INVALID_ARGUMENT,
                 "Blocking: block sizes must be positive");
    BT_CUDA(cudaSetDevice(ctx->impl.device));
    auto* m = new bt_mat;
    Mat& x = m->impl;
    x.ctx = &ctx->impl;
    x.nbr = nbr;
    x.nbc = nbc;
    x.h_rsz.assign(row_sizes, row_sizes + nbr);
    x.h_csz.assign(col_sizes, col_sizes + nbc);
    upload_sizes(x);
    x.init_empty();
    *out = m;
  });
}

int bt_mat_destroy(bt_mat* m) {
  return guard([&] {
    if (!m) return;
    cudaSetDevice(m->impl.ctx->device);
    delete m;
  });
}

int bt_mat_clear(bt_mat* m) {
  return guard([&] {
    check_mat(m);
    m->impl.clear_keep_capacity();
  });
}

int bt_mat_info(const bt_mat* m, int64_t* nblk, int64_t* nelems) {
  return guard([&] {
    check_mat(m);
    if (nblk) *nblk = m->impl.nblk;
    if (nelems) *nelems = m->impl.nelems;
  });
}

int bt_mat_copy(const bt_mat* src, bt_mat* dst) {
  return guard([&] {
    check_mat(src);
    check_mat(dst);
    const Mat& s = src->impl;
    Mat& d = dst->impl;
    BT_REQUIRE(s.h_rsz == d.h_rsz && s.h_csz == d.h_csz, BT_ERR_INVALID_ARGUMENT,
               "bt_mat_copy: blockings differ");
    cudaStream_t st = d.stream();
    if (s.stream() != st) BT_CUDA(cudaStreamSynchronize(s.stream()));
    d.row_ptr.alloc(d.nbr + 1, st);
    BT_CUDA(cudaMemcpyAsync(d.row_ptr.p, s.row_ptr.p, sizeof(int32_t) * (d.nbr + 1),
                            cudaMemcpyDeviceToDevice, st));
    d.col.alloc(std::max<int64_t>(s.nblk, 1), st);
    d.off.alloc(std::max<int64_t>(s.nblk, 1), st);
    d.vals.alloc(std::max<int64_t>(s.nvals, 2), st);
    if (s.nblk) {
      BT_CUDA(cudaMemcpyAsync(d.col.p, s.col.p, sizeof(int32_t) * s.nblk,
                              cudaMemcpyDeviceToDevice, st));
      BT_CUDA(cudaMemcpyAsync(d.off.p, s.off.p, sizeof(int64_t) * s.nblk,
                              cudaMemcpyDeviceToDevice, st));
      BT_CUDA(cudaMemcpyAsync(d.vals.p, s.vals.p, sizeof(double) * s.nvals,
                              cudaMemcpyDeviceToDevice, st));
    }
    d.nblk = s.nblk;
    d.norms_ok = false;
    d.nvals = s.nvals;
    d.nelems = s.nelems;
  });
}

int bt_mat_put_blocks(bt_mat* mh, int64_t n, const int64_t* bi, const int64_t* bj,
                      const double* vals, int accumulate) {
  return guard([&] {
    check_mat(mh);
    Mat& m = mh->impl;
    BT_REQUIRE(n >= 0, BT_ERR_INVALID_ARGUMENT, "negative block count");
    if (n == 0) return;
    BT_REQUIRE(bi && bj && vals, BT_ERR_INVALID_ARGUMENT, "null input arrays");
    Trace tr("put");
    cudaStream_t st = m.stream();
    BT_CUDA(cudaSetDevice(m.ctx->device));
    // validate + compact input offsets
    std::vector<int64_t> in_off(n);
    int64_t in_total = 0;
    for (int64_t t = 0; t < n; ++t) {
      BT_REQUIRE(bi[t] >= 0 && bi[t] < m.nbr && bj[t] >= 0 && bj[t] < m.nbc,
                 BT_ERR_INVALID_ARGUMENT,
                 "put_block: block (" + std::to_string(bi[t]) + "," + std::to_string(bj[t]) +
                     ") out of range");
      in_off[t] = in_total;
      in_total += int64_t(m.h_rsz[bi[t]]) * m.h_csz[bj[t]];
    }
    tr.mark("validate");
    // an empty store's index is known on the host (no D2H: a copy-engine
    // readback would queue behind an asynchronous export's transfer)
    HostIndex old;
    if (m.nblk == 0)
      old.row_ptr.assign(m.nbr + 1, 0);
    else
      old = download_index(m);
    tr.mark("download_index");
    // values first, so the copy runs while the host plans the merge.
    // device: inputs already in this GPU's memory or in mapped page-locked host
    // memory are read in place by the kernel (no staging copy); anything else
    // is staged with one H2D
    cudaPointerAttributes pa{};
    const bool on_device = cudaPointerGetAttributes(&pa, vals) == cudaSuccess &&
                           pa.type == cudaMemoryTypeDevice && pa.device == m.ctx->device;
    cudaGetLastError();  // clear a possible "invalid value" from unregistered host memory
    const double* src_vals = vals;
    if (!on_device) {
      const double* alias =
          zero_copy_enabled() ? static_cast<const double*>(mapped_host_alias(vals)) : nullptr;
      if (alias) {
        src_vals = alias;
      } else {
        double* d_in = m.ctx->ws<double>(23, in_total);  // grow-only staging
        tr.mark("in_alloc");
        BT_CUDA(cudaMemcpyAsync(d_in, vals, sizeof(double) * in_total, cudaMemcpyHostToDevice, st));
        src_vals = d_in;
      }
    }
    tr.mark("h2d_enqueue");
    // stable order of the batch by (i, j)
    std::vector<int64_t> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    bool sorted = true;
    for (int64_t t = 1; t < n && sorted; ++t)
      if (bi[t] < bi[t - 1] || (bi[t] == bi[t - 1] && bj[t] < bj[t - 1])) sorted = false;
    if (!sorted)
      std::stable_sort(perm.begin(), perm.end(), [&](int64_t x, int64_t y) {
        return bi[x] != bi[y] ? bi[x] < bi[y] : bj[x] < bj[y];
      });
    // merge old pattern with batch keys
    std::vector<int32_t> row_ptr(m.nbr + 1, 0), col;
    std::vector<int64_t> off, old_off, inp_ptr{0}, inp_src;
    std::vector<int2> dims;
    col.reserve(m.nblk + n);
    int64_t nv = 0, ne = 0;
    int64_t p = 0;
    for (int64_t i = 0; i < m.nbr; ++i) {
      int64_t e = old.row_ptr[i], e_end = old.row_ptr[i + 1];
      while (e < e_end || (p < n && bi[perm[p]] == i)) {
        int64_t j;
        const bool have_old = e < e_end;
        const bool have_new = p < n && bi[perm[p]] == i;
        if (have_old && (!have_new || old.col[e] <= bj[perm[p]]))
          j = old.col[e];
        else
          j = bj[perm[p]];
        int64_t src_old = -1;
        if (have_old && old.col[e] == j) {
          src_old = old.off[e];
          ++e;
        }
        // inputs with this key, in batch order
        int64_t q = p;
        while (q < n && bi[perm[q]] == i && bj[perm[q]] == j) ++q;
        if (q > p) {
          if (accumulate) {
            for (int64_t t = p; t < q; ++t) inp_src.push_back(in_off[perm[t]]);
          } else {
            src_old = -1;  // replaced: the last input of the batch wins
            inp_src.push_back(in_off[perm[q - 1]]);
          }
        }
        p = q;
        const int64_t L = int64_t(m.h_rsz[i]) * m.h_csz[j];
        col.push_back(static_cast<int32_t>(j));
        off.push_back(nv);
        dims.push_back(make_int2(m.h_rsz[i], m.h_csz[j]));
        old_off.push_back(src_old);
        inp_ptr.push_back(static_cast<int64_t>(inp_src.size()));
        nv += t8_size(m.h_rsz[i], m.h_csz[j]);
        ne += L;
        row_ptr[i + 1]++;
      }
    }
    for (int64_t i = 0; i < m.nbr; ++i) row_ptr[i + 1] += row_ptr[i];
    BT_REQUIRE(col.size() < (size_t(1) << 31), BT_ERR_INVALID_ARGUMENT,
               "store exceeds 2^31 blocks");
    tr.mark("plan");
    const int64_t nout = static_cast<int64_t>(col.size());
    // an empty store (bt_mat_clear keeps its slab as capacity) is refilled in
    // place: a clear + put cycle allocates nothing
    DBuf<double> new_vals;
    if (m.nblk == 0 && m.vals.n >= static_cast<size_t>(std::max<int64_t>(nv, 2)))
      new_vals = std::move(m.vals);
    else
      new_vals.alloc(std::max<int64_t>(nv, 2), st);
    BT_CUDA(cudaMemsetAsync(new_vals.p, 0, sizeof(double) * std::max<int64_t>(nv, 2), st));
    tr.mark("slab_alloc");
    // plan arrays: one device buffer, one packed upload through the pinned stage
    const HostPart parts[5] = {part(off), part(dims), part(old_off), part(inp_ptr), part(inp_src)};
    size_t at[5], total = 0;
    for (int t = 0; t < 5; ++t) {
      at[t] = total;
      total += (parts[t].bytes + 255) & ~size_t(255);
    }
    DBuf<unsigned char> plan(std::max<size_t>(total, 256), st);
    void* dst[5];
    for (int t = 0; t < 5; ++t) dst[t] = plan.p + at[t];
    upload_parts(*m.ctx, parts, 5, dst);
    k_apply_put<<<static_cast<unsigned>(nout), 128, 0, st>>>(
        new_vals.p, static_cast<const int64_t*>(dst[0]), static_cast<const int2*>(dst[1]),
        m.vals.p, static_cast<const int64_t*>(dst[2]), src_vals,
        static_cast<const int64_t*>(dst[3]), static_cast<const int64_t*>(dst[4]), nout);
    check_launch("apply_put");
    count_launch(m.ctx);
    tr.mark("kernel_enqueue");
    m.vals = std::move(new_vals);
    install_pattern(m, row_ptr, col, off, nv, ne);
    BT_CUDA(cudaStreamSynchronize(st));  // host buffers are borrowed for the call only
    tr.mark("sync");
  });
}

static void export_store(const Mat& m, int64_t* bi, int64_t* bj, double* vals, bool async);

int bt_mat_export(const bt_mat* mh, int64_t* bi, int64_t* bj, double* vals) {
  return guard([&] {
    check_mat(mh);
    export_store(mh->impl, bi, bj, vals, false);
  });
}

int bt_mat_export_async(const bt_mat* mh, int64_t* bi, int64_t* bj, double* vals) {
  return guard([&] {
    check_mat(mh);
    export_store(mh->impl, bi, bj, vals, true);
  });
}

static void export_store(const Mat& m, int64_t* bi, int64_t* bj, double* vals, bool async) {
  {
    Ctx& x = *m.ctx;
    BT_CUDA(cudaSetDevice(x.device));
    if (m.nblk == 0) return;
    cudaStream_t st = m.stream();
    Trace tr("export");
    const int64_t n = m.nblk;
    // device plan: (row, col) per entry and the compact offsets (exclusive scan
    // of m*n in canonical order); the total is the store's element count
    int64_t* d_bi = x.ws<int64_t>(24, n);
    int64_t* d_bj = x.ws<int64_t>(25, n);
    int64_t* d_coff = x.ws<int64_t>(26, n + 1);
    const unsigned g = static_cast<unsigned>((n + 255) / 256);
    k_export_plan<<<g, 256, 0, st>>>(m.row_ptr.p, m.col.p, m.rsz.p, m.csz.p, m.nbr, d_bi, d_bj,
                                     d_coff, n);
    check_launch("export_plan");
    count_launch(&x);
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, d_coff, d_coff, n + 1, st);
    void* tmp = x.ensure_scratch(bytes);
    cub::DeviceScan::ExclusiveSum(tmp, bytes, d_coff, d_coff, n + 1, st);
    check_launch("export_scan");
    count_launch(&x);
    // index + chunk offsets into mapped host memory, then one sync of the
    // main stream (which holds no pending value transfer)
    constexpr int kChunks = 8;
    int64_t cb[kChunks + 1];
    for (int c = 0; c <= kChunks; ++c) cb[c] = n * c / kChunks;
    unsigned char* hs = nullptr;
    unsigned char* hs_dev = nullptr;
    if (bi || bj) {
      hs = x.host_stage(2 * sizeof(int64_t) * n);
      hs_dev = x.hstage_dev;
    }
    int64_t* d_cb = x.ws<int64_t>(22, kChunks + 1);
    BT_CUDA(cudaMemcpyAsync(d_cb, cb, sizeof(cb), cudaMemcpyHostToDevice, st));
    int64_t* meta_co = reinterpret_cast<int64_t*>(x.pinned);
    k_export_meta<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(
        d_bi, d_bj, d_coff, n, reinterpret_cast<int64_t*>(hs_dev),
        hs_dev ? reinterpret_cast<int64_t*>(hs_dev) + n : nullptr, d_cb, kChunks + 1,
        reinterpret_cast<int64_t*>(x.pinned_dev));
    check_launch("export_meta");
    count_launch(&x);
    BT_CUDA(cudaEventRecord(x.stage_ev, st));
    BT_CUDA(cudaStreamSynchronize(st));
    if (bi) std::memcpy(bi, hs, sizeof(int64_t) * n);
    if (bj) std::memcpy(bj, hs + sizeof(int64_t) * n, sizeof(int64_t) * n);
    tr.mark("plan");
    if (vals) {
      double* alias = zero_copy_enabled() ? static_cast<double*>(mapped_host_alias(vals)) : nullptr;
      if (alias) {
        // compact straight into mapped page-locked host memory (PCIe writes)
        k_compact<<<static_cast<unsigned>(n), 128, 0, st>>>(alias, d_coff, m.vals.p, m.off.p, d_bi,
                                                            m.col.p, m.rsz.p, m.csz.p, 0, n);
        check_launch("compact");
        count_launch(&x);
      } else {
        // compact in chunks on the main stream into a staging buffer; each
        // chunk's D2H runs on a side stream as soon as it is compacted (the
        // transfer hides the compaction).  Two staging buffers alternate: this
        // export's compaction waits only for the D2H that last read its buffer.
        const int xb = x.xnext;
        x.xnext ^= 1;
        BT_CUDA(cudaStreamWaitEvent(st, x.xfer_done[xb], 0));
        if (x.xstage[xb].n < static_cast<size_t>(std::max<int64_t>(m.nelems, 1)))
          x.xstage[xb].alloc(std::max<int64_t>(m.nelems, 1) + m.nelems / 4, st);
        double* dst = x.xstage[xb].p;
        int64_t eo[kChunks + 1];
        for (int c = 0; c <= kChunks; ++c) eo[c] = meta_co[c];
        // the value D2H runs on the context's transfer stream: kernels of
        // later calls (side-stream numeric launches use aux[]) never queue
        // behind an asynchronous export
        cudaStream_t cs = x.xfer;
        for (int c = 0; c < kChunks; ++c) {
          if (cb[c + 1] == cb[c]) continue;
          k_compact<<<static_cast<unsigned>(cb[c + 1] - cb[c]), 128, 0, st>>>(
              dst, d_coff, m.vals.p, m.off.p, d_bi, m.col.p, m.rsz.p, m.csz.p, cb[c], cb[c + 1]);
          check_launch("compact");
          count_launch(&x);
          BT_CUDA(cudaEventRecord(x.ev_join[c & 3], st));
          BT_CUDA(cudaStreamWaitEvent(cs, x.ev_join[c & 3], 0));
          BT_CUDA(cudaMemcpyAsync(vals + eo[c], dst + eo[c], sizeof(double) * (eo[c + 1] - eo[c]),
                                  cudaMemcpyDeviceToHost, cs));
        }
        BT_CUDA(cudaEventRecord(x.xfer_done[xb], cs));
        // synchronous export: the values are in `vals` when the call returns
        if (!async) BT_CUDA(cudaStreamWaitEvent(st, x.xfer_done[xb], 0));
      }
      tr.mark("compact_enqueue");
    }
    if (!async) BT_CUDA(cudaStreamSynchronize(st));
    tr.mark("d2h");
  }
}

int bt_mat_get_block(const bt_mat* mh, int64_t i, int64_t j, double* out, int* found) {
  return guard([&] {
    check_mat(mh);
    const Mat& m = mh->impl;
    BT_REQUIRE(found, BT_ERR_INVALID_ARGUMENT, "null found flag");
    BT_REQUIRE(i >= 0 && i < m.nbr && j >= 0 && j < m.nbc, BT_ERR_INVALID_ARGUMENT,
               "get_block: index out of range");
    *found = 0;
    if (m.nblk == 0) return;
    cudaStream_t st = m.stream();
    int32_t rp[2];
    BT_CUDA(cudaMemcpyAsync(rp, m.row_ptr.p + i, sizeof(int32_t) * 2, cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaStreamSynchronize(st));
    if (rp[1] == rp[0]) return;
    std::vector<int32_t> cols(rp[1] - rp[0]);
    BT_CUDA(cudaMemcpyAsync(cols.data(), m.col.p + rp[0], sizeof(int32_t) * cols.size(),
                            cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaStreamSynchronize(st));
    auto it = std::lower_bound(cols.begin(), cols.end(), static_cast<int32_t>(j));
    if (it == cols.end() || *it != j) return;
    const int64_t e = rp[0] + (it - cols.begin());
    int64_t o;
    BT_CUDA(cudaMemcpyAsync(&o, m.off.p + e, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaStreamSynchronize(st));
    if (out) {
      const int R = m.h_rsz[i], Cc = m.h_csz[j];
      std::vector<double> slot(t8_size(R, Cc));
      BT_CUDA(cudaMemcpyAsync(slot.data(), m.vals.p + o, sizeof(double) * slot.size(),
                              cudaMemcpyDeviceToHost, st));
      BT_CUDA(cudaStreamSynchronize(st));
      for (int r = 0; r < R; ++r)
        for (int c = 0; c < Cc; ++c) out[int64_t(r) * Cc + c] = slot[t8_pos(r, c, tiles8(Cc))];
    }
    *found = 1;
  });
}

int bt_mat_norms(const bt_mat* mh, double* out) {
  return guard([&] {
    check_mat(mh);
    const Mat& m = mh->impl;
    BT_REQUIRE(out || m.nblk == 0, BT_ERR_INVALID_ARGUMENT, "null output");
    if (m.nblk == 0) return;
    cudaStream_t st = m.stream();
    const double* d = m.norms(st);
    BT_CUDA(cudaMemcpyAsync(out, d, sizeof(double) * m.nblk, cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaStreamSynchronize(st));
  });
}

int bt_filter(bt_mat* mh, double eps) { return bt_filter_report(mh, eps, 0.0, nullptr, nullptr); }

int bt_filter_report(bt_mat* mh, double eps, double band, int64_t* dropped,
                     int64_t* borderline) {
  return guard([&] {
    check_mat(mh);
    Mat& m = mh->impl;
    BT_REQUIRE(band >= 0, BT_ERR_INVALID_ARGUMENT, "filter: negative borderline band");
    if (dropped) *dropped = 0;
    if (borderline) *borderline = 0;
    if (m.nblk == 0 || !(eps > 0)) return;
    cudaStream_t st = m.stream();
    std::vector<double> nrm(m.nblk);
    BT_CUDA(cudaMemcpyAsync(nrm.data(), m.norms(st), sizeof(double) * m.nblk,
                            cudaMemcpyDeviceToHost, st));
    HostIndex h = download_index(m);
    std::vector<int32_t> row_ptr(m.nbr + 1, 0), col;
    std::vector<int64_t> off, src, len;
    int64_t nv = 0, ne = 0;
    int64_t n_drop = 0, n_border = 0;
    for (int64_t i = 0; i < m.nbr; ++i)
      for (int32_t e = h.row_ptr[i]; e < h.row_ptr[i + 1]; ++e) {
        // borderline: a ULP-level difference in the block's values could flip
        // the decision ("Filter semantics")
        if (std::fabs(nrm[e] - eps) <= band * eps) ++n_border;
        if (nrm[e] < eps) {
          ++n_drop;
          continue;
        }
        const int64_t L = int64_t(m.h_rsz[i]) * m.h_csz[h.col[e]];
        const int64_t T = t8_size(m.h_rsz[i], m.h_csz[h.col[e]]);
        col.push_back(h.col[e]);
        off.push_back(nv);
        src.push_back(h.off[e]);
        len.push_back(T);
        nv += T;
        ne += L;
        row_ptr[i + 1]++;
      }
    for (int64_t i = 0; i < m.nbr; ++i) row_ptr[i + 1] += row_ptr[i];
    const int64_t nout = static_cast<int64_t>(col.size());
    DBuf<double> nvals(std::max<int64_t>(nv, 2), st);
    if (nout) {
      auto d_off = upload(off, st);
      auto d_src = upload(src, st);
      auto d_len = upload(len, st);
      k_gather_blocks<<<static_cast<unsigned>((nout * 32 + 255) / 256), 256, 0, st>>>(
          nvals.p, d_off.p, m.vals.p, d_src.p, d_len.p, nout);
      check_launch("gather_blocks");
      count_launch(m.ctx);
    }
    m.vals = std::move(nvals);
    install_pattern(m, row_ptr, col, off, nv, ne);
    BT_CUDA(cudaStreamSynchronize(st));
    if (dropped) *dropped = n_drop;
    if (borderline) *borderline = n_border;
  });
}

}  // extern "C"
