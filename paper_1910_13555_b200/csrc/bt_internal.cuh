// bt_internal.cuh -- shared internals of libbtcuda (device BCSR store, context,
// error plumbing).  See DESIGN.md section 2 for the HBM layout.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <functional>
#include <vector>

#include "btcuda.h"

namespace bt {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

void set_last_error(const std::string& msg);

#define BT_CUDA(x)                                                                         \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw ::bt::Error(e_ == cudaErrorMemoryAllocation ? BT_ERR_OOM : BT_ERR_CUDA,        \
                        std::string("CUDA error ") + cudaGetErrorString(e_) + " at " +     \
                            __FILE__ + ":" + std::to_string(__LINE__));                    \
  } while (0)

#define BT_REQUIRE(cond, code, msg) \
  do {                              \
    if (!(cond)) throw ::bt::Error((code), (msg)); \
  } while (0)

// Device-side invariant checks, compiled in only for the checked build
// (make checked -> libbtcuda_checked.so, -DBT_DEVICE_CHECKS): out-of-range slab
// offsets, descriptor / work-item indices and a bounded spin on the K-panel
// flags trap with a message.  This pool has compute-sanitizer closed, so the
// parity suite run against the checked build is the bounds / race evidence.
#ifdef BT_DEVICE_CHECKS
#define BT_DASSERT(cond, what)                                                         \
  do {                                                                                 \
    if (!(cond)) {                                                                     \
      printf("BT_DASSERT failed: %s (%s:%d) block %d thread %d\n", what, __FILE__,      \
             __LINE__, static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));   \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define BT_DASSERT(cond, what) \
  do {                         \
  } while (0)
#endif

// wraps a C-ABI body: converts exceptions to status codes + bt_last_error()
template <class F>
int guard(F&& f) {
  try {
    f();
    return BT_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return BT_ERR_OOM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return BT_ERR_INTERNAL;
  }
}

// ------------------------------------------------------------------ memory
// Stream-ordered device buffer from the device's default mempool (release
// threshold raised at context creation, so steady-state multiplies never hit
// cudaMalloc).
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t st) { alloc(count, st); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count) BT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), st));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
};

// ----------------------------------------------------------------- context
struct Ctx {
  int device = 0;
  int nranks = 1;
  int rank = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  size_t smem_optin = 227 * 1024;
  int64_t kernels = 0;  // kernels launched through this context
  void* nccl = nullptr; // ncclComm_t when nranks > 1
  // a second communicator of the same ranks (ncclCommSplit, made by the first
  // case-2 gather): the B value all-gather runs on it beside the index gather
  void* nccl_vals = nullptr;
  DBuf<unsigned char> scratch;  // CUB temp storage, reused
  // small mapped page-locked staging for scalar readbacks; layout (bytes):
  //   [0, 1200)      the multiply's sizes block / the export's chunk offsets
  //   [512, 3072)    exchange headers (bt_dist.cu, word 64 on; used between
  //                  multiplies, never while a sizes block is pending)
  //   [3072, ...)    the B-gather size headers (word 384 on, 8 + 3P words)
  //   [kPinnedFlag]  the multiply's sizes-ready flag (last 64 bytes)
  static constexpr size_t kPinnedBytes = 8192, kPinnedFlag = kPinnedBytes - 64;
  void* pinned = nullptr;
  // device alias of `pinned` (mapped page-locked memory): kernels write small
  // results there directly, so reading them back needs no copy-engine D2H --
  // which would queue behind an asynchronous export's bulk transfer
  void* pinned_dev = nullptr;
  unsigned long long size_seq = 0;  // sequence of the multiply's sizes flag (kPinnedFlag)
  // Grow-only pinned host staging for index uploads: one packed H2D per call
  // instead of several pageable copies.  stage_ev marks the last copy that read
  // it; host_stage() waits for it before handing the buffer out again.
  unsigned char* hstage = nullptr;
  unsigned char* hstage_dev = nullptr;  // device alias of hstage (mapped)
  size_t hstage_cap = 0;
  cudaEvent_t stage_ev = nullptr;
  unsigned char* host_stage(size_t bytes);
  // 0: off; 1: CUDA events around the multiply kernels, the call waits for
  // them and fills bt_stats; 2: events only, read later with
  // bt_ctx_last_timing (the call does not wait)
  int timing = 0;
  bool last_had_numeric = false;  // the last multiply launched a numeric phase
  static constexpr int kAux = 16;  // side streams: concurrent per-class numeric kernels
  cudaStream_t aux[kAux] = {};
  cudaEvent_t ev_fork = nullptr;
  cudaEvent_t ev_join[kAux] = {};
  cudaEvent_t ev[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  // Export staging (T8 -> compact values, then D2H on aux[0]): two buffers
  // used alternately; xfer_done[b] marks the last D2H that read buffer b, so a
  // later export compacts into b only after it (asynchronous exports,
  // bt_mat_export_async, leave the main stream free meanwhile).
  DBuf<double> xstage[2];
  cudaStream_t xfer = nullptr;  // the export's D2H stream (not shared with kernels)
  cudaEvent_t xfer_done[2] = {nullptr, nullptr};
  int xnext = 0;
  // waits for every stream of the context (main + side streams)
  void sync_all();
  void* ensure_scratch(size_t bytes);
  // Grow-only per-slot workspace for call-local temporaries (no allocator calls
  // in steady state).  Valid until the next use of the same slot.
  DBuf<unsigned char> ws_slots[28];
  template <class T>
  T* ws(int slot, size_t count) {
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    if (ws_slots[slot].n < bytes) ws_slots[slot].alloc(bytes + bytes / 4, stream);
    return reinterpret_cast<T*>(ws_slots[slot].p);
  }
};

// ------------------------------------------------------------------- store
// One rank's block-CSR store, device resident:
//   row_ptr[nbr+1] int32 over ALL block rows (dense row pointer),
//   col[nblk]      int32 global block column, strictly increasing per row,
//   off[nblk]      int64 offset (in doubles, a multiple of 64) of the block in vals,
//   vals           FP64 slab of blocks in the "T8" layout: each m x n block is
//                  zero-padded to ceil8(m) x ceil8(n) and stored as row-major 8x8
//                  tiles of 64 doubles (512 B), element (r, c) of a tile at
//                  r*8 + (c ^ 4*((r>>1)&1)).  The swizzle makes DMMA A-role
//                  (8x4) and B-role (4x8) fragment reads and the C fragment
//                  16-byte stores bank-conflict free; tile rows are contiguous,
//                  so a 32-row slab of a tall block is one bulk copy.
struct Mat {
  Ctx* ctx = nullptr;
  int64_t nbr = 0, nbc = 0;
  std::vector<int32_t> h_rsz, h_csz;
  DBuf<int32_t> rsz, csz;
  int32_t max_r = 0, max_c = 0;
  bool uniform_r = true, uniform_c = true;
  int64_t nblk = 0;
  int64_t nelems = 0;  // stored (unpadded) elements
  int64_t nvals = 0;   // padded slab length
  DBuf<int32_t> row_ptr;
  DBuf<int32_t> col;
  DBuf<int64_t> off;
  DBuf<double> vals;
  // Block Frobenius norms in storage order (eps filter), computed
  // on first use and kept with the data: every site that changes the pattern
  // or the values assigns nblk and clears norms_ok right after.
  mutable DBuf<double> norm_cache;
  mutable bool norms_ok = false;
  // device pointer to this store's block norms (computed on `st` when stale)
  const double* norms(cudaStream_t st) const;
  cudaStream_t stream() const { return ctx->stream; }
  void init_empty();  // empty pattern (row_ptr all zero)
  // empty pattern, keeping col/off/vals allocated as capacity for the next
  // multiply into this store (bt_mat_clear)
  void clear_keep_capacity();
};

__host__ __device__ inline int64_t pad2(int64_t x) { return (x + 1) & ~int64_t(1); }

// ---- T8 block layout helpers
__host__ __device__ inline int tiles8(int x) { return (x + 7) >> 3; }
// doubles occupied by an m x n block
__host__ __device__ inline int64_t t8_size(int m, int n) {
  return static_cast<int64_t>(tiles8(m)) * tiles8(n) * 64;
}
// position of element (r, c) inside a T8 block with `ntc` tile columns
__host__ __device__ inline int64_t t8_pos(int r, int c, int ntc) {
  return ((static_cast<int64_t>(r >> 3) * ntc + (c >> 3)) << 6) + ((r & 7) << 3) +
         ((c & 7) ^ (((r >> 1) & 1) << 2));
}

// BT_TRACE=1: host-side phase timings on stderr (development aid)
struct Trace {
  const char* what;
  bool on;
  double t0, last;
  static double now();
  explicit Trace(const char* w);
  void mark(const char* phase);
  ~Trace();
};

// launch accounting
inline void count_launch(Ctx* c, int n = 1) { c->kernels += n; }

// implemented in bt_store.cu (one warp per block)
constexpr int kNormThreads = 256;
__global__ void k_block_norms(const double* vals, const int32_t* row_ptr, const int32_t* col,
                              const int64_t* off, const int32_t* rsz, const int32_t* csz,
                              int64_t nbr, double* out, int64_t nblk);
// the norms of two stores (A and B of a filtered multiply) in one launch:
// warps [0, a.nblk) take A's blocks, the rest B's
struct NormSrc {
  const double* vals;
  const int32_t *row_ptr, *col;
  const int64_t* off;
  const int32_t *rsz, *csz;
  int64_t nbr;
  double* out;
  int64_t nblk;
};
__global__ void k_block_norms_pair(NormSrc a, NormSrc b);
void upload_sizes(Mat& m);
void check_launch(const char* what);
// integer environment knob (development / experiments), default when unset
int env_int(const char* name, int dflt);
// Device-usable alias of a host pointer when it is page-locked and mapped
// (cudaHostAlloc / cudaHostRegister under UVA), else nullptr.  Kernels read or
// write such buffers directly over PCIe (no staging copy).
void* mapped_host_alias(const void* p);
// Packs `n` host arrays into the pinned stage (one host pass) and enqueues
// their H2D copies to dst[t] on the context stream (no pageable copies).
struct HostPart {
  const void* src;
  size_t bytes;
};
void upload_parts(Ctx& x, const HostPart* parts, int n, void* const* dst);
// implemented in bt_multiply.cu: C += A*B on one rank's stores (throws bt::Error)
// wait_numeric (optional): the numeric phase waits for this event (B's values
// may still be in flight while the symbolic passes run).
// sync_at_end: wait for the numeric phase before returning (the distributed
// drivers rely on it); the single-GPU C-ABI call returns right after enqueuing
// (stream-ordered: every later call on the context sees the finished C).
// poll_sizes: wait for the pass-1 sizes by polling a mapped flag instead of a
// stream synchronize -- single-GPU calls only: next to in-flight NCCL
// transfers (Cannon shifts) the spinning host thread cost 1 s of a 1.4 s c5
// Cannon multiply on 4 GPUs (profiles/r02/README.md).
void local_multiply(Ctx& x, const Mat& A, const Mat& B, Mat& C, double eps, bt_stats* stats,
                    cudaEvent_t wait_numeric = nullptr, cudaEvent_t numeric_start = nullptr,
                    const std::function<void()>* after_sizes = nullptr, bool sync_at_end = true,
                    bool poll_sizes = false);

}  // namespace bt

struct bt_ctx {
  bt::Ctx impl;
};
struct bt_mat {
  bt::Mat impl;
};
