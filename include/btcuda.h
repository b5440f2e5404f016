/*
 * btcuda.h -- C-ABI drop-in boundary of the B200-native block-sparse FP64
 * multiply (libbtcuda.so).  Plain pointers and sizes only; no torch or C++
 * types cross this line.
 *
 * Each entry point names the reference interface it replaces (paths relative
 * to /root/reference/proj/).  The reference is a header-only C++ library with no
 * FFI of its own (CMakeLists.txt:14-16); its "operator API" is the set of free
 * functions in matrix.hpp / multiply_cannon.hpp / multiply_rect.hpp.  The C++
 * facade include/blocktensor/b200.hpp re-exposes these with the reference's own
 * names and exception types; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - A bt_mat is one rank's LocalStore (matrix.hpp:137-275): a device-resident
 *    block-CSR tile with the matrix's full blockings and global block indices.
 *  - Block values are row-major m x n doubles (DenseBlock, block.hpp:19-41).
 *    Host value arrays are "compact": blocks concatenated in the listed order.
 *  - Host buffers are borrowed for the duration of the call only.  Calls are
 *    synchronous w.r.t. host buffers; device work is ordered on the context's
 *    stream.  All functions return BT_OK (0) or a BT_ERR_* code; the message is
 *    in bt_last_error() (thread-local).
 */
#ifndef BTCUDA_H
#define BTCUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes map 1:1 onto the reference exception classes (errors.hpp:14-53). */
#define BT_OK 0
#define BT_ERR_INVALID_ARGUMENT 1 /* blocktensor::invalid_argument  errors.hpp:20-23 */
#define BT_ERR_OWNERSHIP 2        /* blocktensor::ownership_error   errors.hpp:26-29 */
#define BT_ERR_GRID 3             /* blocktensor::grid_error        errors.hpp:32-35 */
#define BT_ERR_LAYOUT 4           /* blocktensor::layout_error      errors.hpp:39-47 */
#define BT_ERR_DEADLOCK 5         /* blocktensor::deadlock_error    errors.hpp:50-53 */
#define BT_ERR_CUDA 10            /* CUDA runtime failure (base blocktensor::error) */
#define BT_ERR_NCCL 11            /* NCCL failure */
#define BT_ERR_OOM 12             /* device allocation failed */
#define BT_ERR_INTERNAL 13

typedef struct bt_ctx bt_ctx;
typedef struct bt_mat bt_mat;

/* Per-call statistics of a multiply. */
typedef struct bt_stats {
  int64_t candidates;   /* block products A_ik*B_kj with both blocks stored */
  int64_t products;     /* products executed (candidates surviving the eps filter) */
  double flops;         /* useful flops: sum of 2*m*n*k over executed products */
  int64_t c_blocks_in;  /* C blocks before the call */
  int64_t c_blocks_out; /* C blocks after the call */
  int64_t elements_sent;     /* distributed calls: matrix elements sent by this rank */
  int64_t elements_received; /* (ledger units, comm.hpp:41-150) */
  int64_t meta_sent;         /* index words sent (4 per block, matrix.hpp:503-513) */
  int64_t meta_received;
  int32_t kernels; /* kernels launched by the call */
  int32_t reserved;
  /* with bt_ctx_set_timing(ctx, 1): CUDA-event device times of the call */
  double ms_numeric; /* the small-GEMM kernels (the dominant kernel family) */
  double ms_total;   /* the whole call, first to last kernel */
} bt_stats;

const char* bt_last_error(void);
int bt_version(void);

/* ---------------------------------------------------------------- context */
/* Replaces SimComm's construction (comm.hpp:166-175) for the device world:
 * one context per process drives one GPU.  nranks == 1 (nccl_id NULL) is the
 * single-GPU case.  For nranks > 1 every process passes the same 128-byte NCCL
 * unique id (bt_get_unique_id on rank 0, broadcast by the caller) and its rank. */
int bt_get_unique_id(void* id128);
int bt_ctx_create(int device, int nranks, int rank, const void* nccl_id, bt_ctx** out);
/* A subgroup context (SPEC.md tall_skinny subgroups): every process of the
 * parent's NCCL group calls it; processes with the same color form one
 * subgroup (ranks ordered by key) with its own communicator -- ncclCommSplit.
 * A one-rank subgroup is a single-GPU context.  The parent must have nranks > 1. */
int bt_ctx_split(bt_ctx* parent, int color, int key, bt_ctx** out);
int bt_ctx_destroy(bt_ctx* ctx);
/* waits for all device work of the context (incl. asynchronous exports) */
int bt_ctx_sync(bt_ctx* ctx);
int bt_ctx_rank(const bt_ctx* ctx, int* rank, int* nranks);
/* the context's CUDA stream (cudaStream_t), for callers that time with events */
int bt_ctx_stream(bt_ctx* ctx, void** stream);
/* number of kernels this context has launched so far */
int bt_ctx_kernel_count(const bt_ctx* ctx, int64_t* count);
/* 0: off.  1: multiplies record CUDA events around their kernels and report
 * device times in bt_stats (the call waits for its kernels).  2: events only;
 * bt_multiply returns without waiting and bt_ctx_last_timing reads the times
 * of the last multiply (waiting for it).  bt_multiply never waits for its
 * numeric phase otherwise: results are stream-ordered, every later call on
 * the context (export, get_block, ...) sees the finished C. */
int bt_ctx_set_timing(bt_ctx* ctx, int on);
int bt_ctx_last_timing(bt_ctx* ctx, double* ms_numeric, double* ms_total);

/* ----------------------------------------------------------------- matrix */
/* new_matrix (matrix.hpp:404-418) for one rank's store: blockings only; the
 * distribution lives with the caller (facade DistMatrix). */
int bt_mat_create(bt_ctx* ctx, int64_t nbr, const int32_t* row_sizes, int64_t nbc,
                  const int32_t* col_sizes, bt_mat** out);
int bt_mat_destroy(bt_mat* m);
/* LocalStore::clear (matrix.hpp:247-252) */
int bt_mat_clear(bt_mat* m);
/* deep copy of the stored blocks of src into dst (same blockings) */
int bt_mat_copy(const bt_mat* src, bt_mat* dst);
/* DistMatrix::put_block / LocalStore::insert (matrix.hpp:167-189, 305-309), batched:
 * n blocks (bi[t], bj[t]) with compact values in listed order.  accumulate = 0
 * replaces an existing block (later entries of the batch win), 1 adds into it.
 * vals may be host memory (pinned or pageable) or memory of the context's GPU
 * (used in place, no staging copy). */
int bt_mat_put_blocks(bt_mat* m, int64_t n, const int64_t* bi, const int64_t* bj,
                      const double* vals, int accumulate);
/* number of stored blocks and of stored elements (LocalStore::stored_elements) */
int bt_mat_info(const bt_mat* m, int64_t* nblk, int64_t* nelems);
/* Canonical (i, j)-sorted export of all stored blocks into host buffers of
 * nblk / nelems entries (bi, bj may be NULL to skip the index). */
int bt_mat_export(const bt_mat* m, int64_t* bi, int64_t* bj, double* vals);
/* bt_mat_export whose value transfer completes asynchronously: returns once
 * bi/bj are filled and the D2H of the values into `vals` is enqueued on a side
 * stream (the context's main stream stays free, so the next call's uploads and
 * kernels overlap the transfer).  `vals` must stay valid, and must not be read,
 * until bt_ctx_sync(ctx) returns.  Pinned `vals` give full PCIe speed. */
int bt_mat_export_async(const bt_mat* m, int64_t* bi, int64_t* bj, double* vals);
/* DistMatrix::get_block (matrix.hpp:323-325): copies block (i, j) into out
 * (rows*cols doubles); *found = 0 when it is not stored. */
int bt_mat_get_block(const bt_mat* m, int64_t i, int64_t j, double* out, int* found);
/* Frobenius norms of the stored blocks in canonical order (sequential sum of
 * squares, unfused: bit-identical to the oracle's). */
int bt_mat_norms(const bt_mat* m, double* out);

/* --------------------------------------------------------------- multiply */
/* Local batched multiply C += A*B: the device equivalent of
 * detail::multiply_tiles_into (multiply_cannon.hpp:24-44) with order_batches
 * (block.hpp:112-118) and get_or_create (matrix.hpp:191-196) -- C's pattern
 * grows to C_in U {(i,j): some product survives}.  eps > 0 skips products with
 * ||A_ik||_F * ||B_kj||_F < eps (filter; the reference fixes
 * eps = 0).  A and B are const.  stats may be NULL. */
int bt_multiply(bt_ctx* ctx, const bt_mat* a, const bt_mat* b, bt_mat* c, double eps,
                bt_stats* stats);

/* Post-filter: drops C blocks with ||C_ij||_F < eps. */
int bt_filter(bt_mat* m, double eps);
/* bt_filter that also reports: *dropped = blocks removed, *borderline = blocks
 * with | ||C_ij||_F - eps | <= band * eps, whose keep/drop decision could flip
 * under ULP-level value differences (e.g. band = 1e-12).
 * dropped / borderline may be NULL. */
int bt_filter_report(bt_mat* m, double eps, double band, int64_t* dropped, int64_t* borderline);

/* ------------------------------------------------------ distributed layer */
typedef struct bt_grid bt_grid; /* process group + ledger: SimComm (comm.hpp:152-397) */
typedef struct bt_dmat bt_dmat; /* DistMatrix (matrix.hpp:279-401) */

/* A group of nranks ranks.  With a single-rank context all ranks are local
 * "virtual ranks" on the context's GPU (messages are device copies): the
 * reference's one-process SimComm.  With an NCCL context (bt_ctx_create with
 * nranks > 1) the group is the NCCL world and this process owns rank ctx.rank. */
int bt_grid_create(bt_ctx* ctx, int nranks, bt_grid** out);
int bt_grid_destroy(bt_grid* g);
int bt_grid_info(const bt_grid* g, int* nranks, int* first_local, int* nlocal);
/* Ledger (comm.hpp:60-150): what = 0 elements sent, 1 elements received,
 * 2 meta sent, 3 meta received; phase NULL/"" = rank total. */
int bt_grid_ledger(const bt_grid* g, int rank, const char* phase, int what, int64_t* out);
int bt_grid_reset_ledger(bt_grid* g);
/* Sum of n int64 values over the processes of the group (every process passes
 * its local partial; all receive the total).  A no-op for virtual ranks (one
 * process holds every rank).  Used for global counts such as the stored
 * elements behind measured_spec (multiply_rect.hpp:254-265) in NCCL mode. */
int bt_grid_sum(bt_grid* g, int64_t* values, int n);

/* new_matrix (matrix.hpp:404-410): blockings + ProcessGrid dims + Axis
 * distributions; NULL distributions = round robin (new_matrix_round_robin,
 * matrix.hpp:413-418). */
int bt_dmat_create(bt_grid* g, int64_t nbr, const int32_t* row_sizes, int64_t nbc,
                   const int32_t* col_sizes, int grid_rows, int grid_cols,
                   const int32_t* row_dist, const int32_t* col_dist, bt_dmat** out);
int bt_dmat_destroy(bt_dmat* d);
/* the store of a local rank (DistMatrix::local, matrix.hpp:294-295); borrowed */
int bt_dmat_local(bt_dmat* d, int rank, bt_mat** store);
/* DistMatrix::owner_rank (matrix.hpp:297-299) */
int bt_dmat_owner(const bt_dmat* d, int64_t i, int64_t j, int* rank);
/* put_block routed to the owner (matrix.hpp:305-309); BT_ERR_OWNERSHIP when the
 * owner is a rank of another process */
int bt_dmat_put_blocks(bt_dmat* d, int64_t n, const int64_t* bi, const int64_t* bj,
                       const double* vals, int accumulate);
/* redistribute / redistribute_add (matrix.hpp:567-622) onto dst's layout */
int bt_redistribute(const bt_dmat* src, bt_dmat* dst, int transpose, int accumulate,
                    const char* phase);
/* multiply_cannon (multiply_cannon.hpp:62-118) */
int bt_multiply_cannon(const bt_dmat* a, const bt_dmat* b, bt_dmat* c, double eps,
                       bt_stats* stats);
/* multiply_reduce_case1 (multiply_rect.hpp:123-192) */
int bt_multiply_case1(const bt_dmat* a, const bt_dmat* b, bt_dmat* c, int nprocs, double eps,
                      bt_stats* stats);
/* multiply_virtual_case2 (multiply_rect.hpp:199-238); gather = 1 gathers all B
 * slabs in one NVLink step instead of the P-step ring */
int bt_multiply_case2(const bt_dmat* a, const bt_dmat* b, bt_dmat* c, int nprocs, int gather,
                      double eps, bt_stats* stats);

/* ------------------------------------------------------------ tensors */
/* Tensor <-> matrix index remap (the reference has no tensor
 * code).  A rank-ndim (2..4) block-sparse tensor with nblocks[d] blocks of sizes
 * dim_sizes[d][...] along dimension d is stored as a matrix under a
 * matricization map: dims[0..nrow) form the row group, dims[nrow..ndim) the
 * column group, mixed radix with later-listed dimensions fastest, for block
 * indices and for the elements inside a block.  Moves `src` (stored under the
 * src map) into `dst` (blockings induced by the dst map), on the device. */
int bt_tensor_remap(bt_ctx* ctx, int ndim, const int64_t* nblocks,
                    const int32_t* const* dim_sizes, int src_nrow, const int* src_dims,
                    const bt_mat* src, int dst_nrow, const int* dst_dims, bt_mat* dst);

#ifdef __cplusplus
}
#endif
#endif /* BTCUDA_H */
