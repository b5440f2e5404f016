// blocktensor/b200.hpp -- C++ facade with the reference's names and signatures
// (namespace blocktensor) over the C-ABI in btcuda.h, so caller code written
// against /root/reference/proj/include/blocktensor compiles unchanged for the
// multiply path:
//
//   errors.hpp:14-53      error, invalid_argument, ownership_error, grid_error,
//                         layout_error, deadlock_error   (status codes -> exceptions)
//   block.hpp:19-97       DenseBlock, Blocking
//   grid.hpp:17-69        ProcessGrid
//   comm.hpp:152-397      SimComm (+ Ledger, TrafficCounters): the device group --
//                         every rank of the grid is a virtual rank on this
//                         process's GPU, or (SimComm(grid, device, rank, NcclId))
//                         one rank per process over NCCL
//   matrix.hpp:26-418     Axis (explicit and functional), LocalStore (a view),
//                         DistMatrix (+ local, put_block_at, get_block_at,
//                         for_each_global), new_matrix, new_matrix_round_robin,
//                         redistribute, redistribute_add
//   io.hpp:22-198         FileFormat, MatrixData, read/write_matrix_{text,binary},
//                         to_dist_matrix, read_matrix_file, write_matrix_file
//   multiply_cannon.hpp   multiply_cannon
//   (SPEC tensor module) SparseTensor, contract, mixed_radix
//   multiply_rect.hpp     Algorithm, multiply_reduce_case1, multiply_virtual_case2,
//                         multiply_dispatch, select_algorithm, measured_spec
//   cost_model.hpp        MultiplySpec + Eq. 1-5
//
// Differences a caller can see: DistMatrix is created on the
// most recently constructed SimComm (the reference's matrices are plain host
// objects); get_block returns a pointer to a host copy that stays valid until
// the next get_block on the same matrix; filter() and the eps argument of the
// multiplies are extensions (the reference fixes eps = 0).
// Link with -lbtcuda (paper_1910_13555_b200/libbtcuda.so).
#pragma once

#include <algorithm>
#include <cmath>
#include <limits>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <istream>
#include <map>
#include <ostream>
#include <sstream>
#include <charconv>
#include <tuple>
#include <unistd.h>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../btcuda.h"

namespace blocktensor {

// ------------------------------------------------------------------ errors
class error : public std::runtime_error {
 public:
  explicit error(const std::string& what) : std::runtime_error(what) {}
};
class invalid_argument : public error {
 public:
  using error::error;
};
class ownership_error : public error {
 public:
  using error::error;
};
class grid_error : public error {
 public:
  using error::error;
};
class layout_error : public error {
 public:
  layout_error(std::string dimension, const std::string& what)
      : error(what), dimension_(std::move(dimension)) {}
  const std::string& dimension() const noexcept { return dimension_; }

 private:
  std::string dimension_;
};
class deadlock_error : public error {
 public:
  using error::error;
};

namespace detail {
inline void check(int rc) {
  if (rc == BT_OK) return;
  const std::string msg = bt_last_error();
  switch (rc) {
    case BT_ERR_INVALID_ARGUMENT: throw invalid_argument(msg);
    case BT_ERR_OWNERSHIP: throw ownership_error(msg);
    case BT_ERR_GRID: throw grid_error(msg);
    case BT_ERR_LAYOUT: throw layout_error("", msg);
    case BT_ERR_DEADLOCK: throw deadlock_error(msg);
    default: throw error(msg);
  }
}
}  // namespace detail

// ------------------------------------------------------------------ blocks
struct DenseBlock {
  int rows = 0;
  int cols = 0;
  std::vector<double> values;  // row-major
  DenseBlock() = default;
  DenseBlock(int m, int n) : rows(m), cols(n), values(static_cast<std::size_t>(m) * n, 0.0) {
    if (m < 1 || n < 1) throw invalid_argument("DenseBlock: dimensions must be positive");
  }
  DenseBlock(int m, int n, std::vector<double> v) : rows(m), cols(n), values(std::move(v)) {
    if (m < 1 || n < 1) throw invalid_argument("DenseBlock: dimensions must be positive");
    if (values.size() != static_cast<std::size_t>(m) * n)
      throw invalid_argument("DenseBlock: value count does not match dimensions");
  }
  double& at(int i, int j) { return values[static_cast<std::size_t>(i) * cols + j]; }
  double at(int i, int j) const { return values[static_cast<std::size_t>(i) * cols + j]; }
  std::int64_t size() const noexcept { return static_cast<std::int64_t>(rows) * cols; }
  friend bool operator==(const DenseBlock& a, const DenseBlock& b) {
    return a.rows == b.rows && a.cols == b.cols && a.values == b.values;
  }
};

class Blocking {
 public:
  Blocking() = default;
  explicit Blocking(std::vector<int> sizes) : sizes_(std::move(sizes)), offsets_(sizes_.size() + 1, 0) {
    for (std::size_t i = 0; i < sizes_.size(); ++i) {
      if (sizes_[i] < 1) throw invalid_argument("Blocking: block sizes must be positive");
      offsets_[i + 1] = offsets_[i] + sizes_[i];
    }
  }
  static Blocking uniform(std::int64_t n_blocks, int block_size) {
    return Blocking(std::vector<int>(static_cast<std::size_t>(n_blocks), block_size));
  }
  std::int64_t n_blocks() const noexcept { return static_cast<std::int64_t>(sizes_.size()); }
  int size(std::int64_t b) const { return sizes_.at(static_cast<std::size_t>(b)); }
  std::int64_t offset(std::int64_t b) const { return offsets_.at(static_cast<std::size_t>(b)); }
  std::int64_t total() const noexcept { return offsets_.empty() ? 0 : offsets_.back(); }
  const std::vector<int>& sizes() const noexcept { return sizes_; }
  friend bool operator==(const Blocking& a, const Blocking& b) { return a.sizes_ == b.sizes_; }

 private:
  std::vector<int> sizes_;
  std::vector<std::int64_t> offsets_;
};

// -------------------------------------------------------------------- grid
class ProcessGrid {
 public:
  ProcessGrid() : dims_{1}, size_(1) {}
  explicit ProcessGrid(std::vector<int> dims) : dims_(std::move(dims)), size_(1) {
    if (dims_.empty()) throw invalid_argument("ProcessGrid: dims must be non-empty");
    for (int d : dims_) {
      if (d < 1) throw invalid_argument("ProcessGrid: every grid extent must be >= 1");
      size_ *= d;
    }
  }
  int ndims() const noexcept { return static_cast<int>(dims_.size()); }
  int dim(int i) const { return dims_.at(static_cast<std::size_t>(i)); }
  const std::vector<int>& dims() const noexcept { return dims_; }
  int size() const noexcept { return size_; }
  std::vector<int> coords_of(int rank) const {
    if (rank < 0 || rank >= size_) throw invalid_argument("coords_of: rank out of range");
    std::vector<int> c(dims_.size());
    for (int d = ndims() - 1; d >= 0; --d) {
      c[static_cast<std::size_t>(d)] = rank % dims_[static_cast<std::size_t>(d)];
      rank /= dims_[static_cast<std::size_t>(d)];
    }
    return c;
  }
  int rank_of(const std::vector<int>& c) const {
    if (c.size() != dims_.size()) throw invalid_argument("rank_of: coordinate count mismatch");
    int r = 0;
    for (std::size_t d = 0; d < dims_.size(); ++d) {
      if (c[d] < 0 || c[d] >= dims_[d]) throw invalid_argument("rank_of: coordinate out of range");
      r = r * dims_[d] + c[d];
    }
    return r;
  }
  friend bool operator==(const ProcessGrid& a, const ProcessGrid& b) { return a.dims_ == b.dims_; }
  friend bool operator!=(const ProcessGrid& a, const ProcessGrid& b) { return !(a == b); }

 private:
  std::vector<int> dims_;
  int size_;
};

// ------------------------------------------------------------- comm/ledger
enum class Schedule { parallel, sequential };

struct TrafficCounters {
  std::int64_t elements_sent = 0;
  std::int64_t elements_received = 0;
  std::int64_t meta_sent = 0;
  std::int64_t meta_received = 0;
};

class Ledger {
 public:
  explicit Ledger(const bt_grid* g, int n) : g_(g), n_(n) {}
  int nranks() const noexcept { return n_; }
  TrafficCounters rank_total(int rank) const { return read(rank, nullptr); }
  TrafficCounters rank_phase(int rank, const std::string& phase) const {
    return read(rank, phase.c_str());
  }
  std::int64_t total_elements_sent() const {
    std::int64_t s = 0;
    for (int r = 0; r < n_; ++r) s += rank_total(r).elements_sent;
    return s;
  }
  double mean_elements_sent() const { return n_ ? double(total_elements_sent()) / n_ : 0.0; }
  std::int64_t max_elements_sent() const {
    std::int64_t m = 0;
    for (int r = 0; r < n_; ++r) m = std::max(m, rank_total(r).elements_sent);
    return m;
  }

 private:
  TrafficCounters read(int rank, const char* phase) const {
    std::int64_t v[4];
    for (int w = 0; w < 4; ++w) detail::check(bt_grid_ledger(g_, rank, phase, w, &v[w]));
    return TrafficCounters{v[0], v[1], v[2], v[3]};
  }
  const bt_grid* g_;
  int n_;
};

class DistMatrix;

// NCCL unique id of a one-process-per-GPU group (128 bytes, created by rank 0
// and handed to every rank by the caller: a file, MPI, torch.distributed ...)
struct NcclId {
  unsigned char bytes[128] = {};
  static NcclId create() {
    NcclId id;
    detail::check(bt_get_unique_id(id.bytes));
    return id;
  }
};

// The device group (comm.hpp:152-397).
//  * SimComm(grid): every rank of `grid` is a virtual rank on one GPU of this
//    process -- the reference's one-process SimComm, messages are device copies.
//  * SimComm(grid, device, rank, id): one rank per process over NCCL (NVLink /
//    NVSwitch); this process owns rank `rank` of grid.size() ranks on `device`.
// Both keep the reference's Ledger (comm.hpp:60-150) of the local ranks.
class SimComm {
 public:
  explicit SimComm(ProcessGrid grid, Schedule = Schedule::parallel, int device = 0)
      : grid_(std::move(grid)) {
    detail::check(bt_ctx_create(device, 1, 0, nullptr, &ctx_));
    detail::check(bt_grid_create(ctx_, grid_.size(), &g_));
    current() = this;
  }
  SimComm(ProcessGrid grid, int device, int rank, const NcclId& id) : grid_(std::move(grid)) {
    detail::check(bt_ctx_create(device, grid_.size(), rank, id.bytes, &ctx_));
    detail::check(bt_grid_create(ctx_, grid_.size(), &g_));
    current() = this;
  }
  // a group over an existing context (a subgroup from bt_ctx_split); owns it
  SimComm(ProcessGrid grid, bt_ctx* ctx) : grid_(std::move(grid)), ctx_(ctx) {
    detail::check(bt_grid_create(ctx_, grid_.size(), &g_));
    current() = this;
  }
  // this process's ranks: all of them (virtual ranks) or its own (NCCL)
  std::vector<int> local_ranks() const {
    int n = 0, first = 0, nl = 0;
    detail::check(bt_grid_info(g_, &n, &first, &nl));
    std::vector<int> r;
    for (int t = 0; t < nl; ++t) r.push_back(first + t);
    return r;
  }
  bool is_local(int rank) const {
    int n = 0, first = 0, nl = 0;
    detail::check(bt_grid_info(g_, &n, &first, &nl));
    return rank >= first && rank < first + nl;
  }
  // waits for all device work of this process (incl. asynchronous exports)
  void sync() const { detail::check(bt_ctx_sync(ctx_)); }
  SimComm(const SimComm&) = delete;
  SimComm& operator=(const SimComm&) = delete;
  ~SimComm() {
    if (current() == this) current() = nullptr;
    bt_grid_destroy(g_);
    bt_ctx_destroy(ctx_);
  }
  const ProcessGrid& grid() const noexcept { return grid_; }
  int nranks() const noexcept { return grid_.size(); }
  Ledger ledger() const { return Ledger(g_, grid_.size()); }
  void reset_ledger() { detail::check(bt_grid_reset_ledger(g_)); }
  bt_grid* handle() const noexcept { return g_; }
  bt_ctx* context() const noexcept { return ctx_; }
  static SimComm*& current() {
    static thread_local SimComm* c = nullptr;
    return c;
  }

 private:
  ProcessGrid grid_;
  bt_ctx* ctx_ = nullptr;
  bt_grid* g_ = nullptr;
};

// ------------------------------------------------------------------ matrix
// Axis (matrix.hpp:26-130): block sizes and grid coordinates of one matrix
// dimension, explicit arrays or functions (Axis::functional keeps no O(N)
// arrays on the host; the device store holds the sizes it needs).
class Axis {
 public:
  Axis() = default;
  Axis(const Blocking& b, std::vector<int> dist, int extent)
      : n_blocks_(b.n_blocks()), extent_(extent), blocking_(b), dist_(std::move(dist)) {
    if (static_cast<std::int64_t>(dist_.size()) != b.n_blocks())
      throw invalid_argument("Axis: distribution length does not match block count");
    for (int c : dist_)
      if (c < 0 || c >= extent_) throw invalid_argument("Axis: distribution coordinate out of grid range");
  }
  static Axis round_robin(const Blocking& b, int extent) {
    std::vector<int> d(static_cast<std::size_t>(b.n_blocks()));
    for (std::size_t i = 0; i < d.size(); ++i) d[i] = static_cast<int>(i % extent);
    return Axis(b, std::move(d), extent);
  }
  static Axis functional(std::int64_t n_blocks, std::function<int(std::int64_t)> size_fn,
                         std::function<int(std::int64_t)> dist_fn, int extent) {
    if (n_blocks < 0 || extent < 1) throw invalid_argument("Axis: bad functional axis");
    Axis a;
    a.n_blocks_ = n_blocks;
    a.extent_ = extent;
    a.size_fn_ = std::move(size_fn);
    a.dist_fn_ = std::move(dist_fn);
    return a;
  }
  bool is_explicit() const noexcept { return !size_fn_; }
  std::int64_t n_blocks() const noexcept { return n_blocks_; }
  int extent() const noexcept { return extent_; }
  int size(std::int64_t b) const {
    check_block(b);
    return is_explicit() ? blocking_.size(b) : size_fn_(b);
  }
  int dist(std::int64_t b) const {
    check_block(b);
    const int c = is_explicit() ? dist_[static_cast<std::size_t>(b)] : dist_fn_(b);
    if (c < 0 || c >= extent_) throw invalid_argument("Axis: distribution coordinate out of grid range");
    return c;
  }
  std::int64_t total_elements() const {
    if (is_explicit()) return blocking_.total();
    std::int64_t t = 0;
    for (std::int64_t b = 0; b < n_blocks_; ++b) t += size_fn_(b);
    return t;
  }
  // host index entries this axis keeps resident (0 for a functional axis)
  std::int64_t index_entries() const noexcept {
    return is_explicit() ? 2 * n_blocks_ : 0;
  }
  // the blocking (materialized on demand for a functional axis)
  Blocking blocking() const {
    if (is_explicit()) return blocking_;
    std::vector<int> v(static_cast<std::size_t>(n_blocks_));
    for (std::int64_t b = 0; b < n_blocks_; ++b) v[static_cast<std::size_t>(b)] = size_fn_(b);
    return Blocking(std::move(v));
  }
  std::vector<int> dists() const {
    if (is_explicit()) return dist_;
    std::vector<int> v(static_cast<std::size_t>(n_blocks_));
    for (std::int64_t b = 0; b < n_blocks_; ++b) v[static_cast<std::size_t>(b)] = dist(b);
    return v;
  }
  bool same_blocking(const Axis& o) const {
    if (n_blocks_ != o.n_blocks_) return false;
    for (std::int64_t b = 0; b < n_blocks_; ++b)
      if (size(b) != o.size(b)) return false;
    return true;
  }
  bool same_distribution(const Axis& o) const {
    if (n_blocks_ != o.n_blocks_ || extent_ != o.extent_) return false;
    for (std::int64_t b = 0; b < n_blocks_; ++b)
      if (dist(b) != o.dist(b)) return false;
    return true;
  }

 private:
  void check_block(std::int64_t b) const {
    if (b < 0 || b >= n_blocks_) throw invalid_argument("Axis: block index out of range");
  }
  std::int64_t n_blocks_ = 0;
  int extent_ = 1;
  Blocking blocking_;
  std::vector<int> dist_;
  std::function<int(std::int64_t)> size_fn_, dist_fn_;
};

// One rank's store (LocalStore, matrix.hpp:137-275), a view onto the device
// store: the visitors copy the blocks to the host once per call, in (row, col)
// order, as DenseBlocks.
class LocalStore {
 public:
  LocalStore(bt_mat* s, const Axis* rows, const Axis* cols) : s_(s), rows_(rows), cols_(cols) {}
  std::int64_t stored_blocks() const { return info().first; }
  std::int64_t stored_elements() const { return info().second; }
  template <class Fn>
  void for_each(Fn&& fn) const {
    std::vector<std::int64_t> bi, bj;
    std::vector<double> v;
    pull(bi, bj, v);
    std::size_t off = 0;
    for (std::size_t t = 0; t < bi.size(); ++t) {
      const int m = rows_->size(bi[t]), n = cols_->size(bj[t]);
      DenseBlock b(m, n, std::vector<double>(v.begin() + off, v.begin() + off + std::size_t(m) * n));
      off += std::size_t(m) * n;
      fn(bi[t], bj[t], static_cast<const DenseBlock&>(b));
    }
  }
  template <class Fn>
  void for_each_in_row_range(std::int64_t i, std::int64_t col_begin, std::int64_t col_end,
                             Fn&& fn) const {
    for_each([&](std::int64_t r, std::int64_t c, const DenseBlock& b) {
      if (r == i && c >= col_begin && c < col_end) fn(r, c, b);
    });
  }
  bt_mat* handle() const noexcept { return s_; }

 private:
  std::pair<std::int64_t, std::int64_t> info() const {
    int64_t b = 0, e = 0;
    detail::check(bt_mat_info(s_, &b, &e));
    return {b, e};
  }
  void pull(std::vector<std::int64_t>& bi, std::vector<std::int64_t>& bj,
            std::vector<double>& v) const {
    const auto ie = info();
    bi.resize(static_cast<std::size_t>(ie.first));
    bj.resize(static_cast<std::size_t>(ie.first));
    v.resize(static_cast<std::size_t>(ie.second));
    if (ie.first) detail::check(bt_mat_export(s_, bi.data(), bj.data(), v.data()));
  }
  bt_mat* s_;
  const Axis* rows_;
  const Axis* cols_;
};

class DistMatrix {
 public:
  DistMatrix(Axis rows, Axis cols, ProcessGrid grid, SimComm* comm = SimComm::current())
      : rows_(std::move(rows)), cols_(std::move(cols)), grid_(std::move(grid)), comm_(comm) {
    if (!comm_) throw invalid_argument("DistMatrix: construct a SimComm first");
    if (grid_.ndims() != 2) throw invalid_argument("DistMatrix: grid must be 2-dimensional");
    if (rows_.extent() != grid_.dim(0) || cols_.extent() != grid_.dim(1))
      throw invalid_argument("DistMatrix: axis extents do not match the grid");
    const Blocking rb = rows_.blocking(), cb = cols_.blocking();
    const std::vector<int> rdv = rows_.dists(), cdv = cols_.dists();
    std::vector<int32_t> rs(rb.sizes().begin(), rb.sizes().end());
    std::vector<int32_t> cs(cb.sizes().begin(), cb.sizes().end());
    std::vector<int32_t> rd(rdv.begin(), rdv.end());
    std::vector<int32_t> cd(cdv.begin(), cdv.end());
    bt_dmat* h = nullptr;
    detail::check(bt_dmat_create(comm_->handle(), static_cast<int64_t>(rs.size()), rs.data(),
                                 static_cast<int64_t>(cs.size()), cs.data(), grid_.dim(0),
                                 grid_.dim(1), rd.data(), cd.data(), &h));
    h_.reset(h, [](bt_dmat* p) { bt_dmat_destroy(p); });
  }
  const Axis& rows() const noexcept { return rows_; }
  const Axis& cols() const noexcept { return cols_; }
  const ProcessGrid& grid() const noexcept { return grid_; }
  std::int64_t n_block_rows() const noexcept { return rows_.n_blocks(); }
  std::int64_t n_block_cols() const noexcept { return cols_.n_blocks(); }
  int owner_rank(std::int64_t i, std::int64_t j) const {
    return grid_.rank_of({rows_.dist(i), cols_.dist(j)});
  }
  int nranks() const noexcept { return grid_.size(); }
  bt_dmat* handle() const noexcept { return h_.get(); }

  SimComm* comm() const noexcept { return comm_; }

  // the store of rank `rank` (matrix.hpp:294-295); ownership_error when the
  // rank lives in another process
  LocalStore local(int rank) const {
    bt_mat* s = nullptr;
    detail::check(bt_dmat_local(h_.get(), rank, &s));
    return LocalStore(s, &rows_, &cols_);
  }

  void put_block(std::int64_t i, std::int64_t j, DenseBlock block, bool accumulate = false) {
    if (block.rows != rows_.size(i) || block.cols != cols_.size(j))
      throw invalid_argument("put_block: block dimensions do not match the slot");
    detail::check(bt_dmat_put_blocks(h_.get(), 1, &i, &j, block.values.data(), accumulate ? 1 : 0));
  }

  // ownership-checked variant used by rank workers (matrix.hpp:312-321)
  void put_block_at(int rank, std::int64_t i, std::int64_t j, DenseBlock block,
                    bool accumulate = false) {
    const int owner = owner_rank(i, j);
    if (owner != rank)
      throw ownership_error("put_block: rank " + std::to_string(rank) + " does not own block (" +
                            std::to_string(i) + "," + std::to_string(j) + "), rank " +
                            std::to_string(owner) + " does");
    put_block(i, j, std::move(block), accumulate);
  }

  const DenseBlock* get_block_at(int rank, std::int64_t i, std::int64_t j) const {
    const int owner = owner_rank(i, j);
    if (owner != rank)
      throw ownership_error("get_block: rank " + std::to_string(rank) + " does not own block (" +
                            std::to_string(i) + "," + std::to_string(j) + "), rank " +
                            std::to_string(owner) + " does");
    return get_block(i, j);
  }

  // every stored block of this process's ranks in (rank, row, col) order
  // (matrix.hpp:363-368)
  template <class Fn>
  void for_each_global(Fn&& fn) const {
    for (int r = 0; r < grid_.size(); ++r) {
      if (!comm_->is_local(r)) continue;
      local(r).for_each([&](std::int64_t i, std::int64_t j, const DenseBlock& b) { fn(r, i, j, b); });
    }
  }

  const DenseBlock* get_block(std::int64_t i, std::int64_t j) const {
    bt_mat* s = nullptr;
    detail::check(bt_dmat_local(h_.get(), owner_rank(i, j), &s));
    DenseBlock b(rows_.size(i), cols_.size(j));
    int found = 0;
    detail::check(bt_mat_get_block(s, i, j, b.values.data(), &found));
    if (!found) return nullptr;
    cache_[{i, j}] = std::move(b);
    return &cache_[{i, j}];
  }

  std::int64_t stored_blocks() const { return totals().first; }
  std::int64_t stored_elements() const { return totals().second; }
  double occupancy() const {
    const double dense = double(rows_.total_elements()) * double(cols_.total_elements());
    return dense == 0 ? 0.0 : double(stored_elements()) / dense;
  }

 private:
  std::pair<std::int64_t, std::int64_t> totals() const {
    std::int64_t nb = 0, ne = 0;
    for (int r = 0; r < grid_.size(); ++r) {
      bt_mat* s = nullptr;
      if (bt_dmat_local(h_.get(), r, &s) != BT_OK) continue;  // not local to this process
      int64_t b = 0, e = 0;
      detail::check(bt_mat_info(s, &b, &e));
      nb += b;
      ne += e;
    }
    // global counts: summed over the processes of an NCCL group (collective)
    int64_t v[2] = {nb, ne};
    detail::check(bt_grid_sum(comm_->handle(), v, 2));
    return {v[0], v[1]};
  }
  Axis rows_, cols_;
  ProcessGrid grid_;
  SimComm* comm_;
  std::shared_ptr<bt_dmat> h_;
  mutable std::map<std::pair<std::int64_t, std::int64_t>, DenseBlock> cache_;
};

inline DistMatrix new_matrix(const Blocking& rb, const Blocking& cb, const ProcessGrid& grid,
                             std::vector<int> row_dist, std::vector<int> col_dist) {
  if (grid.ndims() != 2) throw invalid_argument("new_matrix: grid must be 2-dimensional");
  return DistMatrix(Axis(rb, std::move(row_dist), grid.dim(0)),
                    Axis(cb, std::move(col_dist), grid.dim(1)), grid);
}

inline DistMatrix new_matrix_round_robin(const Blocking& rb, const Blocking& cb,
                                         const ProcessGrid& grid) {
  if (grid.ndims() != 2) throw invalid_argument("new_matrix: grid must be 2-dimensional");
  return DistMatrix(Axis::round_robin(rb, grid.dim(0)), Axis::round_robin(cb, grid.dim(1)), grid);
}

// ---------------------------------------------------------------- multiply
inline void multiply_cannon(SimComm&, const DistMatrix& a, const DistMatrix& b, DistMatrix& c,
                            double eps = 0.0) {
  detail::check(bt_multiply_cannon(a.handle(), b.handle(), c.handle(), eps, nullptr));
}
inline void multiply_reduce_case1(SimComm&, const DistMatrix& a, const DistMatrix& b,
                                  DistMatrix& c, int nprocs, double eps = 0.0) {
  detail::check(bt_multiply_case1(a.handle(), b.handle(), c.handle(), nprocs, eps, nullptr));
}
inline void multiply_virtual_case2(SimComm&, const DistMatrix& a, const DistMatrix& b,
                                   DistMatrix& c, int nprocs, double eps = 0.0) {
  detail::check(bt_multiply_case2(a.handle(), b.handle(), c.handle(), nprocs, 0, eps, nullptr));
}

enum class Algorithm { cannon, case1, case2 };
inline const char* algorithm_name(Algorithm a) {
  return a == Algorithm::cannon ? "cannon" : a == Algorithm::case1 ? "case1" : "case2";
}

inline void multiply_dispatch(SimComm& comm, Algorithm algo, const DistMatrix& a,
                              const DistMatrix& b, DistMatrix& c, int nprocs) {
  switch (algo) {
    case Algorithm::cannon: multiply_cannon(comm, a, b, c); return;
    case Algorithm::case1: multiply_reduce_case1(comm, a, b, c, nprocs); return;
    case Algorithm::case2: multiply_virtual_case2(comm, a, b, c, nprocs); return;
  }
  throw invalid_argument("multiply_dispatch: unknown algorithm");
}

inline void filter(DistMatrix& m, double eps) {
  for (int r = 0; r < m.nranks(); ++r) {
    bt_mat* s = nullptr;
    if (bt_dmat_local(m.handle(), r, &s) != BT_OK) continue;
    detail::check(bt_filter(s, eps));
  }
}

// ----------------------------------------------------------- redistribution
// redistribute (matrix.hpp:567-600): `src` onto a new layout on the device
// (owner split + NVLink/device exchange + merge), each block moved at most
// once and only blocks that change ranks charged to the ledger; with
// `transpose`, block (i,j) lands transposed at (j,i).
inline DistMatrix redistribute(SimComm& comm, const DistMatrix& src, Axis new_rows, Axis new_cols,
                               const ProcessGrid& new_grid, bool transpose = false,
                               const std::string& phase = "redistribute") {
  if (!transpose) {
    if (!src.rows().same_blocking(new_rows) || !src.cols().same_blocking(new_cols))
      throw invalid_argument("redistribute: target blockings do not match the source");
  } else if (!src.rows().same_blocking(new_cols) || !src.cols().same_blocking(new_rows)) {
    throw invalid_argument("redistribute: transposed target blockings do not match");
  }
  if (comm.nranks() < src.grid().size() || comm.nranks() < new_grid.size())
    throw invalid_argument("redistribute: communicator smaller than the involved grids");
  DistMatrix dst(std::move(new_rows), std::move(new_cols), new_grid, &comm);
  detail::check(bt_redistribute(src.handle(), dst.handle(), transpose ? 1 : 0, 0, phase.c_str()));
  return dst;
}

// redistribute_add (matrix.hpp:604-622): every stored block of `src` routed
// into `dst`, accumulating into blocks already present.
inline void redistribute_add(SimComm& comm, const DistMatrix& src, DistMatrix& dst,
                             const std::string& phase = "redistribute") {
  if (!src.rows().same_blocking(dst.rows()) || !src.cols().same_blocking(dst.cols()))
    throw invalid_argument("redistribute_add: blockings do not conform");
  if (comm.nranks() < src.grid().size() || comm.nranks() < dst.grid().size())
    throw invalid_argument("redistribute_add: communicator smaller than the involved grids");
  detail::check(bt_redistribute(src.handle(), dst.handle(), 0, 1, phase.c_str()));
}

// -------------------------------------------------------------- fixture I/O
// Fixture files in the reference's formats (io.hpp:22-198), same signatures:
//  text   "rows cols nblkrows nblkcols" / row block sizes / column block sizes /
//         per block "i j" and its row-major values (shortest round-trip
//         decimal, std::to_chars);
//  binary the same fields as little-endian int64 / 8-byte doubles.
// Blocks are written in (i, j) order.  A DistMatrix's blocks are read from the
// device; with one rank per process (NCCL) a writer sees only its own ranks'
// blocks.
enum class FileFormat { text, binary };

struct MatrixData {
  Blocking rows;
  Blocking cols;
  std::vector<std::tuple<std::int64_t, std::int64_t, DenseBlock>> blocks;
};

namespace detail {
inline std::string format_double(double v) {
  char buf[64];
  auto res = std::to_chars(buf, buf + sizeof(buf), v);
  if (res.ec != std::errc()) throw error("format_double failed");
  return std::string(buf, res.ptr);
}
inline void put_i64(std::ostream& os, std::int64_t v) {
  unsigned char b[8];
  const auto u = static_cast<std::uint64_t>(v);
  for (int t = 0; t < 8; ++t) b[t] = static_cast<unsigned char>((u >> (8 * t)) & 0xff);
  os.write(reinterpret_cast<const char*>(b), 8);
}
inline bool get_i64(std::istream& is, std::int64_t& v) {
  unsigned char b[8];
  if (!is.read(reinterpret_cast<char*>(b), 8)) return false;
  std::uint64_t u = 0;
  for (int t = 7; t >= 0; --t) u = (u << 8) | b[t];
  v = static_cast<std::int64_t>(u);
  return true;
}
inline void put_f64(std::ostream& os, double v) {
  std::uint64_t u;
  std::memcpy(&u, &v, 8);
  put_i64(os, static_cast<std::int64_t>(u));
}
inline bool get_f64(std::istream& is, double& v) {
  std::int64_t i;
  if (!get_i64(is, i)) return false;
  const auto u = static_cast<std::uint64_t>(i);
  std::memcpy(&v, &u, 8);
  return true;
}
// this process's blocks in (i, j) order
inline std::vector<std::tuple<std::int64_t, std::int64_t, DenseBlock>> sorted_blocks(
    const DistMatrix& m) {
  std::vector<std::tuple<std::int64_t, std::int64_t, DenseBlock>> all;
  m.for_each_global([&](int, std::int64_t i, std::int64_t j, const DenseBlock& b) {
    all.emplace_back(i, j, b);
  });
  std::sort(all.begin(), all.end(), [](const auto& x, const auto& y) {
    return std::make_pair(std::get<0>(x), std::get<1>(x)) <
           std::make_pair(std::get<0>(y), std::get<1>(y));
  });
  return all;
}
inline MatrixData read_header(std::istream& is, bool binary) {
  std::int64_t rows = 0, cols = 0, nbr = 0, nbc = 0;
  if (binary) {
    if (!get_i64(is, rows) || !get_i64(is, cols) || !get_i64(is, nbr) || !get_i64(is, nbc))
      throw error("matrix file: bad binary header");
  } else if (!(is >> rows >> cols >> nbr >> nbc)) {
    throw error("matrix file: bad header");
  }
  if (nbr < 0 || nbc < 0) throw error("matrix file: bad header");
  std::vector<int> rs(static_cast<std::size_t>(nbr)), cs(static_cast<std::size_t>(nbc));
  for (int pass = 0; pass < 2; ++pass)
    for (auto& x : pass ? cs : rs) {
      std::int64_t v = 0;
      const bool ok = binary ? get_i64(is, v) : static_cast<bool>(is >> v);
      if (!ok) throw error(pass ? "matrix file: bad column blocking" : "matrix file: bad row blocking");
      x = static_cast<int>(v);
    }
  MatrixData d{Blocking(rs), Blocking(cs), {}};
  if (d.rows.total() != rows || d.cols.total() != cols)
    throw error("matrix file: blocking does not sum to the header dimensions");
  return d;
}
}  // namespace detail

inline void write_matrix_text(std::ostream& os, const DistMatrix& m) {
  os << m.rows().total_elements() << ' ' << m.cols().total_elements() << ' '
     << m.n_block_rows() << ' ' << m.n_block_cols() << '\n';
  for (std::int64_t b = 0; b < m.n_block_rows(); ++b)
    os << m.rows().size(b) << (b + 1 < m.n_block_rows() ? ' ' : '\n');
  if (m.n_block_rows() == 0) os << '\n';
  for (std::int64_t b = 0; b < m.n_block_cols(); ++b)
    os << m.cols().size(b) << (b + 1 < m.n_block_cols() ? ' ' : '\n');
  if (m.n_block_cols() == 0) os << '\n';
  for (const auto& ijb : detail::sorted_blocks(m)) {
    os << std::get<0>(ijb) << ' ' << std::get<1>(ijb) << '\n';
    const auto& v = std::get<2>(ijb).values;
    for (std::size_t t = 0; t < v.size(); ++t)
      os << detail::format_double(v[t]) << (t + 1 < v.size() ? ' ' : '\n');
  }
}

inline MatrixData read_matrix_data_text(std::istream& is) {
  MatrixData d = detail::read_header(is, false);
  std::int64_t i, j;
  while (is >> i >> j) {
    if (i < 0 || i >= d.rows.n_blocks() || j < 0 || j >= d.cols.n_blocks())
      throw error("matrix file: block index out of range");
    DenseBlock b(d.rows.size(i), d.cols.size(j));
    for (auto& v : b.values)
      if (!(is >> v)) throw error("matrix file: truncated block values");
    d.blocks.emplace_back(i, j, std::move(b));
  }
  return d;
}

inline void write_matrix_binary(std::ostream& os, const DistMatrix& m) {
  detail::put_i64(os, m.rows().total_elements());
  detail::put_i64(os, m.cols().total_elements());
  detail::put_i64(os, m.n_block_rows());
  detail::put_i64(os, m.n_block_cols());
  for (std::int64_t b = 0; b < m.n_block_rows(); ++b) detail::put_i64(os, m.rows().size(b));
  for (std::int64_t b = 0; b < m.n_block_cols(); ++b) detail::put_i64(os, m.cols().size(b));
  for (const auto& ijb : detail::sorted_blocks(m)) {
    detail::put_i64(os, std::get<0>(ijb));
    detail::put_i64(os, std::get<1>(ijb));
    for (double v : std::get<2>(ijb).values) detail::put_f64(os, v);
  }
}

inline MatrixData read_matrix_data_binary(std::istream& is) {
  MatrixData d = detail::read_header(is, true);
  std::int64_t i;
  while (detail::get_i64(is, i)) {
    std::int64_t j;
    if (!detail::get_i64(is, j)) throw error("matrix file: truncated block header");
    if (i < 0 || i >= d.rows.n_blocks() || j < 0 || j >= d.cols.n_blocks())
      throw error("matrix file: block index out of range");
    DenseBlock b(d.rows.size(i), d.cols.size(j));
    for (auto& v : b.values)
      if (!detail::get_f64(is, v)) throw error("matrix file: truncated block values");
    d.blocks.emplace_back(i, j, std::move(b));
  }
  return d;
}

// to_dist_matrix (io.hpp:181-185): round robin on `grid`; the blocks this
// process owns go to the device in one batched upload (with one rank per
// process every process reads the file and keeps its share)
inline DistMatrix to_dist_matrix(MatrixData&& data, const ProcessGrid& grid) {
  DistMatrix m = new_matrix_round_robin(data.rows, data.cols, grid);
  std::vector<std::int64_t> bi, bj;
  std::vector<double> v;
  for (auto& t : data.blocks) {
    const std::int64_t i = std::get<0>(t), j = std::get<1>(t);
    if (!m.comm()->is_local(m.owner_rank(i, j))) continue;
    const DenseBlock& b = std::get<2>(t);
    if (b.rows != data.rows.size(i) || b.cols != data.cols.size(j))
      throw invalid_argument("put_block: block dimensions do not match the slot");
    bi.push_back(i);
    bj.push_back(j);
    v.insert(v.end(), b.values.begin(), b.values.end());
  }
  if (!bi.empty())
    detail::check(bt_dmat_put_blocks(m.handle(), static_cast<int64_t>(bi.size()), bi.data(),
                                     bj.data(), v.data(), 0));
  data.blocks.clear();
  return m;
}

inline void write_matrix_file(const std::string& path, const DistMatrix& m, FileFormat format) {
  std::ofstream os(path, format == FileFormat::binary ? std::ios::binary : std::ios::out);
  if (!os) throw error("cannot open " + path + " for writing");
  if (format == FileFormat::binary) write_matrix_binary(os, m); else write_matrix_text(os, m);
  if (!os) throw error("write to " + path + " failed");
}

inline MatrixData read_matrix_file(const std::string& path, FileFormat format) {
  std::ifstream is(path, format == FileFormat::binary ? std::ios::binary : std::ios::in);
  if (!is) throw error("cannot open " + path);
  return format == FileFormat::binary ? read_matrix_data_binary(is) : read_matrix_data_text(is);
}

// -------------------------------------------------------------- cost model
struct MultiplySpec {
  double m = 0, n = 0, k = 0, occ_a = 1.0, occ_b = 1.0, occ_c = 1.0, nprocs = 1;
  double stored_a() const { return occ_a * m * k; }
  double stored_b() const { return occ_b * k * n; }
  double stored_c() const { return occ_c * m * n; }
  void validate() const {
    if (m < 1 || n < 1 || k < 1) throw invalid_argument("MultiplySpec: dims must be >= 1");
    if (nprocs < 1) throw invalid_argument("MultiplySpec: process count must be >= 1");
    for (double o : {occ_a, occ_b, occ_c})
      if (o < 0.0 || o > 1.0) throw invalid_argument("MultiplySpec: occupancies must be in [0,1]");
  }
};
// Eq. 1, 2, 5 of the paper (volumes in elements per process)
inline double cannon_volume(const MultiplySpec& s) {
  s.validate();
  return (s.stored_a() + s.stored_b()) / std::sqrt(s.nprocs);
}
inline double case1_volume(const MultiplySpec& s) {
  s.validate();
  return (s.stored_a() + s.stored_b()) / s.nprocs + s.stored_c();
}
inline double case2_volume(const MultiplySpec& s) {
  s.validate();
  return (s.stored_a() + s.stored_b() + s.stored_c()) / s.nprocs + s.stored_b();
}
inline Algorithm select_algorithm(double m, double n, double k, double oa, double ob, double oc,
                                  double p) {
  MultiplySpec s{m, n, k, oa, ob, oc, p};
  Algorithm best = Algorithm::cannon;
  double v = cannon_volume(s);
  if (case1_volume(s) < v) {
    best = Algorithm::case1;
    v = case1_volume(s);
  }
  if (case2_volume(s) < v) best = Algorithm::case2;
  return best;
}
// Extension: NVLink/NVSwitch-aware time model, seconds per
// multiply on s.nprocs B200s -- the mirror of dist.py predicted_time_b200,
// with the rates FITTED to the measured times of every algorithm on 2 and 4
// B200s (tests/golden/algo_times_b200.jsonl, tools/algo_sweep.py).
struct B200Machine {
  double fp64_flops = 25.6e12;    // local multiply, useful FP64
  double hbm_bytes = 6.55e12;     // C written once
  double cannon_bytes = 237e9;    // Cannon panel shifts
  double redist_bytes = 126e9;    // layout changes of case 1 / case 2
  double reduce_bytes = 265e9;    // case 1 partial-C reduction
  double gather_bytes = 33.1e9;   // case 2 B gather incl. assembly
  double cannon_overhead = 0.86e-3, case1_overhead = 2.92e-3, case2_overhead = 0.0;
};
inline double predicted_time_b200(Algorithm algo, const MultiplySpec& s,
                                  const B200Machine& hw = B200Machine{}) {
  s.validate();
  const double p = s.nprocs;
  const double flops = 2.0 * s.m * s.n * s.k * s.occ_a * s.occ_b;
  const double sa = s.stored_a(), sb = s.stored_b(), sc = s.stored_c();
  const double compute = flops / (p * hw.fp64_flops) + 8.0 * sc / p / hw.hbm_bytes;
  switch (algo) {
    case Algorithm::cannon: {
      const double q = std::round(std::sqrt(p));
      if (q * q != p) return std::numeric_limits<double>::infinity();
      if (p == 1) return compute;
      return std::max(compute, 8.0 * cannon_volume(s) / hw.cannon_bytes) + hw.cannon_overhead;
    }
    case Algorithm::case1:
      if (p == 1) return compute;
      return flops / (p * hw.fp64_flops) + 8.0 * sc / hw.hbm_bytes +
             8.0 * (sa + sb) / p / hw.redist_bytes + 8.0 * sc * (p - 1) / p / hw.reduce_bytes +
             hw.case1_overhead;
    case Algorithm::case2:
      if (p == 1) return compute;
      return std::max(compute, 8.0 * sb * (p - 1) / p / hw.gather_bytes) +
             8.0 * (sa + sc) / p / hw.redist_bytes + hw.case2_overhead;
  }
  throw invalid_argument("predicted_time_b200: unknown algorithm");
}
inline Algorithm select_algorithm_b200(double m, double n, double k, double oa, double ob,
                                       double oc, double p,
                                       const B200Machine& hw = B200Machine{}) {
  MultiplySpec s{m, n, k, oa, ob, oc, p};
  Algorithm best = Algorithm::cannon;
  double t = predicted_time_b200(best, s, hw);
  for (Algorithm a : {Algorithm::case1, Algorithm::case2}) {
    const double ta = predicted_time_b200(a, s, hw);
    if (ta < t) {
      best = a;
      t = ta;
    }
  }
  return best;
}
inline MultiplySpec measured_spec(const DistMatrix& a, const DistMatrix& b, double occ_c,
                                  int nprocs) {
  MultiplySpec s;
  s.m = double(a.rows().total_elements());
  s.k = double(a.cols().total_elements());
  s.n = double(b.cols().total_elements());
  s.occ_a = a.occupancy();
  s.occ_b = b.occupancy();
  s.occ_c = occ_c;
  s.nprocs = nprocs;
  return s;
}

// multiply_dispatch with the algorithm chosen by the fitted B200 model among
// those whose layout preconditions hold (Cannon: square grid of nprocs, C =
// A rows x B cols); case 2 runs as the one-step NVLink gather.  Mirrors
// dist.py select_for / multiply_dispatch(Algorithm.auto).  Returns the choice.
inline Algorithm multiply_auto(SimComm& comm, const DistMatrix& a, const DistMatrix& b,
                               DistMatrix& c, int nprocs, double eps = 0.0,
                               const B200Machine& hw = B200Machine{}) {
  MultiplySpec s = measured_spec(a, b, 0.0, nprocs);
  const double p = std::min(std::max(s.occ_a * s.occ_b, 0.0), 1.0);
  s.occ_c = std::min(1.0, std::max(0.0, 1.0 - std::pow(1.0 - p, double(a.n_block_cols()))));
  const ProcessGrid& g = a.grid();
  const bool cannon_ok = g.ndims() == 2 && g.dim(0) == g.dim(1) && g.dim(0) * g.dim(1) == nprocs &&
                         b.grid() == g && c.grid() == g && c.rows().same_distribution(a.rows()) &&
                         c.cols().same_distribution(b.cols()) &&
                         a.cols().same_distribution(b.rows());
  Algorithm best = Algorithm::case1;
  double t = predicted_time_b200(Algorithm::case1, s, hw);
  if (cannon_ok && predicted_time_b200(Algorithm::cannon, s, hw) <= t) {
    best = Algorithm::cannon;
    t = predicted_time_b200(Algorithm::cannon, s, hw);
  }
  if (predicted_time_b200(Algorithm::case2, s, hw) < t) best = Algorithm::case2;
  switch (best) {
    case Algorithm::cannon: multiply_cannon(comm, a, b, c, eps); break;
    case Algorithm::case1: multiply_reduce_case1(comm, a, b, c, nprocs, eps); break;
    case Algorithm::case2:
      detail::check(bt_multiply_case2(a.handle(), b.handle(), c.handle(), nprocs, 1, eps, nullptr));
      break;
  }
  return best;
}


// ------------------------------------------------------------- tall-skinny
// SPEC.md:415-477 (the reference has this module only in its spec): a
// tall-and-skinny matrix split along its long dimension into f approximately
// square submatrices, index data along that dimension supplied by functions
// (IndexFuncs, the spec's form of Axis::functional) so no host array spans the
// full split dimension.  Submatrix s lives on SUBGROUP s of the ranks:
//  * one rank per process (NCCL): ranks [s*P/f, (s+1)*P/f) with their own
//    communicator (bt_ctx_split); this process holds its subgroup's submatrix
//    only, and the subgroups multiply concurrently;
//  * virtual ranks (one process): one SimComm per subgroup on this GPU, the
//    subgroups run one after another (the spec's sequential schedule).
// multiply_tall_skinny supports the K split (A split on columns, B on rows,
// C a plain DistMatrix of the parent group): C += sum_s A_s B_s, the partial
// C of every subgroup reduced into C with redistribute_add on the parent
// group (ledger phase "ts_reduce", the spec's cross-subgroup reduction).
struct IndexFuncs {
  std::int64_t n_blocks = 0;
  std::function<int(std::int64_t)> block_size_fn;
  std::function<int(std::int64_t)> dist_fn;
  int size(std::int64_t b) const {
    if (b < 0 || b >= n_blocks) throw invalid_argument("IndexFuncs: block out of range");
    const int v = block_size_fn(b);
    if (v < 1) throw invalid_argument("IndexFuncs: block sizes must be >= 1");
    return v;
  }
  int dist(std::int64_t b) const { return dist_fn(b); }
};

// ceiling partition: the first submatrices get ceil(n/f) block indices
inline std::vector<std::pair<std::int64_t, std::int64_t>> ceil_partition(std::int64_t n, int f) {
  if (f < 1) throw invalid_argument("ceil_partition: factor must be >= 1");
  const std::int64_t w = n ? (n + f - 1) / f : 0;
  std::vector<std::pair<std::int64_t, std::int64_t>> out;
  for (int s = 0; s < f; ++s) out.emplace_back(std::min(n, s * w), std::min(n, (s + 1) * w));
  return out;
}

// argmin over f in 1..P of |long/f - short| in element units, ties to smaller f
inline int choose_split_factor(double long_elems, double short_elems, int nprocs) {
  if (long_elems <= 0 || short_elems <= 0 || nprocs < 1)
    throw invalid_argument("choose_split_factor: inputs must be positive");
  int best = 1;
  double bd = std::fabs(long_elems - short_elems);
  for (int f = 2; f <= nprocs; ++f) {
    const double d = std::fabs(long_elems / f - short_elems);
    if (d < bd) {
      best = f;
      bd = d;
    }
  }
  return best;
}

// The f subgroups of a parent group (shared by every tall-skinny matrix of
// one contraction): P/f ranks each, contiguous, on a sub_grid of that size.
class Subgroups {
 public:
  Subgroups(SimComm& parent, int factor, ProcessGrid sub_grid)
      : parent_(&parent), f_(factor), sub_grid_(std::move(sub_grid)) {
    const int P = parent.nranks();
    if (factor < 1 || P % factor != 0 || sub_grid_.size() != P / factor)
      throw invalid_argument("Subgroups: factor must divide the group and sub_grid hold P/f ranks");
    const std::vector<int> mine = parent.local_ranks();
    if (static_cast<int>(mine.size()) == P) {  // virtual ranks: one SimComm per subgroup
      for (int s = 0; s < f_; ++s) {
        local_.push_back(s);
        comms_.emplace_back(new SimComm(sub_grid_));
      }
    } else {                                    // NCCL: this process's subgroup
      const int r = mine.at(0), s = r / (P / f_);
      bt_ctx* sub = nullptr;
      detail::check(bt_ctx_split(parent.context(), s, r, &sub));
      local_.push_back(s);
      comms_.emplace_back(new SimComm(sub_grid_, sub));
    }
    SimComm::current() = &parent;
  }
  int factor() const noexcept { return f_; }
  const ProcessGrid& sub_grid() const noexcept { return sub_grid_; }
  SimComm& parent() const noexcept { return *parent_; }
  // subgroups held by this process and their communicators
  const std::vector<int>& local() const noexcept { return local_; }
  SimComm& comm_of(int s) const {
    for (std::size_t t = 0; t < local_.size(); ++t)
      if (local_[t] == s) return *comms_[t];
    throw ownership_error("Subgroups: subgroup " + std::to_string(s) + " lives in another process");
  }
  int first_parent_rank(int s) const { return s * sub_grid_.size(); }

 private:
  SimComm* parent_;
  int f_;
  ProcessGrid sub_grid_;
  std::vector<int> local_;
  std::vector<std::unique_ptr<SimComm>> comms_;
};

enum class SplitDim { rows, cols };

class TallSkinnyMatrix {
 public:
  TallSkinnyMatrix(Subgroups& groups, IndexFuncs rows, IndexFuncs cols, SplitDim dim)
      : groups_(&groups), rows_(std::move(rows)), cols_(std::move(cols)), dim_(dim) {
    const std::int64_t n = dim == SplitDim::rows ? rows_.n_blocks : cols_.n_blocks;
    ranges_ = ceil_partition(n, groups.factor());
    const ProcessGrid& g = groups.sub_grid();
    for (int s : groups.local()) {
      const auto r = ranges_[static_cast<std::size_t>(s)];
      // functional axes over the submatrix's range only (no full-length arrays)
      auto axis = [&](const IndexFuncs& f, std::int64_t b0, std::int64_t nb, int extent) {
        const IndexFuncs fc = f;
        return Axis::functional(
            nb, [fc, b0](std::int64_t b) { return fc.size(b0 + b); },
            [fc, b0, extent](std::int64_t b) { return ((fc.dist(b0 + b) % extent) + extent) % extent; },
            extent);
      };
      Axis ra = dim == SplitDim::rows ? axis(rows_, r.first, r.second - r.first, g.dim(0))
                                      : axis(rows_, 0, rows_.n_blocks, g.dim(0));
      Axis ca = dim == SplitDim::cols ? axis(cols_, r.first, r.second - r.first, g.dim(1))
                                      : axis(cols_, 0, cols_.n_blocks, g.dim(1));
      subs_.emplace_back(s, std::unique_ptr<DistMatrix>(
                                new DistMatrix(std::move(ra), std::move(ca), g, &groups.comm_of(s))));
      index_len_.push_back(r.second - r.first);
    }
  }
  SplitDim split_dim() const noexcept { return dim_; }
  int factor() const noexcept { return groups_->factor(); }
  const IndexFuncs& rows() const noexcept { return rows_; }
  const IndexFuncs& cols() const noexcept { return cols_; }
  Subgroups& groups() const noexcept { return *groups_; }
  const std::vector<std::pair<std::int64_t, std::int64_t>>& ranges() const noexcept { return ranges_; }
  // global split-dimension block -> (submatrix, local index), and back
  std::pair<int, std::int64_t> locate(std::int64_t b) const {
    const std::int64_t n = ranges_.empty() ? 0 : ranges_.back().second;
    if (b < 0 || b >= n) throw invalid_argument("TallSkinnyMatrix: block out of range");
    const std::int64_t w = ranges_[0].second - ranges_[0].first;
    const int s = static_cast<int>(b / w);
    return {s, b - ranges_[static_cast<std::size_t>(s)].first};
  }
  std::int64_t global_index(int s, std::int64_t local) const {
    const auto r = ranges_.at(static_cast<std::size_t>(s));
    if (local < 0 || local >= r.second - r.first) throw invalid_argument("TallSkinnyMatrix: local index out of range");
    return r.first + local;
  }
  bool holds(int s) const {
    for (const auto& p : subs_)
      if (p.first == s) return true;
    return false;
  }
  DistMatrix& sub(int s) const {
    for (const auto& p : subs_)
      if (p.first == s) return *p.second;
    throw ownership_error("TallSkinnyMatrix: submatrix " + std::to_string(s) + " lives in another process");
  }
  // put_block routed to its submatrix; blocks of another process's subgroup
  // are skipped (each process puts its own share) -- returns whether stored
  bool put_block(std::int64_t i, std::int64_t j, DenseBlock block, bool accumulate = false) {
    const auto loc = locate(dim_ == SplitDim::rows ? i : j);
    if (!holds(loc.first)) return false;
    DistMatrix& m = sub(loc.first);
    const std::int64_t li = dim_ == SplitDim::rows ? loc.second : i;
    const std::int64_t lj = dim_ == SplitDim::rows ? j : loc.second;
    if (!m.comm()->is_local(m.owner_rank(li, lj))) return false;
    m.put_block(li, lj, std::move(block), accumulate);
    return true;
  }
  // host index entries along the split dimension resident in this process
  // (functional axes: none) and the longest device index range (one submatrix)
  std::int64_t host_index_entries() const {
    std::int64_t e = 0;
    for (const auto& p : subs_) e += p.second->rows().index_entries() + p.second->cols().index_entries();
    return e;
  }
  std::int64_t max_device_index_range() const {
    std::int64_t m = 0;
    for (auto v : index_len_) m = std::max(m, v);
    return m;
  }

 private:
  Subgroups* groups_;
  IndexFuncs rows_, cols_;
  SplitDim dim_;
  std::vector<std::pair<std::int64_t, std::int64_t>> ranges_;
  std::vector<std::pair<int, std::unique_ptr<DistMatrix>>> subs_;
  std::vector<std::int64_t> index_len_;
};

// C += A * B with A split on K (columns) and B on K (rows) over the same
// subgroups; C is a DistMatrix of the parent group.  Each subgroup multiplies
// its pair (multiply_auto picks the algorithm on the subgroup), then the
// partial C blocks are reduced into C across subgroups (redistribute_add on
// the parent group, ledger phase "ts_reduce").
inline void multiply_tall_skinny(const TallSkinnyMatrix& a, const TallSkinnyMatrix& b,
                                 DistMatrix& c, double eps = 0.0) {
  if (a.split_dim() != SplitDim::cols || b.split_dim() != SplitDim::rows)
    throw layout_error("k", "multiply_tall_skinny: the C++ layer runs the K split (A split on "
                            "columns, B on rows); M/N splits: paper_1910_13555_b200/tall_skinny.py");
  if (&a.groups() != &b.groups())
    throw layout_error("k", "multiply_tall_skinny: A and B must share their subgroups");
  if (a.cols().n_blocks != b.rows().n_blocks)
    throw layout_error("k", "multiply_tall_skinny: contracted dimension splits differ");
  for (std::int64_t t = 0; t < a.cols().n_blocks; ++t)
    if (a.cols().size(t) != b.rows().size(t))
      throw layout_error("k", "multiply_tall_skinny: contracted dimension blockings differ");
  Subgroups& g = a.groups();
  SimComm& parent = g.parent();
  // partial C of every local subgroup, then staged into a parent-group matrix
  DistMatrix partial(Axis::round_robin(c.rows().blocking(), c.grid().dim(0)),
                     Axis::round_robin(c.cols().blocking(), c.grid().dim(1)), c.grid(), &parent);
  for (int s : g.local()) {
    SimComm& sc = g.comm_of(s);
    const ProcessGrid& sg = g.sub_grid();
    DistMatrix cs(Axis::round_robin(c.rows().blocking(), sg.dim(0)),
                  Axis::round_robin(c.cols().blocking(), sg.dim(1)), sg, &sc);
    multiply_auto(sc, a.sub(s), b.sub(s), cs, sg.size(), eps);
    for (int r = 0; r < sg.size(); ++r) {
      if (!sc.is_local(r)) continue;
      bt_mat* src = cs.local(r).handle();
      const int pr = g.first_parent_rank(s) + r;
      if (!parent.is_local(pr)) continue;
      bt_mat* dst = partial.local(pr).handle();
      detail::check(bt_mat_copy(src, dst));
    }
  }
  redistribute_add(parent, partial, c, "ts_reduce");
  SimComm::current() = &parent;
}

// ------------------------------------------------------------------ tensors
// SPEC.md:479-545 (the tensor module exists only in the reference's spec):
// block-sparse tensors of rank 2..4 stored as a device matrix under a
// matricization map (row-group dims | col-group dims), mixed radix with later
// dimensions fastest for block indices and for the elements inside a block
// (SPEC.md:505-513, 533).  Mirror of paper_1910_13555_b200/tensor.py; the
// index remap runs on the device (bt_tensor_remap), the contraction through
// the block-sparse multiply (bt_multiply).
inline std::int64_t mixed_radix(const std::vector<std::int64_t>& coords,
                                const std::vector<std::int64_t>& extents) {
  if (coords.size() != extents.size()) throw invalid_argument("mixed_radix: rank mismatch");
  std::int64_t idx = 0;
  for (std::size_t d = 0; d < coords.size(); ++d) {
    if (coords[d] < 0 || coords[d] >= extents[d])
      throw invalid_argument("tensor index out of range");
    idx = idx * extents[d] + coords[d];
  }
  return idx;
}

class SparseTensor {
 public:
  SparseTensor(SimComm& comm, std::vector<Blocking> dims, std::vector<int> row_dims,
               std::vector<int> col_dims)
      : ctx_(comm.context()), dims_(std::move(dims)), row_(std::move(row_dims)),
        col_(std::move(col_dims)) {
    const int n = static_cast<int>(dims_.size());
    if (n < 2 || n > 4) throw invalid_argument("tensor: rank must be in [2, 4]");
    std::vector<int> all(row_);
    all.insert(all.end(), col_.begin(), col_.end());
    std::vector<int> sorted_all(all);
    std::sort(sorted_all.begin(), sorted_all.end());
    for (int d = 0; d < n; ++d)
      if (static_cast<int>(sorted_all.size()) != n || sorted_all[d] != d || row_.empty() ||
          col_.empty())
        throw invalid_argument(
            "tensor: map is not a partition of the dimensions into two non-empty groups");
    const std::vector<int> rs = group_sizes(row_), cs = group_sizes(col_);
    detail::check(bt_mat_create(ctx_, static_cast<std::int64_t>(rs.size()), rs.data(),
                                static_cast<std::int64_t>(cs.size()), cs.data(), &m_));
  }
  SparseTensor(const SparseTensor&) = delete;
  SparseTensor& operator=(const SparseTensor&) = delete;
  SparseTensor(SparseTensor&& o) noexcept
      : ctx_(o.ctx_), dims_(std::move(o.dims_)), row_(std::move(o.row_)),
        col_(std::move(o.col_)), m_(o.m_) {
    o.m_ = nullptr;
  }
  ~SparseTensor() {
    if (m_) bt_mat_destroy(m_);
  }

  int rank() const noexcept { return static_cast<int>(dims_.size()); }
  const std::vector<Blocking>& dims() const noexcept { return dims_; }
  const std::vector<int>& row_dims() const noexcept { return row_; }
  const std::vector<int>& col_dims() const noexcept { return col_; }
  bt_mat* store() const noexcept { return m_; }

  // tensor_to_matrix_index
  std::pair<std::int64_t, std::int64_t> to_matrix_index(
      const std::vector<std::int64_t>& coords) const {
    if (static_cast<int>(coords.size()) != rank()) throw invalid_argument("tensor: rank mismatch");
    return {group_index(row_, coords), group_index(col_, coords)};
  }
  std::vector<int> block_shape(const std::vector<std::int64_t>& coords) const {
    std::vector<int> sh(dims_.size());
    for (std::size_t d = 0; d < dims_.size(); ++d) sh[d] = dims_[d].size(coords[d]);
    return sh;
  }
  // values row-major over the tensor dimensions (dimension 0 slowest)
  void put_block(const std::vector<std::int64_t>& coords, const std::vector<double>& values,
                 bool accumulate = false) {
    const auto sh = block_shape(coords);
    std::int64_t n = 1;
    for (int s : sh) n *= s;
    if (static_cast<std::int64_t>(values.size()) != n)
      throw invalid_argument("tensor put_block: value count does not match the block shape");
    const auto ij = to_matrix_index(coords);
    const std::vector<double> mat = permute(values, sh, order(), false);
    const std::int64_t i = ij.first, j = ij.second;
    const double* v = mat.data();
    detail::check(bt_mat_put_blocks(m_, 1, &i, &j, v, accumulate ? 1 : 0));
  }
  bool get_block(const std::vector<std::int64_t>& coords, std::vector<double>& out) const {
    const auto sh = block_shape(coords);
    std::int64_t n = 1;
    for (int s : sh) n *= s;
    std::vector<double> mat(static_cast<std::size_t>(n));
    const auto ij = to_matrix_index(coords);
    int found = 0;
    detail::check(bt_mat_get_block(m_, ij.first, ij.second, mat.data(), &found));
    if (!found) return false;
    out = permute(mat, sh, order(), true);
    return true;
  }
  // the same tensor under another map (device remap kernel)
  SparseTensor remap(SimComm& comm, std::vector<int> row_dims, std::vector<int> col_dims) const {
    SparseTensor out(comm, dims_, row_dims, col_dims);
    std::vector<std::int64_t> nb(dims_.size());
    std::vector<std::vector<std::int32_t>> sz(dims_.size());
    std::vector<const std::int32_t*> szp(dims_.size());
    for (std::size_t d = 0; d < dims_.size(); ++d) {
      nb[d] = dims_[d].n_blocks();
      for (std::int64_t b = 0; b < nb[d]; ++b) sz[d].push_back(dims_[d].size(b));
      szp[d] = sz[d].data();
    }
    std::vector<int> src(row_), dst(row_dims);
    src.insert(src.end(), col_.begin(), col_.end());
    dst.insert(dst.end(), col_dims.begin(), col_dims.end());
    detail::check(bt_tensor_remap(ctx_, rank(), nb.data(), szp.data(),
                                  static_cast<int>(row_.size()), src.data(), m_,
                                  static_cast<int>(row_dims.size()), dst.data(), out.m_));
    return out;
  }

 private:
  std::vector<int> order() const {
    std::vector<int> o(row_);
    o.insert(o.end(), col_.begin(), col_.end());
    return o;
  }
  std::vector<int> group_sizes(const std::vector<int>& g) const {
    std::vector<int> out{1};
    for (int d : g) {
      std::vector<int> nx;
      for (int a : out)
        for (std::int64_t b = 0; b < dims_[d].n_blocks(); ++b) nx.push_back(a * dims_[d].size(b));
      out.swap(nx);
    }
    return out;
  }
  std::int64_t group_index(const std::vector<int>& g, const std::vector<std::int64_t>& c) const {
    std::vector<std::int64_t> cc, ext;
    for (int d : g) {
      cc.push_back(c[d]);
      ext.push_back(dims_[d].n_blocks());
    }
    return mixed_radix(cc, ext);
  }
  // tensor-order values <-> matrix-order values (axes permuted by `perm`)
  static std::vector<double> permute(const std::vector<double>& in, const std::vector<int>& sh,
                                     const std::vector<int>& perm, bool inverse) {
    const int n = static_cast<int>(sh.size());
    std::vector<std::int64_t> tstride(n), pstride(n);
    std::int64_t s = 1;
    for (int d = n - 1; d >= 0; --d) {
      tstride[d] = s;
      s *= sh[d];
    }
    s = 1;
    for (int q = n - 1; q >= 0; --q) {  // stride of tensor dim perm[q] in permuted order
      pstride[perm[q]] = s;
      s *= sh[perm[q]];
    }
    std::vector<double> out(in.size());
    std::vector<int> idx(n, 0);
    for (std::int64_t t = 0; t < static_cast<std::int64_t>(in.size()); ++t) {
      std::int64_t to = 0, po = 0;
      for (int d = 0; d < n; ++d) {
        to += idx[d] * tstride[d];
        po += idx[d] * pstride[d];
      }
      if (inverse) out[to] = in[po]; else out[po] = in[to];
      for (int d = n - 1; d >= 0; --d) {
        if (++idx[d] < sh[d]) break;
        idx[d] = 0;
      }
    }
    return out;
  }

  bt_ctx* ctx_ = nullptr;
  std::vector<Blocking> dims_;
  std::vector<int> row_, col_;
  bt_mat* m_ = nullptr;
};

// contract: C += sum over (A dims ca) == (B dims cb) of A * B.
// C's dimensions are A's retained dimensions (ascending) then B's.  Operands in
// compatible maps are used as they are; others are remapped on the device
// first, and C is remapped back to its own map.
inline void contract(SimComm& comm, const SparseTensor& a, const SparseTensor& b,
                     const std::vector<int>& ca, const std::vector<int>& cb, SparseTensor& c,
                     double eps = 0.0) {
  if (ca.size() != cb.size() || ca.empty())
    throw invalid_argument("contract: contracted index lists must be non-empty and equal in length");
  for (std::size_t q = 0; q < ca.size(); ++q)
    if (!(a.dims()[ca[q]].sizes() == b.dims()[cb[q]].sizes()))
      throw invalid_argument("contract: blockings of contracted indices differ");
  std::vector<int> ra, rb;
  for (int d = 0; d < a.rank(); ++d)
    if (std::find(ca.begin(), ca.end(), d) == ca.end()) ra.push_back(d);
  for (int d = 0; d < b.rank(); ++d)
    if (std::find(cb.begin(), cb.end(), d) == cb.end()) rb.push_back(d);
  if (c.rank() != static_cast<int>(ra.size() + rb.size()))
    throw invalid_argument("contract: C rank does not match the retained indices");
  std::vector<int> crow, ccol;
  for (int q = 0; q < c.rank(); ++q) (q < static_cast<int>(ra.size()) ? crow : ccol).push_back(q);
  const bool a_ok = a.row_dims() == ra && a.col_dims() == ca;
  const bool b_ok = b.row_dims() == cb && b.col_dims() == rb;
  const bool c_ok = c.row_dims() == crow && c.col_dims() == ccol;
  std::unique_ptr<SparseTensor> am, bm, cm;
  if (!a_ok) am.reset(new SparseTensor(a.remap(comm, ra, ca)));
  if (!b_ok) bm.reset(new SparseTensor(b.remap(comm, cb, rb)));
  if (!c_ok) cm.reset(new SparseTensor(c.remap(comm, crow, ccol)));
  bt_stats st{};
  detail::check(bt_multiply(comm.context(), am ? am->store() : a.store(),
                            bm ? bm->store() : b.store(), cm ? cm->store() : c.store(), eps, &st));
  if (!c_ok) {
    SparseTensor back = cm->remap(comm, c.row_dims(), c.col_dims());
    detail::check(bt_mat_copy(back.store(), c.store()));
  }
}

}  // namespace blocktensor
