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
//                         process's GPU (or, via SimComm::nccl, one rank per process)
//   matrix.hpp:26-418     Axis, DistMatrix, new_matrix, new_matrix_round_robin
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
#include <map>
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

// The device group: SimComm(grid) puts every rank of `grid` on one GPU of this
// process (device BT_DEVICE, default 0) as virtual ranks.
class SimComm {
 public:
  explicit SimComm(ProcessGrid grid, Schedule = Schedule::parallel, int device = 0)
      : grid_(std::move(grid)) {
    detail::check(bt_ctx_create(device, 1, 0, nullptr, &ctx_));
    detail::check(bt_grid_create(ctx_, grid_.size(), &g_));
    current() = this;
  }
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
class Axis {
 public:
  Axis() = default;
  Axis(const Blocking& b, std::vector<int> dist, int extent)
      : blocking_(b), dist_(std::move(dist)), extent_(extent) {
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
  std::int64_t n_blocks() const noexcept { return blocking_.n_blocks(); }
  int extent() const noexcept { return extent_; }
  int size(std::int64_t b) const { return blocking_.size(b); }
  int dist(std::int64_t b) const { return dist_.at(static_cast<std::size_t>(b)); }
  std::int64_t total_elements() const { return blocking_.total(); }
  const Blocking& blocking() const noexcept { return blocking_; }
  const std::vector<int>& dists() const noexcept { return dist_; }
  bool same_blocking(const Axis& o) const { return blocking_ == o.blocking_; }
  bool same_distribution(const Axis& o) const { return extent_ == o.extent_ && dist_ == o.dist_; }

 private:
  Blocking blocking_;
  std::vector<int> dist_;
  int extent_ = 1;
};

class DistMatrix {
 public:
  DistMatrix(Axis rows, Axis cols, ProcessGrid grid, SimComm* comm = SimComm::current())
      : rows_(std::move(rows)), cols_(std::move(cols)), grid_(std::move(grid)), comm_(comm) {
    if (!comm_) throw invalid_argument("DistMatrix: construct a SimComm first");
    if (grid_.ndims() != 2) throw invalid_argument("DistMatrix: grid must be 2-dimensional");
    if (rows_.extent() != grid_.dim(0) || cols_.extent() != grid_.dim(1))
      throw invalid_argument("DistMatrix: axis extents do not match the grid");
    std::vector<int32_t> rs(rows_.blocking().sizes().begin(), rows_.blocking().sizes().end());
    std::vector<int32_t> cs(cols_.blocking().sizes().begin(), cols_.blocking().sizes().end());
    std::vector<int32_t> rd(rows_.dists().begin(), rows_.dists().end());
    std::vector<int32_t> cd(cols_.dists().begin(), cols_.dists().end());
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

  void put_block(std::int64_t i, std::int64_t j, DenseBlock block, bool accumulate = false) {
    if (block.rows != rows_.size(i) || block.cols != cols_.size(j))
      throw invalid_argument("put_block: block dimensions do not match the slot");
    detail::check(bt_dmat_put_blocks(h_.get(), 1, &i, &j, block.values.data(), accumulate ? 1 : 0));
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
    return {nb, ne};
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

// -------------------------------------------------------------- fixture I/O
// Binary matrix files in the reference's format (io.hpp:132-178): little-endian
// int64 header rows, cols, nblkrows, nblkcols, the two blocking lists, then per
// block i, j and the row-major values, blocks in (i, j) order.
struct MatrixData {
  Blocking rows, cols;
  std::vector<std::int64_t> bi, bj;
  std::vector<double> values;  // blocks concatenated in listed order
};

namespace detail {
inline std::int64_t rd64(std::FILE* f, bool& ok) {
  unsigned char b[8];
  ok = ok && std::fread(b, 1, 8, f) == 8;
  std::uint64_t u = 0;
  for (int t = 7; t >= 0; --t) u = (u << 8) | b[t];
  return static_cast<std::int64_t>(u);
}
inline void wr64(std::FILE* f, std::uint64_t u) {
  unsigned char b[8];
  for (int t = 0; t < 8; ++t) b[t] = static_cast<unsigned char>((u >> (8 * t)) & 0xff);
  std::fwrite(b, 1, 8, f);
}
}  // namespace detail

inline MatrixData read_matrix_binary(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw error("cannot open " + path);
  bool ok = true;
  const std::int64_t rows = detail::rd64(f, ok), cols = detail::rd64(f, ok);
  const std::int64_t nbr = detail::rd64(f, ok), nbc = detail::rd64(f, ok);
  if (!ok || nbr < 0 || nbc < 0) {
    std::fclose(f);
    throw error("matrix file: bad binary header");
  }
  std::vector<int> rs(static_cast<std::size_t>(nbr)), cs(static_cast<std::size_t>(nbc));
  for (auto& x : rs) x = static_cast<int>(detail::rd64(f, ok));
  for (auto& x : cs) x = static_cast<int>(detail::rd64(f, ok));
  if (!ok) {
    std::fclose(f);
    throw error("matrix file: bad blocking");
  }
  MatrixData d{Blocking(rs), Blocking(cs), {}, {}, {}};
  if (d.rows.total() != rows || d.cols.total() != cols) {
    std::fclose(f);
    throw error("matrix file: blocking does not sum to the header dimensions");
  }
  for (;;) {
    bool more = true;
    const std::int64_t i = detail::rd64(f, more);
    if (!more) break;
    const std::int64_t j = detail::rd64(f, ok);
    if (!ok || i < 0 || i >= nbr || j < 0 || j >= nbc) {
      std::fclose(f);
      throw error("matrix file: block index out of range");
    }
    d.bi.push_back(i);
    d.bj.push_back(j);
    const std::int64_t n = std::int64_t(rs[i]) * cs[j];
    for (std::int64_t t = 0; t < n; ++t) {
      const std::int64_t u = detail::rd64(f, ok);
      double v;
      std::memcpy(&v, &u, 8);
      d.values.push_back(v);
    }
    if (!ok) {
      std::fclose(f);
      throw error("matrix file: truncated block values");
    }
  }
  std::fclose(f);
  return d;
}

// to_dist_matrix (io.hpp:181-185): round-robin on `grid`, one batched upload
inline DistMatrix to_dist_matrix(const MatrixData& d, const ProcessGrid& grid) {
  DistMatrix m = new_matrix_round_robin(d.rows, d.cols, grid);
  if (!d.bi.empty())
    detail::check(bt_dmat_put_blocks(m.handle(), static_cast<int64_t>(d.bi.size()), d.bi.data(),
                                     d.bj.data(), d.values.data(), 0));
  return m;
}

// write_matrix_binary (io.hpp:134-148) for the blocks held by this process
inline void write_matrix_binary(const std::string& path, const DistMatrix& m) {
  std::vector<std::int64_t> bi, bj;
  std::vector<double> vals;
  std::vector<std::pair<std::pair<std::int64_t, std::int64_t>, std::size_t>> order;
  std::vector<std::vector<double>> blocks;
  for (int r = 0; r < m.nranks(); ++r) {
    bt_mat* s = nullptr;
    if (bt_dmat_local(m.handle(), r, &s) != BT_OK) continue;
    int64_t nb = 0, ne = 0;
    detail::check(bt_mat_info(s, &nb, &ne));
    std::vector<std::int64_t> i(nb), j(nb);
    std::vector<double> v(ne);
    detail::check(bt_mat_export(s, i.data(), j.data(), v.data()));
    std::size_t off = 0;
    for (int64_t t = 0; t < nb; ++t) {
      const std::size_t n = std::size_t(m.rows().size(i[t])) * m.cols().size(j[t]);
      order.push_back({{i[t], j[t]}, blocks.size()});
      blocks.emplace_back(v.begin() + off, v.begin() + off + n);
      off += n;
    }
  }
  std::sort(order.begin(), order.end());
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw error("cannot open " + path + " for writing");
  detail::wr64(f, m.rows().total_elements());
  detail::wr64(f, m.cols().total_elements());
  detail::wr64(f, m.n_block_rows());
  detail::wr64(f, m.n_block_cols());
  for (std::int64_t b = 0; b < m.n_block_rows(); ++b) detail::wr64(f, m.rows().size(b));
  for (std::int64_t b = 0; b < m.n_block_cols(); ++b) detail::wr64(f, m.cols().size(b));
  for (const auto& o : order) {
    detail::wr64(f, o.first.first);
    detail::wr64(f, o.first.second);
    for (double v : blocks[o.second]) {
      std::uint64_t u;
      std::memcpy(&u, &v, 8);
      detail::wr64(f, u);
    }
  }
  std::fclose(f);
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
// multiply on s.nprocs B200s (mirror of dist.py predicted_time_b200).  Cannon
// overlaps its shifts with the local multiply (square grids only); case 1's C
// reduction follows the multiply; case 2's B gather is half hidden behind the
// symbolic passes.
struct B200Machine {
  double fp64_flops = 26e12;  // k_smm_dmma useful FP64, c1
  double link_bytes = 770e9;  // NVLink peer copy per direction
  double hbm_bytes = 6.55e12; // HBM copy
};
inline double predicted_time_b200(Algorithm algo, const MultiplySpec& s,
                                  const B200Machine& hw = B200Machine{}) {
  s.validate();
  const double p = s.nprocs;
  const double flops = 2.0 * s.m * s.n * s.k * s.occ_a * s.occ_b;
  const double compute = flops / (p * hw.fp64_flops) + 8.0 * s.stored_c() / p / hw.hbm_bytes;
  switch (algo) {
    case Algorithm::cannon: {
      const double q = std::round(std::sqrt(p));
      if (q * q != p) return std::numeric_limits<double>::infinity();
      return std::max(compute, 8.0 * cannon_volume(s) / hw.link_bytes);
    }
    case Algorithm::case1: return compute + 8.0 * case1_volume(s) / hw.link_bytes;
    case Algorithm::case2: return compute + 0.5 * 8.0 * case2_volume(s) / hw.link_bytes;
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
