// ref_shim.cpp -- extern "C" shim that compiles the UNMODIFIED reference headers
// from /root/reference/proj/include (and tests/support/oracles.hpp) into
// oracle/_ref/libbtref.so.  TEST INFRASTRUCTURE ONLY: used by tests/ to pin the
// oracle restatement and by bench.py --impl reference / cpu_baseline to time the
// reference's own CPU path.  No reference source is copied into this repo; the
// headers are #included from /root/reference at build time (oracle/Makefile),
// with the reference's CMake Release flags (-O3 -DNDEBUG, no -march;
// proj/CMakeLists.txt:8-10).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <tuple>
#include <vector>

#include "blocktensor/cost_model.hpp"
#include "blocktensor/io.hpp"
#include "blocktensor/matrix.hpp"
#include "blocktensor/multiply_cannon.hpp"
#include "blocktensor/multiply_rect.hpp"
#include "blocktensor/random.hpp"
#include "support/oracles.hpp"

using namespace blocktensor;

namespace {

thread_local std::string g_err;

struct Result {
  std::vector<std::int64_t> bi, bj;
  std::vector<double> vals;
  double seconds = 0;
  Ledger ledger;
  int nranks = 0;
};

Blocking make_blocking(std::int64_t n, const std::int32_t* sz) {
  return Blocking(std::vector<int>(sz, sz + n));
}

void fill(DistMatrix& m, std::int64_t nblk, const std::int64_t* bi, const std::int64_t* bj,
          const double* vals) {
  std::size_t v = 0;
  for (std::int64_t t = 0; t < nblk; ++t) {
    const int r = m.rows().size(bi[t]);
    const int c = m.cols().size(bj[t]);
    std::vector<double> data(vals + v, vals + v + static_cast<std::size_t>(r) * c);
    v += static_cast<std::size_t>(r) * c;
    m.put_block(bi[t], bj[t], DenseBlock(r, c, std::move(data)));
  }
}

Result* collect(const DistMatrix& c) {
  auto* res = new Result;
  std::vector<std::tuple<std::int64_t, std::int64_t, const DenseBlock*>> all;
  c.for_each_global([&](int, std::int64_t i, std::int64_t j, const DenseBlock& b) {
    all.emplace_back(i, j, &b);
  });
  std::sort(all.begin(), all.end(), [](const auto& x, const auto& y) {
    return std::pair(std::get<0>(x), std::get<1>(x)) < std::pair(std::get<0>(y), std::get<1>(y));
  });
  for (auto& [i, j, b] : all) {
    res->bi.push_back(i);
    res->bj.push_back(j);
    res->vals.insert(res->vals.end(), b->values.begin(), b->values.end());
  }
  return res;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// block_gemm_acc (block.hpp:45-60) on caller buffers.
int ref_block_gemm_acc(double* c, const double* a, const double* b, int m, int n, int k) {
  try {
    DenseBlock cb(m, n, std::vector<double>(c, c + static_cast<std::size_t>(m) * n));
    DenseBlock ab(m, k, std::vector<double>(a, a + static_cast<std::size_t>(m) * k));
    DenseBlock bb(k, n, std::vector<double>(b, b + static_cast<std::size_t>(k) * n));
    block_gemm_acc(cb, ab, bb);
    std::memcpy(c, cb.values.data(), sizeof(double) * cb.values.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// testsupport::random_matrix (oracles.hpp:74-85) on a 1x1 grid, canonical export.
void* ref_random_matrix(std::uint64_t seed, std::int64_t nbr, const std::int32_t* rsz,
                        std::int64_t nbc, const std::int32_t* csz, double occ) {
  try {
    Rng rng(seed);
    auto m = testsupport::random_matrix(rng, make_blocking(nbr, rsz), make_blocking(nbc, csz),
                                        ProcessGrid({1, 1}), occ);
    return collect(m);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// Runs multiply_dispatch (multiply_rect.hpp:242-250) with algo 0 = cannon
// (on a grid_q x grid_q grid), 1 = case1, 2 = case2 (linear grid of nprocs).
// Operands are created round-robin on the q x q grid (new_matrix_round_robin,
// matrix.hpp:413-418).  schedule 0 = parallel threads, 1 = sequential.
void* ref_multiply(int algo, int grid_q, int nprocs, int schedule, std::int64_t m_nb,
                   const std::int32_t* m_sz, std::int64_t k_nb, const std::int32_t* k_sz,
                   std::int64_t n_nb, const std::int32_t* n_sz, std::int64_t a_nblk,
                   const std::int64_t* a_i, const std::int64_t* a_j, const double* a_v,
                   std::int64_t b_nblk, const std::int64_t* b_i, const std::int64_t* b_j,
                   const double* b_v, std::int64_t c_nblk, const std::int64_t* c_i,
                   const std::int64_t* c_j, const double* c_v) {
  try {
    ProcessGrid grid({grid_q, grid_q});
    Blocking mb = make_blocking(m_nb, m_sz), kb = make_blocking(k_nb, k_sz),
             nb = make_blocking(n_nb, n_sz);
    DistMatrix a = new_matrix_round_robin(mb, kb, grid);
    DistMatrix b = new_matrix_round_robin(kb, nb, grid);
    DistMatrix c = new_matrix_round_robin(mb, nb, grid);
    fill(a, a_nblk, a_i, a_j, a_v);
    fill(b, b_nblk, b_i, b_j, b_v);
    fill(c, c_nblk, c_i, c_j, c_v);
    const int world = std::max(grid.size(), algo == 0 ? 1 : nprocs);
    SimComm comm(ProcessGrid({world}), schedule ? Schedule::sequential : Schedule::parallel);
    const Algorithm al = algo == 0 ? Algorithm::cannon : algo == 1 ? Algorithm::case1
                                                                   : Algorithm::case2;
    auto t0 = std::chrono::steady_clock::now();
    multiply_dispatch(comm, al, a, b, c, nprocs);
    auto t1 = std::chrono::steady_clock::now();
    Result* res = collect(c);
    res->seconds = std::chrono::duration<double>(t1 - t0).count();
    res->ledger = comm.ledger();
    res->nranks = world;
    return res;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

std::int64_t ref_res_nblk(void* h) { return static_cast<std::int64_t>(static_cast<Result*>(h)->bi.size()); }
std::int64_t ref_res_nvals(void* h) { return static_cast<std::int64_t>(static_cast<Result*>(h)->vals.size()); }
double ref_res_seconds(void* h) { return static_cast<Result*>(h)->seconds; }
int ref_res_nranks(void* h) { return static_cast<Result*>(h)->nranks; }
void ref_res_copy(void* h, std::int64_t* bi, std::int64_t* bj, double* vals) {
  auto* r = static_cast<Result*>(h);
  std::copy(r->bi.begin(), r->bi.end(), bi);
  std::copy(r->bj.begin(), r->bj.end(), bj);
  std::copy(r->vals.begin(), r->vals.end(), vals);
}
// what: 0 elements_sent, 1 elements_received, 2 meta_sent, 3 meta_received.
// phase == nullptr or "" gives the rank total.
std::int64_t ref_res_ledger(void* h, int rank, const char* phase, int what) {
  auto* r = static_cast<Result*>(h);
  TrafficCounters t = (phase && *phase) ? r->ledger.rank_phase(rank, phase)
                                        : r->ledger.rank_total(rank);
  switch (what) {
    case 0: return t.elements_sent;
    case 1: return t.elements_received;
    case 2: return t.meta_sent;
    default: return t.meta_received;
  }
}
void ref_res_free(void* h) { delete static_cast<Result*>(h); }

// cost model (cost_model.hpp:43-88) and selector (multiply_rect.hpp:45-63)
double ref_cost(int which, double m, double n, double k, double oa, double ob, double oc,
                double p) {
  MultiplySpec s;
  s.m = m; s.n = n; s.k = k; s.occ_a = oa; s.occ_b = ob; s.occ_c = oc; s.nprocs = p;
  try {
    switch (which) {
      case 0: return cannon_volume(s);
      case 1: return case1_volume(s);
      case 2: return case2_volume(s);
      case 3: return occupancy_limit_case1(s);
      case 4: return occupancy_ratio_bound(m, n, k, p);
      case 5: return static_cast<double>(select_algorithm(m, n, k, oa, ob, oc, p));
      default: return estimate_result_occupancy(oa, ob, static_cast<std::int64_t>(k));
    }
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

// Fixture I/O through the reference's own io.hpp (write_matrix_file /
// read_matrix_file): pins the facade's readers and writers byte for byte.
// fmt: 0 text, 1 binary.
int ref_io_write(const char* path, int fmt, std::int64_t nbr, const std::int32_t* rsz,
                 std::int64_t nbc, const std::int32_t* csz, std::int64_t nblk,
                 const std::int64_t* bi, const std::int64_t* bj, const double* vals) {
  try {
    ProcessGrid grid({1, 1});
    DistMatrix m = new_matrix_round_robin(make_blocking(nbr, rsz), make_blocking(nbc, csz), grid);
    fill(m, nblk, bi, bj, vals);
    write_matrix_file(path, m, fmt ? FileFormat::binary : FileFormat::text);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

void* ref_io_read(const char* path, int fmt) {
  try {
    MatrixData d = read_matrix_file(path, fmt ? FileFormat::binary : FileFormat::text);
    DistMatrix m = to_dist_matrix(std::move(d), ProcessGrid({1, 1}));
    return collect(m);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

}  // extern "C"
