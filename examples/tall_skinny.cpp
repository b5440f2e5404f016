// tall_skinny.cpp -- the tall-and-skinny layer through the
// facade: C (M x N) += A (M x K) * B (K x N) with K split into f subgroups.
//
//   tall_skinny <f> <sub_grid rows> <sub_grid cols> A.bin B.bin Cout.bin
//
// Parent group: P = f * sub_grid ranks; C on a round-robin grid of the parent
// (2x2 for P = 4, P x 1 otherwise).  One process: virtual ranks, subgroups run
// one after another; under torchrun (WORLD_SIZE = P): one rank per GPU, the
// subgroups are NCCL communicators split from the parent and multiply
// concurrently.  Cout.bin (.rank<r> under torchrun) holds this process's C
// blocks.  Also prints the index-memory property for a 10^4-block split
// dimension: host index entries along it (0: functional axes) and the longest
// device index range (one submatrix).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <thread>

#include "blocktensor/b200.hpp"

using namespace blocktensor;

static int env_int(const char* k, int d) {
  const char* v = std::getenv(k);
  return v && *v ? std::atoi(v) : d;
}

static NcclId exchange_id(int rank) {
  const char* f = std::getenv("BT_NCCL_ID_FILE");
  const std::string path = f && *f ? f : "/tmp/bt_nccl_id_ts";
  NcclId id;
  if (rank == 0) {
    id = NcclId::create();
    const std::string tmp = path + ".tmp";
    std::ofstream(tmp, std::ios::binary).write(reinterpret_cast<const char*>(id.bytes), 128);
    std::rename(tmp.c_str(), path.c_str());
    return id;
  }
  for (int t = 0; t < 6000; ++t) {
    std::ifstream is(path, std::ios::binary);
    if (is && is.read(reinterpret_cast<char*>(id.bytes), 128)) return id;
    std::this_thread::sleep_for(std::chrono::milliseconds(10));
  }
  throw error("timed out waiting for the NCCL id");
}

static IndexFuncs funcs_of(const Blocking& b, int extent) {
  return IndexFuncs{b.n_blocks(), [b](std::int64_t i) { return b.size(i); },
                    [extent](std::int64_t i) { return static_cast<int>(i % extent); }};
}

int main(int argc, char** argv) {
  if (argc != 7) {
    std::fprintf(stderr, "usage: %s f sub_rows sub_cols A B Cout\n", argv[0]);
    return 2;
  }
  const int f = std::stoi(argv[1]);
  const ProcessGrid sub({std::stoi(argv[2]), std::stoi(argv[3])});
  const int P = f * sub.size();
  const int world = env_int("WORLD_SIZE", 1), rank = env_int("RANK", 0);
  try {
    std::unique_ptr<SimComm> parent;
    if (world > 1) {
      if (world != P) throw invalid_argument("WORLD_SIZE must equal f * sub_grid size");
      parent.reset(new SimComm(ProcessGrid({P}), env_int("LOCAL_RANK", 0), rank, exchange_id(rank)));
    } else {
      parent.reset(new SimComm(ProcessGrid({P})));
    }
    Subgroups groups(*parent, f, sub);
    MatrixData A = read_matrix_file(argv[4], FileFormat::binary);
    MatrixData B = read_matrix_file(argv[5], FileFormat::binary);
    TallSkinnyMatrix ta(groups, funcs_of(A.rows, sub.dim(0)), funcs_of(A.cols, sub.dim(1)),
                        SplitDim::cols);
    TallSkinnyMatrix tb(groups, funcs_of(B.rows, sub.dim(0)), funcs_of(B.cols, sub.dim(1)),
                        SplitDim::rows);
    for (auto& t : A.blocks) ta.put_block(std::get<0>(t), std::get<1>(t), std::get<2>(t));
    for (auto& t : B.blocks) tb.put_block(std::get<0>(t), std::get<1>(t), std::get<2>(t));
    const int q = P == 4 ? 2 : 1;
    ProcessGrid cgrid = P == 4 ? ProcessGrid({2, 2}) : ProcessGrid({P, 1});
    (void)q;
    DistMatrix c = new_matrix_round_robin(A.rows, B.cols, cgrid);
    parent->reset_ledger();
    multiply_tall_skinny(ta, tb, c);
    const std::string out = world > 1 ? std::string(argv[6]) + ".rank" + std::to_string(rank)
                                      : std::string(argv[6]);
    write_matrix_file(out, c, FileFormat::binary);
    std::int64_t reduce_sent = 0;
    for (int r : parent->local_ranks())
      reduce_sent += parent->ledger().rank_phase(r, "ts_reduce").elements_sent;
    // memory property: a 10^4-block split dimension
    IndexFuncs longk{10000, [](std::int64_t) { return 4; }, [](std::int64_t i) { return int(i % 7); }};
    IndexFuncs shortm{8, [](std::int64_t) { return 4; }, [](std::int64_t i) { return int(i); }};
    TallSkinnyMatrix big(groups, shortm, longk, SplitDim::cols);
    std::printf("rank %d: subgroups %zu local, C local blocks %lld, ts_reduce elements sent %lld, "
                "host index entries %lld, max device index range %lld of 10000\n",
                rank, groups.local().size(), static_cast<long long>(c.local(rank).stored_blocks()),
                static_cast<long long>(reduce_sent),
                static_cast<long long>(big.host_index_entries()),
                static_cast<long long>(big.max_device_index_range()));
  } catch (const error& e) {
    std::fprintf(stderr, "blocktensor error: %s\n", e.what());
    return 1;
  }
  return 0;
}
