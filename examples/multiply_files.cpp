// multiply_files.cpp -- a caller written against the reference API, compiled
// against the B200 facade instead (include/blocktensor/b200.hpp).
//
//   multiply_files <cannon|case1|case2|auto> <grid q> <nprocs> A B C Cout [text|binary]
//
// Fixtures in the reference's formats (io.hpp:22-198, default binary).
// One process: every rank is a virtual rank on this process's GPU.  Under
// torchrun (WORLD_SIZE > 1): one rank per process and GPU over NCCL -- rank 0
// creates the NCCL id and hands it over through a file (BT_NCCL_ID_FILE), every
// process reads the inputs and keeps its own blocks, multiplies, and writes
// the C blocks of its rank to Cout.rank<r> (same format).
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

// rank 0 writes the id atomically (tmp + rename), the others wait for it
static NcclId exchange_id(int rank) {
  const char* f = std::getenv("BT_NCCL_ID_FILE");
  const std::string path = f && *f ? f : "/tmp/bt_nccl_id_" + std::to_string(env_int("MASTER_PORT", 0));
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
  throw error("timed out waiting for the NCCL id in " + path);
}

int main(int argc, char** argv) {
  if (argc != 8 && argc != 9) {
    std::fprintf(stderr, "usage: %s algo q nprocs A B C Cout [text|binary]\n", argv[0]);
    return 2;
  }
  const std::string algo = argv[1];
  const int q = std::stoi(argv[2]), nprocs = std::stoi(argv[3]);
  const FileFormat fmt =
      argc == 9 && std::string(argv[8]) == "text" ? FileFormat::text : FileFormat::binary;
  const int world = env_int("WORLD_SIZE", 1), rank = env_int("RANK", 0);
  try {
    ProcessGrid grid({q, q});
    std::unique_ptr<SimComm> comm;
    if (world > 1)
      comm.reset(new SimComm(ProcessGrid({world}), env_int("LOCAL_RANK", 0), rank,
                             exchange_id(rank)));
    else
      comm.reset(new SimComm(ProcessGrid({std::max(q * q, nprocs)})));
    DistMatrix a = to_dist_matrix(read_matrix_file(argv[4], fmt), grid);
    DistMatrix b = to_dist_matrix(read_matrix_file(argv[5], fmt), grid);
    DistMatrix c = to_dist_matrix(read_matrix_file(argv[6], fmt), grid);
    if (algo == "auto") {
      const Algorithm al = multiply_auto(*comm, a, b, c, nprocs);
      std::printf("auto selected %s\n", algorithm_name(al));
    } else {
      const Algorithm al = algo == "cannon" ? Algorithm::cannon
                           : algo == "case1" ? Algorithm::case1 : Algorithm::case2;
      multiply_dispatch(*comm, al, a, b, c, nprocs);
    }
    const std::string out = world > 1 ? std::string(argv[7]) + ".rank" + std::to_string(rank)
                                      : std::string(argv[7]);
    write_matrix_file(out, c, fmt);
    std::printf("%s rank %d/%d: C has %lld local blocks, elements sent by rank %d: %lld\n",
                algo.c_str(), rank, world, static_cast<long long>(c.stored_blocks()), rank,
                static_cast<long long>(comm->ledger().rank_total(rank).elements_sent));
  } catch (const error& e) {
    std::fprintf(stderr, "blocktensor error: %s\n", e.what());
    return 1;
  }
  return 0;
}
