// multiply_files.cpp -- a caller written against the reference API, compiled
// against the B200 facade instead (include/blocktensor/b200.hpp).
//   multiply_files <algo: cannon|case1|case2> <grid q> <nprocs> A.bin B.bin C.bin Cout.bin
// Files use the reference's binary matrix format (io.hpp:132-178).
#include <cstdio>
#include <string>

#include "blocktensor/b200.hpp"

using namespace blocktensor;

int main(int argc, char** argv) {
  if (argc != 8) {
    std::fprintf(stderr, "usage: %s algo q nprocs A B C Cout\n", argv[0]);
    return 2;
  }
  const std::string algo = argv[1];
  const int q = std::stoi(argv[2]), nprocs = std::stoi(argv[3]);
  try {
    ProcessGrid grid({q, q});
    SimComm comm(ProcessGrid({std::max(q * q, nprocs)}));
    DistMatrix a = to_dist_matrix(read_matrix_binary(argv[4]), grid);
    DistMatrix b = to_dist_matrix(read_matrix_binary(argv[5]), grid);
    DistMatrix c = to_dist_matrix(read_matrix_binary(argv[6]), grid);
    const Algorithm al = algo == "cannon" ? Algorithm::cannon
                         : algo == "case1" ? Algorithm::case1 : Algorithm::case2;
    multiply_dispatch(comm, al, a, b, c, nprocs);
    write_matrix_binary(argv[7], c);
    std::printf("%s: C has %lld blocks, mean elements sent per rank %.1f\n", algo.c_str(),
                static_cast<long long>(c.stored_blocks()), comm.ledger().mean_elements_sent());
  } catch (const error& e) {
    std::fprintf(stderr, "blocktensor error: %s\n", e.what());
    return 1;
  }
  return 0;
}
