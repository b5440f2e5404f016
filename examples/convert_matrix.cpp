// convert_matrix.cpp -- fixture I/O through the facade (io.hpp signatures):
//   convert_matrix <in> <text|binary> <out> <text|binary>
// read_matrix_file -> to_dist_matrix (device) -> write_matrix_file.
#include <cstdio>
#include <string>

#include "blocktensor/b200.hpp"

using namespace blocktensor;

static FileFormat fmt(const std::string& s) {
  return s == "text" ? FileFormat::text : FileFormat::binary;
}

int main(int argc, char** argv) {
  if (argc != 5) {
    std::fprintf(stderr, "usage: %s in fmt out fmt\n", argv[0]);
    return 2;
  }
  try {
    SimComm comm(ProcessGrid({1}));
    DistMatrix m = to_dist_matrix(read_matrix_file(argv[1], fmt(argv[2])), ProcessGrid({1, 1}));
    write_matrix_file(argv[3], m, fmt(argv[4]));
  } catch (const error& e) {
    std::fprintf(stderr, "blocktensor error: %s\n", e.what());
    return 1;
  }
  return 0;
}
