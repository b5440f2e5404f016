// Example caller of the facade's tensor module: the RPA-like
// rank-3 contraction R_(ab)Q = sum_P T_(ab)P * M_PQ of BASELINE config 4 at a
// small size, with T stored under a map that needs a device remap first.
// Checks C against a dense host evaluation and prints the Frobenius-relative
// error; exit code 0 iff it is <= 1e-12.
#include <cmath>
#include <cstdio>
#include <random>

#include "blocktensor/b200.hpp"

using namespace blocktensor;

int main() {
  try {
    SimComm comm(ProcessGrid({1}));
    const Blocking ao({13, 23, 13, 23, 13}), aux({13, 23, 13, 23, 13, 23});
    // T(a,b,P) stored as rows (a) x cols (b,P): not the contraction map
    SparseTensor T(comm, {ao, ao, aux}, {0}, {1, 2});
    SparseTensor M(comm, {aux, aux}, {0}, {1});
    SparseTensor R(comm, {ao, ao, aux}, {0, 1}, {2});
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd(0.0, 1.0);
    std::uniform_real_distribution<double> ud(0.0, 1.0);
    const int na = 5, np = 6;
    // dense host copies for the check
    const int A = static_cast<int>(ao.total()), P = static_cast<int>(aux.total());
    std::vector<double> dT(static_cast<size_t>(A) * A * P, 0.0), dM(static_cast<size_t>(P) * P, 0.0);
    for (int a = 0; a < na; ++a)
      for (int b = 0; b < na; ++b)
        for (int p = 0; p < np; ++p) {
          if (ud(rng) > 0.3) continue;
          const int sa = ao.size(a), sb = ao.size(b), sp = aux.size(p);
          std::vector<double> v(static_cast<size_t>(sa) * sb * sp);
          for (auto& x : v) x = nd(rng);
          T.put_block({a, b, p}, v);
          for (int i = 0; i < sa; ++i)
            for (int j = 0; j < sb; ++j)
              for (int k = 0; k < sp; ++k)
                dT[(static_cast<size_t>(ao.offset(a) + i) * A + ao.offset(b) + j) * P +
                   aux.offset(p) + k] = v[(static_cast<size_t>(i) * sb + j) * sp + k];
        }
    for (int p = 0; p < np; ++p)
      for (int q = 0; q < np; ++q) {
        if (std::abs(p - q) > 1) continue;  // banded (P|Q)
        const int sp = aux.size(p), sq = aux.size(q);
        std::vector<double> v(static_cast<size_t>(sp) * sq);
        for (auto& x : v) x = nd(rng);
        M.put_block({p, q}, v);
        for (int i = 0; i < sp; ++i)
          for (int j = 0; j < sq; ++j)
            dM[static_cast<size_t>(aux.offset(p) + i) * P + aux.offset(q) + j] =
                v[static_cast<size_t>(i) * sq + j];
      }
    contract(comm, T, M, {2}, {0}, R);
    // dense reference and comparison
    double num = 0.0, den = 0.0;
    for (int a = 0; a < na; ++a)
      for (int b = 0; b < na; ++b)
        for (int q = 0; q < np; ++q) {
          std::vector<double> got;
          const bool found = R.get_block({a, b, q}, got);
          const int sa = ao.size(a), sb = ao.size(b), sq = aux.size(q);
          for (int i = 0; i < sa; ++i)
            for (int j = 0; j < sb; ++j)
              for (int k = 0; k < sq; ++k) {
                double want = 0.0;
                const size_t ab = static_cast<size_t>(ao.offset(a) + i) * A + ao.offset(b) + j;
                for (int p = 0; p < P; ++p)
                  want += dT[ab * P + p] * dM[static_cast<size_t>(p) * P + aux.offset(q) + k];
                const double g = found ? got[(static_cast<size_t>(i) * sb + j) * sq + k] : 0.0;
                num += (g - want) * (g - want);
                den += want * want;
              }
        }
    const double err = den > 0 ? std::sqrt(num / den) : std::sqrt(num);
    std::printf("contract (ab|P)(P|Q): frobenius rel err %.3e\n", err);
    return err <= 1e-12 ? 0 : 2;
  } catch (const error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
