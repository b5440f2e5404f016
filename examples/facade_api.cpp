// facade_api.cpp -- the reference matrix API surface beyond multiply, through
// the facade: Axis::functional (matrix.hpp:50-58), DistMatrix::local /
// LocalStore::for_each (matrix.hpp:199-205, 294-295), put_block_at /
// get_block_at ownership checks (matrix.hpp:312-334), for_each_global,
// redistribute (+transpose) / redistribute_add (matrix.hpp:567-622) with the
// ledger.  Prints one line per check; exit 0 iff all pass.
#include <cmath>
#include <cstdio>
#include <map>
#include <string>

#include "blocktensor/b200.hpp"

using namespace blocktensor;

static int failures = 0;
static void check(bool ok, const std::string& what) {
  std::printf("%s: %s\n", ok ? "OK" : "FAIL", what.c_str());
  if (!ok) ++failures;
}

int main() {
  try {
    ProcessGrid grid({2, 2});
    SimComm comm(grid);
    const std::int64_t nb = 12;
    auto size_fn = [](std::int64_t b) { return static_cast<int>(3 + (b * 7) % 5); };
    auto dist_fn = [](std::int64_t b) { return static_cast<int>((b / 3) % 2); };
    Axis rows = Axis::functional(nb, size_fn, dist_fn, 2);
    Axis cols = Axis::functional(nb, size_fn, [](std::int64_t b) { return static_cast<int>(b % 2); }, 2);
    check(rows.index_entries() == 0 && !rows.is_explicit(), "functional axis keeps no host index");
    DistMatrix a(rows, cols, grid);
    std::map<std::pair<std::int64_t, std::int64_t>, DenseBlock> want;
    for (std::int64_t i = 0; i < nb; ++i)
      for (std::int64_t j = 0; j < nb; ++j) {
        if ((i * 5 + j * 3) % 4 != 0) continue;
        DenseBlock b(size_fn(i), size_fn(j));
        for (int t = 0; t < b.rows * b.cols; ++t) b.values[t] = std::sin(1.0 + i * 100 + j + t * 0.01);
        const int owner = a.owner_rank(i, j);
        bool threw = false;
        try {
          a.put_block_at((owner + 1) % 4, i, j, b);
        } catch (const ownership_error&) {
          threw = true;
        }
        if (!threw) check(false, "put_block_at on a foreign rank must throw ownership_error");
        a.put_block_at(owner, i, j, b);
        want[{i, j}] = b;
      }
    // local stores hold exactly their owned blocks, in (row, col) order
    std::size_t seen = 0;
    bool owners_ok = true, order_ok = true, values_ok = true;
    for (int r = 0; r < 4; ++r) {
      std::int64_t pi = -1, pj = -1;
      a.local(r).for_each([&](std::int64_t i, std::int64_t j, const DenseBlock& b) {
        ++seen;
        if (a.owner_rank(i, j) != r) owners_ok = false;
        if (i < pi || (i == pi && j <= pj)) order_ok = false;
        pi = i;
        pj = j;
        if (!(b == want[{i, j}])) values_ok = false;
      });
    }
    check(seen == want.size() && owners_ok, "every block stored by its owner");
    check(order_ok && values_ok, "LocalStore::for_each visits (row, col) order, exact values");
    std::size_t g = 0;
    a.for_each_global([&](int r, std::int64_t i, std::int64_t j, const DenseBlock&) {
      g += a.owner_rank(i, j) == r;
    });
    check(g == want.size(), "for_each_global visits every block once");
    bool threw = false;
    try {
      auto it = want.begin();
      a.get_block_at((a.owner_rank(it->first.first, it->first.second) + 1) % 4, it->first.first,
                     it->first.second);
    } catch (const ownership_error&) {
      threw = true;
    }
    check(threw, "get_block_at on a foreign rank throws ownership_error");

    // redistribute (transpose) onto a 1 x 4 grid, then back with redistribute_add
    comm.reset_ledger();
    ProcessGrid g14({1, 4});
    DistMatrix t = redistribute(comm, a, Axis::round_robin(cols.blocking(), 1),
                                Axis::round_robin(rows.blocking(), 4), g14, true, "to_t");
    bool tr_ok = true;
    for (const auto& kv : want) {
      const DenseBlock* b = t.get_block(kv.first.second, kv.first.first);
      if (!b) { tr_ok = false; continue; }
      for (int r = 0; r < kv.second.rows; ++r)
        for (int c = 0; c < kv.second.cols; ++c)
          if (b->at(c, r) != kv.second.at(r, c)) tr_ok = false;
    }
    check(tr_ok && t.stored_blocks() == static_cast<std::int64_t>(want.size()),
          "redistribute(transpose) moves every block, transposed");
    const std::int64_t sent = comm.ledger().total_elements_sent();
    check(sent > 0 && sent <= a.stored_elements(), "ledger charges only blocks that change ranks");
    DistMatrix back = redistribute(comm, t, Axis::round_robin(rows.blocking(), 2),
                                   Axis::round_robin(cols.blocking(), 2), grid, true, "back");
    redistribute_add(comm, a, back, "add");   // back = 2 a
    bool add_ok = true;
    for (const auto& kv : want) {
      const DenseBlock* b = back.get_block(kv.first.first, kv.first.second);
      if (!b) { add_ok = false; continue; }
      for (std::size_t q = 0; q < b->values.size(); ++q)
        if (b->values[q] != 2.0 * kv.second.values[q]) add_ok = false;
    }
    check(add_ok, "redistribute_add accumulates into existing blocks (exactly 2a)");
    check(comm.ledger().rank_phase(0, "add").elements_sent >= 0, "ledger phases by name");
  } catch (const error& e) {
    std::printf("FAIL: blocktensor error: %s\n", e.what());
    return 1;
  }
  return failures ? 1 : 0;
}
