// bt_smm.cuh -- the libsmm_acc-equivalent small-GEMM family for sm_100a (FP64).
//
// Reference op: block_gemm_acc (block.hpp:45-60), c += a*b over a batch ordered
// by (row, col, k) (order_batches, block.hpp:112-118).
//
// Data path:
//  * Operands live in the native T8 layout (bt_internal.cuh): zero-padded 8x8
//    swizzled tiles, so A-role (8x4) and B-role (4x8) fragment reads from
//    shared memory are bank-conflict free and need no k-masking, and C tiles
//    are read/written as coalesced 16-byte pairs.
//  * Each product is a (A slab, B block) pair moved by the bulk-async copy engine
//    (cp.async.bulk, TMA 1D) into a per-warp ring of shared-memory stages that
//    complete on mbarriers; the producer runs `stages` products ahead.
//  * One warp owns one C tile (<= 32 x 32) for its whole product chain: the
//    accumulators stay in registers, C is read (C_in) and written exactly once.
//  * Warps pull C tiles from a global atomic counter over an L2-friendly band
//    order.
#pragma once

#include <type_traits>

#include "bt_internal.cuh"
#include "bt_ptx.cuh"

namespace bt {

// One C tile of work: rows [r0, r0 + rows) x columns [c0, c0 + 32) of C block
// (i, j) (c0 = 0 and all columns unless the block is wider than 32).  32 bytes.
struct Item {
  int64_t c_off;    // element offset of the tile's first 8x8 tile in the C_out slab
  int64_t cin_off;  // same for C_in, or -1
  int64_t p0r8;     // first product (bits 0-43) | r0 / 8 (bits 44-56) | c0 / 8 (bits 57-63)
  int32_t np;       // number of products
  int16_t rows;     // rows in this tile (<= TM)
  int16_t n;        // C block columns (the block's, not the tile's)
};
constexpr int kItemP0Bits = 44;
constexpr int kItemMaxR8 = (1 << 13) - 1;  // rows of a block <= 65 528
constexpr int kItemMaxC8 = (1 << 7) - 1;   // columns of a wide block <= 1 016
__host__ __device__ inline int64_t item_pack(int64_t p0, int r8, int c8) {
  return p0 | (static_cast<int64_t>(r8) << kItemP0Bits) | (static_cast<int64_t>(c8) << 57);
}

// Product descriptor: offsets of the A and B blocks in units of one 8x8 tile
// (64 doubles) and the number of 4-wide k chunks.
using Desc = int4;  // {a_unit, b_unit, kc, 0}

struct NumArgs {
  const Item* items;
  int64_t item_lo;
  int64_t nitems;
  unsigned long long* counter;
  const Desc* desc;
  const double* at;  // A values (T8)
  const double* bt;  // B values (T8)
  const double* cin;
  double* cout;
  int stages;
  int stage_doubles;  // per-stage shared memory in doubles
  int a_region;       // doubles of the A part of a stage
  // K panels in one launch (npanels > 1): ticket t is item t % nitems of panel
  // t / nitems (items of panel p at items + p * panel_stride); panels p > 0
  // accumulate into C_out in place once tile_flag[item] says panel p - 1 of
  // the same tile has stored its C
  int npanels;
  int64_t panel_stride;
  int* tile_flag;
  // slab lengths in doubles (device checks of the checked build)
  int64_t a_len, b_len, cin_len, cout_len;
  // tickets are drawn from `counter` in batches of this many consecutive
  // items (>= 1): one global atomic per batch instead of per item
  int ticket_batch;
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__host__ __device__ __forceinline__ int64_t item_p0(const Item& it) {
  return it.p0r8 & ((int64_t(1) << kItemP0Bits) - 1);
}
__host__ __device__ __forceinline__ int item_r8(const Item& it) {
  return static_cast<int>((static_cast<uint64_t>(it.p0r8) >> kItemP0Bits) & kItemMaxR8);
}
__host__ __device__ __forceinline__ int item_c8(const Item& it) {
  return static_cast<int>((static_cast<uint64_t>(it.p0r8) >> 57) & kItemMaxC8);
}

// FP64 DMMA tile kernel: warp <-> C tile of up to TM = 8*TMT rows and exactly
// TN = 8*TNT padded columns.
//
// Warps take tickets for items of the ordered item list from a global
// counter (load balance; the warps in flight work on neighbouring C tiles).
// Producer side (lane 0 issues the bulk copies) runs `S` products ahead of the
// consumer.  All producer bookkeeping lives in shared memory and is prefetched
// with cp.async so no global-load latency sits on the DMMA critical path and
// the register budget stays small enough for 20 resident warps per SM:
//   * item structs: slot n % QN holds the n-th item of this warp; the struct of
//     item n+2 is requested when item n starts, its ticket one item earlier;
//   * product descriptors: streamed in chunks of 32 through two slots, the
//     following chunk requested when a chunk starts.
// Resident CTAs targeted by the register allocator: 5 x 4 warps for tiles up to
// 24x24 (<= 96 registers, 20 warps/SM fit the shared-memory ring), 3 for larger.
template <int TMT, int TNT>
constexpr int dmma_min_blocks() {
  return TMT * TNT <= 9 ? 5 : 3;
}
// MULTI: one launch for every DMMA class of a mixed-size multiply -- TMT x TNT
// is then the largest tile, each item's own tile shape comes from its rows and
// columns, and the consumer dispatches to the matching instantiation of the
// tile body (so small classes do not pay for the large accumulators).
// PANELS: every K panel of a single-class multiply in one launch (NumArgs
// npanels / panel_stride / tile_flag); a separate instantiation so the common
// path carries none of its bookkeeping.
// WIDE (with MULTI): blocks wider than 32 columns arrive as 32-column tiles
// (item c8: the tile's first 8-column tile; the C and B rows are strided by
// the block's tile columns) and products with more than kKTCap k tiles are
// staged in k slices of <= kKTCap tiles, each its own stage (stage_kc bit 8
// marks a product's last slice): the DMMA path then takes every block size.
constexpr int kKTCap = 4;
template <int TMT, int TNT, int WARPS, int S, bool MULTI = false, bool PANELS = false,
          bool WIDE = false>
__global__ void __launch_bounds__(WARPS * 32, (dmma_min_blocks<TMT, TNT>())) k_smm_dmma(const NumArgs g) {
  constexpr int QN = 8;     // item slots per warp
  constexpr int CTL = 1536; // control block bytes per warp
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  // per-lane T8 positions of the DMMA fragments (bt_internal.cuh layout)
  const int sw_g = ((gq >> 1) & 1) << 2;
  const int la0 = gq * 8 + (tq ^ sw_g), la1 = gq * 8 + ((4 + tq) ^ sw_g);  // A (g, 4h+t)
  const int swt = ((tq >> 1) & 1) << 2;
  const int lb0 = tq * 8 + (gq ^ swt), lb1 = (4 + tq) * 8 + (gq ^ swt);    // B (4h+t, g)
  const int lc = gq * 8 + ((2 * tq) ^ sw_g);                               // C (g, 2t..2t+1)
  // control block: mbarriers | stage kc | item slots | 2 descriptor chunks
  unsigned char* ctl = smem + wid * CTL;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ctl);
  int* stage_kc = reinterpret_cast<int*>(ctl + 64);
  Item* q_items = reinterpret_cast<Item*>(ctl + 128);
  int64_t* q_tick = reinterpret_cast<int64_t*>(ctl + 384);  // ticket of each item slot
  Desc* dring = reinterpret_cast<Desc*>(ctl + 512);  // [2][32]
  double* stages = reinterpret_cast<double*>(smem + WARPS * CTL) +
                   static_cast<int64_t>(wid) * S * g.stage_doubles;
  const Item* items = g.items + g.item_lo;
  const int64_t ntickets = PANELS ? g.nitems * g.npanels : g.nitems;
  auto item_at = [&](int64_t id) -> const Item* {
    if constexpr (!PANELS) return items + id;
    const int64_t p = id / g.nitems;
    return items + p * g.panel_stride + (id - p * g.nitems);
  };

  // ---- ticket source (lane 0): batches of TB consecutive tickets, the next
  // batch's base drawn one batch ahead so its atomic latency is hidden.  One
  // global counter hit per item was the top stall of small-block multiplies
  // (c2: 36 % of all warp stall samples on the atomicAdd, ncu).  A warp still
  // works its tickets in increasing order (the K-panel deadlock argument holds).
  const unsigned long long TB = g.ticket_batch > 1 ? static_cast<unsigned long long>(g.ticket_batch) : 1ull;
  unsigned long long b_next = 0, b_end = 0, b_pre = 0;
  // (MULTI instantiations only -- the small-block launches; single-class
  // launches keep one ticket per item and none of this state: with it the
  // c1 kernel went 0.591 -> 0.623 ms at batch 1)
  auto draw = [&]() -> unsigned long long {
    if constexpr (!MULTI) {
      return atomicAdd(g.counter, 1ull);
    } else {
      if (b_next == b_end) {
        b_next = b_pre;
        b_end = b_pre + TB;
        b_pre = atomicAdd(g.counter, TB);
      }
      return b_next++;
    }
  };
  // ---- prologue: tickets for items 0 and 1, their structs, ticket for item 2
  unsigned long long tk = 0;  // lane 0: ticket of the item two ahead
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    if constexpr (MULTI) b_pre = atomicAdd(g.counter, TB);
    for (int n = 0; n < 2; ++n) {
      const unsigned long long id = draw();
      if (static_cast<int64_t>(id) < ntickets) {
        const Item* src = item_at(static_cast<int64_t>(id));
        cp_async16(&q_items[n], src);
        cp_async16(reinterpret_cast<char*>(&q_items[n]) + 16,
                   reinterpret_cast<const char*>(src) + 16);
        if constexpr (PANELS) q_tick[n] = static_cast<int64_t>(id);
      } else {
        q_items[n].np = -1;  // end of work
      }
    }
    tk = draw();
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncwarp();

  // descriptor chunk streaming
  int cs = 0;                  // slot of the chunk being issued from
  int64_t c_base = -1;         // global desc index of dring[cs][0]
  int pf_n = -1;               // prefetched chunk in dring[cs ^ 1]: item seq and offset
  int64_t pf_base = -1;
  auto load_chunk = [&](int slot, int64_t base, int cnt) {
    if (lane < cnt) cp_async16(&dring[slot * 32 + lane], &g.desc[base + lane]);
  };

  uint32_t issued = 0, consumed = 0;
  int s_issue = 0, s_cons = 0;
  uint32_t cons_phase = 0;
  int qh = 0, qt = 0;  // consumer / producer item sequence numbers
  int64_t p_pos = 0, p_end = 0;
  int p_r8 = 0, p_mt = 0;
  int p_nt = TNT;  // B tile columns of the item being issued (MULTI: per item)
  // WIDE: the block's tile columns, the tile's first tile column, the stage's
  // B row stride (the tile body's CN), the k slice of the product being issued
  int p_ntf = TNT, p_c8 = 0, p_cs = TNT, p_sub = 0;
  bool p_more = true;

  // next chunk after (item seq n, desc index pos) -- returns false if unknown yet
  auto following = [&](int n, int64_t pos, int64_t end, int& fn, int64_t& fbase, int& fcnt) {
    if (pos + 32 < end) {
      fn = n;
      fbase = pos + 32;
      fcnt = static_cast<int>(end - fbase < 32 ? end - fbase : 32);
      return true;
    }
    const Item& nx = q_items[(n + 1) % QN];
    if (nx.np <= 0) return false;
    fn = n + 1;
    fbase = item_p0(nx);
    fcnt = min(32, nx.np);
    return true;
  };
  // cp.async groups of the bookkeeping, oldest first: ... the prefetched
  // descriptor chunk, then (at an item start) the struct request of the item
  // two ahead.  Entering a prefetched chunk waits for all but that last
  // request: a full wait there stalled every item start for one global-memory
  // round trip on the request just issued (c2: ~1 product per item).
  bool struct_pending = false;  // a struct request was committed after the prefetch
  // make dring[cs] hold the chunk starting at `pos` of item seq n
  auto enter_chunk = [&](int n, int64_t pos, int64_t end) {
    bool prefetched = pf_base == pos && pf_n == n;
    if (prefetched) {
      cs ^= 1;
    } else {     // slow path: load now
      load_chunk(cs ^ 1, pos, static_cast<int>(end - pos < 32 ? end - pos : 32));
      cs ^= 1;
      cp_async_commit();
    }
    c_base = pos;
    int fn;
    int64_t fb;
    int fc;
    // (PANELS launches keep the full wait: measured 1.3 % slower on c3 without)
    if (!PANELS && prefetched && struct_pending)
      cp_async_wait_but_last();
    else
      cp_async_wait_all();
    struct_pending = false;
    __syncwarp();
    if (following(n, pos, end, fn, fb, fc)) {
      load_chunk(cs ^ 1, fb, fc);
      pf_n = fn;
      pf_base = fb;
    } else {
      pf_n = -1;
      pf_base = -1;
    }
    cp_async_commit();
  };

  auto top_up = [&]() {
    while (issued - consumed < static_cast<uint32_t>(S)) {
      if (p_pos >= p_end) {
        // ---- start the next item (seq qt) if its slot pipeline allows
        if (!p_more || qt + 2 - qh >= QN) return;
        cp_async_wait_all();
        __syncwarp();
        const Item& it = q_items[qt % QN];
        if (it.np < 0) {
          p_more = false;
          return;
        }
        // request the struct of item qt+2 (ticket drawn one item ago) and the
        // ticket of item qt+3
        if (lane == 0) {
          Item* dst = &q_items[(qt + 2) % QN];
          if (static_cast<int64_t>(tk) < ntickets) {
            const Item* src = item_at(static_cast<int64_t>(tk));
            cp_async16(dst, src);
            cp_async16(reinterpret_cast<char*>(dst) + 16, reinterpret_cast<const char*>(src) + 16);
            if constexpr (PANELS) q_tick[(qt + 2) % QN] = static_cast<int64_t>(tk);
            tk = draw();
          } else {
            dst->np = -1;
          }
        }
        cp_async_commit();
        struct_pending = true;
        p_pos = item_p0(it);
        p_end = p_pos + it.np;
        p_r8 = item_r8(it);
        p_mt = (it.rows + 7) >> 3;
        if constexpr (WIDE) {
          p_ntf = (it.n + 7) >> 3;
          p_c8 = item_c8(it);
          p_cs = p_ntf < 4 ? p_ntf : 4;  // the class width (4 for a wide block)
          p_nt = p_ntf - p_c8 < 4 ? p_ntf - p_c8 : 4;
          p_sub = 0;
        } else if constexpr (MULTI) {
          p_nt = (it.n + 7) >> 3;
        }
        ++qt;
        if (p_pos < p_end) enter_chunk(qt - 1, p_pos, p_end);
        continue;
      }
      if (p_pos - c_base >= 32) enter_chunk(qt - 1, p_pos, p_end);
      const int s = s_issue;
      s_issue = (s_issue + 1 == S) ? 0 : s_issue + 1;
      if constexpr (WIDE) {
        // every lane reads the descriptor: the slice bookkeeping is warp-uniform
        const Desc d = dring[cs * 32 + static_cast<int>(p_pos - c_base)];
        const int KTF = (d.z + 1) >> 1;  // the product's 8-wide k tiles
        const int h0 = p_sub * kKTCap;
        const int KTS = KTF - h0 < kKTCap ? KTF - h0 : kKTCap;
        const int kcs = d.z - 2 * h0 < 2 * kKTCap ? d.z - 2 * h0 : 2 * kKTCap;
        const bool last = h0 + KTS >= KTF;
        if (lane == 0) {
          const uint32_t ba = static_cast<uint32_t>(p_mt * KTS) * 512u;
          const uint32_t bb = static_cast<uint32_t>(KTS * p_nt) * 512u;
          double* st = stages + static_cast<int64_t>(s) * g.stage_doubles;
          stage_kc[s] = kcs | (last ? 0x100 : 0);
          fence_proxy_async_smem();
          BT_DASSERT((static_cast<int64_t>(d.x) + static_cast<int64_t>(p_r8 + p_mt) * KTF) * 64 <=
                         g.a_len, "A slab range (wide)");
          BT_DASSERT((static_cast<int64_t>(d.y) + static_cast<int64_t>(KTF) * p_ntf) * 64 <= g.b_len,
                     "B slab range (wide)");
          BT_DASSERT(p_mt * KTS * 64 <= g.a_region &&
                         g.a_region + KTS * p_cs * 64 <= g.stage_doubles, "stage capacity (wide)");
          mbar_arrive_expect_tx(&bars[s], ba + bb);
          // A: rows r8.. of the block, k tiles [h0, h0 + KTS) (one copy when whole rows)
          const double* a0 = g.at + (static_cast<int64_t>(d.x) + static_cast<int64_t>(p_r8) * KTF + h0) * 64;
          if (KTS == KTF) {
            bulk_g2s(st, a0, ba, &bars[s]);
          } else {
            for (int tm = 0; tm < p_mt; ++tm)
              bulk_g2s(st + tm * KTS * 64, a0 + static_cast<int64_t>(tm) * KTF * 64,
                       static_cast<uint32_t>(KTS) * 512u, &bars[s]);
          }
          // B: k tiles [h0, h0 + KTS) x tile columns [c8, c8 + p_nt), rows p_cs apart
          const double* b0 = g.bt + (static_cast<int64_t>(d.y) + static_cast<int64_t>(h0) * p_ntf + p_c8) * 64;
          if (p_nt == p_ntf && p_nt == p_cs) {
            bulk_g2s(st + g.a_region, b0, bb, &bars[s]);
          } else {
            for (int kt = 0; kt < KTS; ++kt)
              bulk_g2s(st + g.a_region + kt * p_cs * 64, b0 + static_cast<int64_t>(kt) * p_ntf * 64,
                       static_cast<uint32_t>(p_nt) * 512u, &bars[s]);
          }
        }
        ++issued;
        if (last) {
          ++p_pos;
          p_sub = 0;
        } else {
          ++p_sub;
        }
        continue;
      }
      if (lane == 0) {
        const Desc d = dring[cs * 32 + static_cast<int>(p_pos - c_base)];
        const int KT = (d.z + 1) >> 1;  // 8-wide k tiles
        const uint32_t ba = static_cast<uint32_t>(p_mt * KT) * 512u;
        const uint32_t bb = static_cast<uint32_t>(KT * p_nt) * 512u;
        double* st = stages + static_cast<int64_t>(s) * g.stage_doubles;
        stage_kc[s] = d.z;
        fence_proxy_async_smem();
        BT_DASSERT((static_cast<int64_t>(d.x) + static_cast<int64_t>(p_r8) * KT) * 64 + ba / 8 <=
                       g.a_len, "A slab range");
        BT_DASSERT(static_cast<int64_t>(d.y) * 64 + bb / 8 <= g.b_len, "B slab range");
        BT_DASSERT(ba + bb <= static_cast<uint32_t>(g.stage_doubles) * 8u, "stage capacity");
        mbar_arrive_expect_tx(&bars[s], ba + bb);
        // (an L2 evict_last hint on these copies measured neutral on c1/c3)
        bulk_g2s(st, g.at + (static_cast<int64_t>(d.x) + static_cast<int64_t>(p_r8) * KT) * 64,
                 ba, &bars[s]);
        bulk_g2s(st + g.a_region, g.bt + static_cast<int64_t>(d.y) * 64, bb, &bars[s]);
        // (an L2 bulk prefetch of the following product measured 1-3 % slower)
      }
      ++issued;
      ++p_pos;
    }
  };

  top_up();
  __syncwarp();
  while (qh < qt) {
    const Item it = q_items[qh % QN];
    const int mt = (it.rows + 7) >> 3;  // 8-row tiles present in this C tile
    // panels in one launch: wait until the previous panel of this tile is stored
    int panel = 0;
    int* flag = nullptr;
    if constexpr (PANELS) {
      const int64_t tick = q_tick[qh % QN];
      panel = static_cast<int>(tick / g.nitems);
      flag = g.tile_flag + (tick - static_cast<int64_t>(panel) * g.nitems);
      if (panel > 0) {
        if (lane == 0) {
          long long spins = 0;
          while (ld_acquire_gpu(flag) < panel) {
            __nanosleep(32);
            BT_DASSERT(++spins < (1ll << 28), "K-panel flag wait (deadlock)");
          }
          (void)spins;
        }
        __syncwarp();
      }
    }
    const double* cin = panel > 0 ? g.cout : g.cin;
    if (it.np == 0 && it.cin_off == it.c_off && cin == g.cout) {  // in-place, no products
      if constexpr (PANELS)
        if (lane == 0) st_release_gpu(flag, panel + 1);
      ++qh;
      top_up();
      __syncwarp();
      continue;
    }
    // the tile body for a CM x CN tile (8-row x 8-column DMMA tiles)
    auto tile = [&](auto cm_c, auto cn_c) {
      constexpr int CM = decltype(cm_c)::value, CN = decltype(cn_c)::value;
      double acc[CM][CN][2];
#pragma unroll
      for (int tm = 0; tm < CM; ++tm)
#pragma unroll
        for (int tn = 0; tn < CN; ++tn) {
          acc[tm][tn][0] = 0.0;
          acc[tm][tn][1] = 0.0;
        }
      // C rows are RS 8x8 tiles apart (the block's tile columns; CN unless a
      // WIDE item is a 32-column tile of a wider block, which has NTI tiles)
      const int RS = WIDE ? (it.n + 7) >> 3 : CN;
      const int NTI = WIDE ? (RS - item_c8(it) < CN ? RS - item_c8(it) : CN) : CN;
      if (it.cin_off >= 0) {
#pragma unroll
        for (int tm = 0; tm < CM; ++tm)
          if (tm < mt) {
#pragma unroll
            for (int tn = 0; tn < CN; ++tn) {
              if (WIDE && tn >= NTI) continue;
              // PANELS: L2 loads, the tile may have been stored by another SM
              const double2* src = reinterpret_cast<const double2*>(
                  cin + it.cin_off + ((tm * RS + tn) << 6) + lc);
              const double2 v = PANELS ? __ldcg(src) : *src;
              acc[tm][tn][0] = v.x;
              acc[tm][tn][1] = v.y;
            }
          }
      }
      for (int t = 0; t < it.np; ++t) {
       bool last_slice = false;
       while (!last_slice) {  // (one pass unless WIDE splits the product's k)
        const int s = s_cons;
        mbar_wait(&bars[s], cons_phase);
        if (++s_cons == S) {
          s_cons = 0;
          cons_phase ^= 1u;
        }
        const int kcw = stage_kc[s];
        const int kc = WIDE ? (kcw & 0xff) : kcw;
        last_slice = WIDE ? (kcw >> 8) != 0 : true;
        const int KT = (kc + 1) >> 1;
        const double* sA = stages + static_cast<int64_t>(s) * g.stage_doubles;
        const double* sB = sA + g.a_region;
        // one 8-wide k tile: two 4-wide k chunks (the second may be padding)
        auto ktile = [&](int kt) {
          double af[2][CM], bf[2][CN];
#pragma unroll
          for (int tm = 0; tm < CM; ++tm) {
            af[0][tm] = sA[((tm * KT + kt) << 6) + la0];
            af[1][tm] = sA[((tm * KT + kt) << 6) + la1];
          }
#pragma unroll
          for (int tn = 0; tn < CN; ++tn) {
            bf[0][tn] = sB[((kt * CN + tn) << 6) + lb0];
            bf[1][tn] = sB[((kt * CN + tn) << 6) + lb1];
          }
#pragma unroll
          for (int tm = 0; tm < CM; ++tm)
#pragma unroll
            for (int tn = 0; tn < CN; ++tn)
              dmma_884(acc[tm][tn][0], acc[tm][tn][1], af[0][tm], bf[0][tn]);
          if (2 * kt + 1 < kc) {
#pragma unroll
            for (int tm = 0; tm < CM; ++tm)
#pragma unroll
              for (int tn = 0; tn < CN; ++tn)
                dmma_884(acc[tm][tn][0], acc[tm][tn][1], af[1][tm], bf[1][tn]);
          }
        };
        // k tiles, not unrolled (at most 8 per product, 4 per WIDE slice).
        // Measured against the loop unrolled by 4 with uniform guards: the
        // MULTI / WIDE launches carry up to 16 tile bodies (the producer
        // inlined into each) and the unrolled bodies overflowed the
        // instruction cache (ncu, WIDE: 27-72 % of stall samples on "no
        // instructions"; big40 1.05 -> 0.84 ms, c2 numeric 102 -> 96 us, c4
        // 3.00 -> 2.96 ms), and even the single-body launches run faster
        // rolled (c1 numeric 0.594 -> 0.585 ms, c3 1.751 -> 1.677 ms)
#pragma unroll 1
        for (int kt = 0; kt < KT; ++kt) ktile(kt);
        __syncwarp();
        ++consumed;
        top_up();
       }
      }
      double* dst = g.cout + it.c_off;
      BT_DASSERT(it.c_off >= 0 &&
                     it.c_off + (static_cast<int64_t>(mt - 1) * RS + NTI) * 64 <= g.cout_len,
                 "C tile range");
      BT_DASSERT(it.cin_off < 0 || it.cin_off + (static_cast<int64_t>(mt - 1) * RS + NTI) * 64 <=
                                       (cin == g.cout ? g.cout_len : g.cin_len),
                 "C_in tile range");
#pragma unroll
      for (int tm = 0; tm < CM; ++tm)
        if (tm < mt) {
#pragma unroll
          for (int tn = 0; tn < CN; ++tn) {
            if (WIDE && tn >= NTI) continue;
            __stcs(reinterpret_cast<double2*>(dst + ((tm * RS + tn) << 6) + lc),
                   make_double2(acc[tm][tn][0], acc[tm][tn][1]));
          }
        }
      if constexpr (PANELS) {  // publish: this panel of the tile is stored
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release_gpu(flag, panel + 1);
      }
    };
    if constexpr (MULTI) {
      // (WIDE: every tile of a wide block runs the 32-column body, the last,
      // narrower one with its columns beyond the block unstored -- measured:
      // dispatching it on its own width, a 40-column block's last tile on the
      // 8-column body with 4 accumulator chains, made big40 1.05 -> 1.85 ms)
      int ntc = (it.n + 7) >> 3;
      if (WIDE && ntc > 4) ntc = 4;
      const int cls = (mt - 1) * 4 + (ntc - 1);
      using std::integral_constant;
#define BT_TILE(cm, cn)                                                   \
  case (cm - 1) * 4 + (cn - 1):                                           \
    if constexpr (cm <= TMT && cn <= TNT)                                 \
      tile(integral_constant<int, cm>{}, integral_constant<int, cn>{});   \
    break;
      switch (cls) {
        BT_TILE(1, 1) BT_TILE(1, 2) BT_TILE(1, 3) BT_TILE(1, 4)
        BT_TILE(2, 1) BT_TILE(2, 2) BT_TILE(2, 3) BT_TILE(2, 4)
        BT_TILE(3, 1) BT_TILE(3, 2) BT_TILE(3, 3) BT_TILE(3, 4)
        BT_TILE(4, 1) BT_TILE(4, 2) BT_TILE(4, 3) BT_TILE(4, 4)
        default: break;
      }
#undef BT_TILE
    } else {
      tile(std::integral_constant<int, TMT>{}, std::integral_constant<int, TNT>{});
    }
    ++qh;
    top_up();
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// CUDA-core FP64 FMA (DFMA) small-GEMM for tiny C blocks (m, n <= 5): the
// shapes that do not tile onto the 8x8 DMMA fragment -- a 5x5x5 product uses
// 24 % of an 8x8x8 DMMA tile, 4x4x4 12.5 %, 1x1x1 0.2 %.  One THREAD owns one
// C block for its whole product chain: the MM x NN accumulators stay in
// registers, every k step is one B row (NN doubles from the T8 tile row, the
// XOR swizzle undone in registers) and MM A elements, MM*NN DFMAs, over the
// exact k of each product (no k padding work).  Products in ascending k per C
// block (block.hpp:45-60 order); the whole 8x8 T8 slot is written (padding 0).
// A warp works 32 C blocks at once, so its loads of 32 independent blocks
// are in flight together (memory-level parallelism without a staging ring).
template <int MM, int NN>
__global__ void __launch_bounds__(128) k_smm_dfma(const NumArgs g, const int32_t* __restrict__ k_sz) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= g.nitems) return;
  const Item it = g.items[g.item_lo + t];
  const int m = it.rows, n = it.n;
  const double* cin = g.cin;  // later K panels: the host passes C_out (in place)
  double acc[MM][NN];
#pragma unroll
  for (int r = 0; r < MM; ++r)
#pragma unroll
    for (int c = 0; c < NN; ++c) {
      double v = 0.0;
      if (it.cin_off >= 0 && r < m && c < n) v = cin[it.cin_off + r * 8 + (c ^ (((r >> 1) & 1) << 2))];
      acc[r][c] = v;
    }
  const int64_t p0 = item_p0(it);
  for (int p = 0; p < it.np; ++p) {
    const Desc d = g.desc[p0 + p];
    const int k = k_sz[d.w];
    const int KT = (d.z + 1) >> 1;
    const double* A = g.at + static_cast<int64_t>(d.x) * 64;
    const double* B = g.bt + static_cast<int64_t>(d.y) * 64;
    BT_DASSERT(static_cast<int64_t>(d.x) * 64 + static_cast<int64_t>(KT) * 64 <= g.a_len,
               "dfma A range");
    BT_DASSERT(static_cast<int64_t>(d.y) * 64 + static_cast<int64_t>(KT) * 64 <= g.b_len,
               "dfma B range");
    (void)KT;
    for (int kk = 0; kk < k; ++kk) {
      // B row kk (NT = 1: one tile column): 8 doubles of tile row kk & 7 of
      // k tile kk >> 3, stored with column u at u ^ sw
      const double* brow = B + ((kk >> 3) << 6) + ((kk & 7) << 3);
      const int sw = ((kk >> 1) & 1) << 2;
      double b[NN];
#pragma unroll
      for (int c = 0; c < NN; ++c) b[c] = c < n ? __ldg(brow + (c ^ sw)) : 0.0;
      // A column kk: element (r, kk) of the m x k block, k tile kk >> 3 of the
      // block's first (only) 8-row tile row
      const double* acol = A + ((kk >> 3) << 6);
#pragma unroll
      for (int r = 0; r < MM; ++r)
        if (r < m) {
          const double a = __ldg(acol + r * 8 + ((kk & 7) ^ (((r >> 1) & 1) << 2)));
#pragma unroll
          for (int c = 0; c < NN; ++c) acc[r][c] = fma(a, b[c], acc[r][c]);
        }
    }
  }
  // the full 8x8 slot, rows as 16-byte pairs; padding rows / columns zero
  double* dst = g.cout + it.c_off;
  BT_DASSERT(it.c_off >= 0 && it.c_off + 64 <= g.cout_len, "dfma C range");
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    double row[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) row[u] = 0.0;
#pragma unroll
    for (int c = 0; c < NN; ++c)
      if (r < MM && r < m && c < n) row[c ^ (((r >> 1) & 1) << 2)] = acc[r < MM ? r : 0][c];
#pragma unroll
    for (int h = 0; h < 4; ++h)
      __stcs(reinterpret_cast<double2*>(dst + r * 8 + 2 * h), make_double2(row[2 * h], row[2 * h + 1]));
  }
}

// Generic small-GEMM for blocks the DMMA tile kernels do not take (n > 32 or
// k > 64): one CTA of 256 threads per C block, the block swept in 64 x 64
// output sub-tiles, each thread owning a 4 x 4 register micro-tile
// (CUDA-core DFMA).  Per product, k is walked in chunks of 16: the 64 x 16
// A panel and 16 x 64 B panel are gathered from the T8 slots into shared
// memory (padding outside the block as zeros), then every k step is 4 A and
// 4 B shared-memory reads for 16 DFMAs.  Products in ascending k per C
// element (block.hpp:45-60 order); the whole T8 slot is written, padding as
// zeros (norms, the eps filter and DMMA reads of this block as an operand
// rely on zero padding).
constexpr int kGenT = 64;   // output sub-tile edge
constexpr int kGenK = 16;   // k chunk
__global__ void __launch_bounds__(256) k_smm_generic(const NumArgs g, const int32_t* __restrict__ k_sz) {
  __shared__ __align__(16) double sA[kGenK][kGenT + 2];  // [k][row] (+2: 16-byte rows)
  __shared__ __align__(16) double sB[kGenK][kGenT + 2];  // [k][col]
  const int64_t id = g.item_lo + blockIdx.x;
  if (blockIdx.x >= g.nitems) return;
  const Item it = g.items[id];
  const int m = it.rows, n = it.n;
  const int NT = tiles8(n), MT = tiles8(m);
  const int MP = MT * 8, NP = NT * 8;  // padded extents of the slot
  const int64_t p0 = item_p0(it);
  const int t = threadIdx.x;
  const int tr = (t >> 4) * 4, tc = (t & 15) * 4;  // this thread's micro-tile
  for (int r0 = 0; r0 < MP; r0 += kGenT)
    for (int c0 = 0; c0 < NP; c0 += kGenT) {
      double acc[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int r = r0 + tr + u, c = c0 + tc + v;
          acc[u][v] = (it.cin_off >= 0 && r < m && c < n) ? g.cin[it.cin_off + t8_pos(r, c, NT)]
                                                          : 0.0;
        }
      for (int p = 0; p < it.np; ++p) {
        const Desc d = g.desc[p0 + p];
        const int k = k_sz[d.w];
        const int KT = (d.z + 1) >> 1;
        const double* A = g.at + static_cast<int64_t>(d.x) * 64;
        const double* B = g.bt + static_cast<int64_t>(d.y) * 64;
        BT_DASSERT(static_cast<int64_t>(d.x) * 64 + static_cast<int64_t>(MT) * KT * 64 <= g.a_len,
                   "generic A range");
        BT_DASSERT(static_cast<int64_t>(d.y) * 64 + static_cast<int64_t>(KT) * NT * 64 <= g.b_len,
                   "generic B range");
        for (int k0 = 0; k0 < k; k0 += kGenK) {
          __syncthreads();  // the previous chunk's reads are done
          // gather the A panel (64 rows x 16 k) and the B panel (16 k x 64 cols)
          for (int e = t; e < kGenT * kGenK; e += 256) {
            const int kk = e % kGenK, rr = e / kGenK;     // A: k fastest (T8 rows)
            const int r = r0 + rr, kc = k0 + kk;
            sA[kk][rr] = (r < m && kc < k) ? A[t8_pos(r, kc, KT)] : 0.0;
            const int cc = e % kGenT, kb = e / kGenT;     // B: columns fastest
            const int c = c0 + cc, kr = k0 + kb;
            sB[kb][cc] = (c < n && kr < k) ? B[t8_pos(kr, c, NT)] : 0.0;
          }
          __syncthreads();
          const int kn = min(kGenK, k - k0);
          for (int kk = 0; kk < kn; ++kk) {
            double a[4], b[4];  // 16-byte shared-memory reads (two per operand)
            const double2 a01 = *reinterpret_cast<const double2*>(&sA[kk][tr]);
            const double2 a23 = *reinterpret_cast<const double2*>(&sA[kk][tr + 2]);
            const double2 b01 = *reinterpret_cast<const double2*>(&sB[kk][tc]);
            const double2 b23 = *reinterpret_cast<const double2*>(&sB[kk][tc + 2]);
            a[0] = a01.x; a[1] = a01.y; a[2] = a23.x; a[3] = a23.y;
            b[0] = b01.x; b[1] = b01.y; b[2] = b23.x; b[3] = b23.y;
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
          }
        }
      }
      // store the sub-tile: padding positions of the slot as zeros
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int r = r0 + tr + u, c = c0 + tc + v;
          if (r < MP && c < NP) {
            const int64_t cp = t8_pos(r, c, NT);
            BT_DASSERT(it.c_off + cp < g.cout_len, "generic C range");
            g.cout[it.c_off + cp] = (r < m && c < n) ? acc[u][v] : 0.0;
          }
        }
    }
}

}  // namespace bt
