// bt_multiply.cu -- the hot path: local block-sparse C += A*B on one B200.
//
// Device equivalent of detail::multiply_tiles_into (multiply_cannon.hpp:24-44):
//   reference                                here (device-resident)
//   std::map b_by_k + BatchItem list    ->   k_row_count / k_row_fill: one CTA per C
//   (multiply_cannon.hpp:27-36)              block-row walks A(i,:) x B(k,:) Gustavson
//                                            style with per-column counters in smem
//   order_batches (block.hpp:112-118)   ->   products emitted per C block in ascending
//                                            k (k loop is sequential per row)
//   get_or_create (matrix.hpp:191-196)  ->   C_out pattern = C_in U products, built
//                                            in the same two passes
//   block_gemm_acc (block.hpp:45-60)    ->   k_smm_dmma<TM,TN> (bt_smm.cuh)
// Accumulation per C element follows the reference order over k-blocks
// (ascending), each C block written exactly once (no atomics): results are
// deterministic run to run.  One host synchronisation per call (sizes).
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <tuple>
#include <mutex>
#include <map>
#include <array>
#include <cstdlib>

#include "bt_internal.cuh"
#include "bt_smm.cuh"

namespace bt {

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// DMMA tile classes 0..15, GENERIC (n > 32 or k > 64), TINY (m, n <= 5: the
// CUDA-core DFMA kernel)
enum { NCLASS = 18, GENERIC = 16, TINY = 17 };
constexpr int kTinyMax = 5;
// Work-item segments: (tile class, column band).  Within a class the bands are
// consecutive, band-major, so the numeric phase sweeps C in column bands and
// only B(:, band) has to stay resident in L2.
constexpr int kMaxBands = 8;
constexpr int NSEG = NCLASS * kMaxBands;
constexpr uint32_t kCinFlag = 0x80000000u;

// Tile classes: 16 DMMA tile shapes (ceil(m/8) in 1..4 -- blocks taller than
// `tr` rows (24 or 32) are cut in tr-row tiles -- times ceil(n/8) in 1..4;
// wide blocks (n > 32) are cut in 32-column tiles of the n/8 = 4 classes) +
// GENERIC (the CUDA-core kernel: only with wide = false, for n > 32 or k > 64).
__host__ __device__ inline int shape_class(int m, int n, bool dmma_ok, int tr, bool tiny,
                                           bool wide) {
  if (tiny && m <= kTinyMax && n <= kTinyMax) return TINY;
  if (!dmma_ok || (n > 32 && !wide)) return GENERIC;
  const int mc = m > tr ? tr / 8 : (m + 7) / 8;
  const int nc = n > 32 ? 4 : (n + 7) / 8;
  return (mc - 1) * 4 + (nc - 1);
}
// work items (C tiles) of one C block: row tiles x column tiles
__host__ __device__ inline int row_tiles(int m, int cls, int tr) {
  return (cls < GENERIC && m > tr) ? (m + tr - 1) / tr : 1;
}
__host__ __device__ inline int col_tiles(int n, int cls) {
  return (cls < GENERIC && n > 32) ? (n + 31) / 32 : 1;
}
__host__ __device__ inline int class_tiles(int m, int n, int cls, int tr) {
  return row_tiles(m, cls, tr) * col_tiles(n, cls);
}

__device__ __forceinline__ bool keep_product(const double* na, const double* nb, int32_t e,
                                             int32_t f, double eps) {
  return !(eps > 0.0) || __dmul_rn(na[e], nb[f]) >= eps;
}

struct RowArgs;
__device__ __forceinline__ int band_of(int64_t j, const RowArgs& g);

struct RowArgs {
  const int32_t *a_rp, *a_col, *b_rp, *b_col, *c_rp, *c_col;  // A, B, C_in patterns
  const int64_t *a_off, *b_off, *c_off;                        // T8 offsets (doubles)
  const int32_t *m_sz, *n_sz, *k_sz;                           // C rows, C cols, A cols
  const double *na, *nb;                                       // block norms (eps > 0)
  double eps;
  int64_t ncols;  // N (block columns of C)
  int nbands;     // column bands of the numeric sweep (1..kMaxBands)
  int sort_min;   // rows with more A entries per chunk emit by window sort
  bool colmask;   // k_row_fill has a 64-bit per-column mask array (N <= kMaskCols)
  int tall_rows;  // tile height for blocks taller than 32 rows (24 or 32)
  bool tiny;      // m, n <= kTinyMax C blocks go to the DFMA kernel (class TINY)
  // column chunk width of the symbolic passes: rows are processed in chunks
  // of `colw` block columns (per-column counters in shared memory are sized
  // for one chunk), so C may have any number of block columns
  int64_t colw;
  int splits;     // k_row_fill CTAs per C row (long rows: chunk ranges)
  int64_t pair_smem_off;  // k_row_fill<512>: byte offset of the pair caches
  // split-count mode (few long rows): [M][splits + 1][ncols] column counts of
  // each CTA's range of A chunks (k_row_count_split), turned by pass 1 into
  // the kept pairs of the earlier ranges (slot s) and the row total (slot
  // splits), so the fill CTAs of a row need not recount it; null otherwise
  int32_t* snap;
  // warp-row fill (short rows, k_wrow_fill): pass 1 flags and lists the rows
  // that do not fit a warp (more than 64 A entries, more than wcap_k products
  // or wcap_d C blocks); k_row_fill_list takes those (grid-stride)
  int32_t* wflag;                // [M] 1 = row left to the CTA fill (null: no warp fill)
  int32_t* wlist;                // those rows
  unsigned long long* wlist_n;   // their count
  int wcap_k, wcap_d;
  bool dmma_ok;
  bool wide;      // blocks wider than 32 columns in 32-column DMMA tiles (else GENERIC)
  // pass 1 outputs
  int32_t* row_nnz;
  int64_t* row_prod;
  int64_t* row_vals;
  unsigned long long* totals;       // [0] candidates [1] sum m*n*k [2] stored elements
  unsigned long long* class_items;  // [NSEG]
  // pass 2 inputs/outputs
  const int32_t* out_rp;
  const int64_t* prod_base;  // exclusive scan of row_prod
  const int64_t* val_base;   // exclusive scan of row_vals
  int32_t* out_col;
  int32_t* out_row;
  int64_t* out_off;
  int64_t* cin_map;
  int32_t* out_np;  // products per C entry
  int64_t* out_p0;  // first product per C entry
  Desc* desc;
  // work items, written by the fill pass into per-class segments
  unsigned long long* class_cursor;  // [NSEG], initialised to the segment bases
  Item* items;
  int64_t nprod_total, nitems_total;  // device checks of the checked build
};

__device__ __forceinline__ int band_of(int64_t j, const RowArgs& g) {
  if (g.nbands == 1) return 0;
  // 32-bit division (j * nbands < 2^31 for any N the stores allow with <= 8 bands
  // below 2^28 columns); the 64-bit one costs ~70 instructions per call
  if (g.ncols < (int64_t(1) << 27))
    return static_cast<int>(static_cast<uint32_t>(j * g.nbands) / static_cast<uint32_t>(g.ncols));
  return static_cast<int>((j * g.nbands) / g.ncols);
}

// The work items of one C block (row tiles of tall_rows rows x 32-column
// tiles of a wide block) at items[at, at + class_tiles).
__device__ __forceinline__ void emit_items(const RowArgs& g, unsigned long long at, int m, int n,
                                           int cls, int64_t c_off, int64_t cin, int64_t p0,
                                           int np);

// Row walk helpers.  A(i,:) x B(k,:) pairs are enumerated load-balanced: the A
// entries of a chunk are staged in shared memory with the prefix of their B-row
// lengths, and every thread takes flat pair indices (binary search into the
// prefix), so all global loads of a chunk are independent (no per-k latency
// chain).
// The symbolic kernels are instantiated for CH = 256 threads per row (long
// rows: c1, c3, c5) and CH = 64 (short rows, many of them: c2, c4 -- four
// times the rows in flight per SM).  CH A entries are staged per chunk
// (= blockDim); emission windows hold pair_pt * CH pairs.
constexpr int kChunkA = 256;   // the wide variant (host-side chunk arithmetic)
// pairs per thread in the window sort (4 at 512 threads: the static shared
// memory of the sort and the pair caches stays under 48 KB)
template <int CH>
constexpr int pair_pt() { return CH >= 512 ? 4 : 8; }
template <int CH>
constexpr int pair_cap() { return pair_pt<CH>() * CH; }

template <int CH>
struct RowChunk {  // shared-memory staging of up to CH A entries
  int32_t k[CH];
  int32_t b0[CH];
  int32_t pref[CH + 1];
  int32_t ksz[CH];  // block size along k
  int32_t au[CH];   // T8 tile offset of the A block (offset / 64)
};

// first position in b_col[lo, hi) with column >= j (B rows are column sorted)
__device__ __forceinline__ int32_t col_lower_bound(const int32_t* __restrict__ col, int32_t lo,
                                                   int32_t hi, int64_t j) {
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (col[mid] < j) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Stage A entries [e0, e0 + kChunkA) of row i; returns the pair count of the
// chunk.  Pairs are restricted to C columns [j0, j1) (the current column chunk;
// the whole row when [0, ncols)).
template <int CH>
__device__ int64_t stage_chunk(const RowArgs& g, int32_t e0, int32_t e1, RowChunk<CH>& rc,
                               int64_t j0, int64_t j1) {
  using BS = cub::BlockScan<int32_t, CH>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int32_t total;
  const int32_t e = e0 + threadIdx.x;
  int32_t len = 0;
  if (e < e1) {
    const int32_t k = g.a_col[e];
    int32_t b0 = g.b_rp[k], b1 = g.b_rp[k + 1];
    if (j0 > 0) b0 = col_lower_bound(g.b_col, b0, b1, j0);
    if (j1 < g.ncols) b1 = col_lower_bound(g.b_col, b0, b1, j1);
    len = b1 - b0;
    rc.k[threadIdx.x] = k;
    rc.b0[threadIdx.x] = b0;
    // per-entry constants the emission loops need, loaded once here (in
    // parallel) so those loops touch shared memory only
    rc.ksz[threadIdx.x] = g.k_sz[k];
    rc.au[threadIdx.x] = static_cast<int32_t>(g.a_off[e] >> 6);
  }
  int32_t ex, tot;
  BS(tmp).ExclusiveSum(len, ex, tot);
  rc.pref[threadIdx.x] = ex;
  if (threadIdx.x == 0) {
    rc.pref[CH] = tot;
    total = tot;
  }
  __syncthreads();
  return total;
}

// local A entry of flat pair t: last l with pref[l] <= t
template <int CH>
__device__ __forceinline__ int find_entry(const RowChunk<CH>& rc, int n, int32_t t) {
  int lo = 0, hi = n;  // pref[lo] <= t < pref[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (rc.pref[mid] <= t) lo = mid; else hi = mid;
  }
  return lo;
}

// cnt[j]: products of C(i,j) (kept by the eps filter) | kCinFlag for C_in blocks;
// bits[j/32]: column j touched.  The column passes then visit touched columns
// only (word by word), so their cost is O(N/32 + touched) per row.
// cache_j / cache_bu (fill pass, optional): for a row that is one chunk of
// at most kPairCap pairs, pair t's column (0xffffffff if filtered out) and B
// tile offset are kept in shared memory so the emission sweeps need no global
// loads; returns whether the cache is valid.
// before / split_c0 (split fill CTAs): before[j] also counts the kept pairs of
// the A entries ahead of split_c0 (the chunks of the earlier CTAs of the row).
// Counters are local to the column chunk [j0, j0 + jw): cnt[j - j0].
template <int CH>
__device__ bool row_products(const RowArgs& g, int64_t i, uint32_t* cnt, uint32_t* bits,
                             RowChunk<CH>& rc, unsigned long long* cand, unsigned long long* mnk,
                             int64_t j0, int64_t jw,
                             uint32_t* cache_j = nullptr, int32_t* cache_bu = nullptr,
                             int16_t* cache_l = nullptr,
                             uint32_t* before = nullptr, int32_t split_c0 = 0) {
  const int nw = static_cast<int>((jw + 31) >> 5);
  for (int64_t j = threadIdx.x; j < jw; j += blockDim.x) cnt[j] = 0u;
  if (before)
    for (int64_t j = threadIdx.x; j < jw; j += blockDim.x) before[j] = 0u;
  for (int w = threadIdx.x; w < nw; w += blockDim.x) bits[w] = 0u;
  __syncthreads();
  for (int32_t e = g.c_rp[i] + threadIdx.x; e < g.c_rp[i + 1]; e += blockDim.x) {
    const int64_t j = g.c_col[e] - j0;
    if (j < 0 || j >= jw) continue;
    cnt[j] = kCinFlag;
    atomicOr(&bits[j >> 5], 1u << (j & 31));
  }
  const int32_t a0 = g.a_rp[i], a1 = g.a_rp[i + 1];
  bool cached = false;
  for (int32_t c0 = a0; c0 < a1; c0 += CH) {
    const int n = min(CH, a1 - c0);
    const int64_t T = stage_chunk<CH>(g, c0, a1, rc, j0, j0 + jw);
    const bool cache = cache_j && a1 - a0 <= CH && T <= pair_cap<CH>();
    const bool ahead = before && c0 < split_c0;
    for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
      const int l = find_entry(rc, n, static_cast<int32_t>(t));
      const int32_t f = rc.b0[l] + static_cast<int32_t>(t - rc.pref[l]);
      if (cand) ++*cand;
      if (!keep_product(g.na, g.nb, c0 + l, f, g.eps)) {
        if (cache) cache_j[t] = 0xffffffffu;
        continue;
      }
      const int32_t j = static_cast<int32_t>(g.b_col[f] - j0);
      if (cache) {
        cache_j[t] = static_cast<uint32_t>(j);
        cache_bu[t] = static_cast<int32_t>(g.b_off[f] >> 6);
        cache_l[t] = static_cast<int16_t>(l);  // the emission sweeps skip the search
      }
      if (atomicAdd(&cnt[j], 1u) == 0u) atomicOr(&bits[j >> 5], 1u << (j & 31));
      if (ahead) atomicAdd(&before[j], 1u);
      if (mnk) *mnk += static_cast<unsigned long long>(rc.ksz[l]) * g.n_sz[j + j0];
    }
    __syncthreads();
    cached = cache;
  }
  return cached;
}

// Split-count mode: the column counts of row i from pass 1's snapshots
// (DESIGN.md 4.2).  finalize (pass 1): sums the per-range counts, leaves the
// exclusive prefix per range in slot s and the total in slot S; fill: reads
// the total and, for range `split` > 0, the earlier ranges' pairs (`before`).
// Then the touched bits and the C_in flags as row_products sets them.
__device__ __forceinline__ void snap_counts(const RowArgs& g, int64_t i, uint32_t* cnt,
                                            uint32_t* bits, uint32_t* before, int split,
                                            bool finalize) {
  const int S = g.splits;
  const int64_t N = g.ncols;
  int32_t* row = g.snap + i * (S + 1) * N;
  for (int w = threadIdx.x; w < static_cast<int>((N + 31) >> 5); w += blockDim.x) bits[w] = 0u;
  for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
    uint32_t tot;
    if (finalize) {
      int32_t run = 0;
      for (int s = 0; s < S; ++s) {
        const int32_t v = row[s * N + j];
        row[s * N + j] = run;
        run += v;
      }
      row[S * N + j] = run;
      tot = static_cast<uint32_t>(run);
    } else {
      tot = static_cast<uint32_t>(row[S * N + j]);
      if (before) before[j] = static_cast<uint32_t>(row[split * N + j]);
    }
    cnt[j] = tot;
  }
  __syncthreads();
  for (int64_t j = threadIdx.x; j < N; j += blockDim.x)
    if (cnt[j]) atomicOr(&bits[j >> 5], 1u << (j & 31));
  for (int32_t e = g.c_rp[i] + threadIdx.x; e < g.c_rp[i + 1]; e += blockDim.x) {
    const int64_t j = g.c_col[e];
    cnt[j] |= kCinFlag;
    atomicOr(&bits[j >> 5], 1u << (j & 31));
  }
  __syncthreads();
}

// Warp-aggregated shared-memory atomicAdd: lanes adding to the same counter
// (same class) are combined, one atomic per group; returns each lane's slot.
__device__ __forceinline__ unsigned long long agg_add(unsigned long long* ctr, int key,
                                                      unsigned long long v) {
  const unsigned active = __activemask();
  const unsigned peers = __match_any_sync(active, key);
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(peers) - 1;
  const unsigned below = peers & ((1u << lane) - 1u);
  // all members of a group add the same v here (v depends on the key only)
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(ctr, v * static_cast<unsigned long long>(__popc(peers)));
  base = __shfl_sync(peers, base, leader);
  return base + v * static_cast<unsigned long long>(__popc(below));
}

// Adds the work items of one C block to its segment counter; returns the
// lane's slot.  Blocks up to 32 columns: the count depends on the segment
// alone (the row's m, the class), so the warp-aggregated add applies; a wide
// block's count also depends on its n (column tiles): one atomic per lane.
__device__ __forceinline__ unsigned long long tiles_add(unsigned long long* ctr, int seg, int n,
                                                        unsigned long long v) {
  if (n > 32) return atomicAdd(ctr, v);
  return agg_add(ctr, seg, v);
}

// Touched columns of the row in ascending order -> tcol[0..n); returns n.
template <int CH>
__device__ int compact_touched(const uint32_t* bits, int nw, int32_t* tcol) {
  using BS = cub::BlockScan<int, CH>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int total;
  int run = 0;
  for (int w0 = 0; w0 < nw; w0 += blockDim.x) {
    const int w = w0 + threadIdx.x;
    const uint32_t word = w < nw ? bits[w] : 0u;
    int ex, tot;
    BS(tmp).ExclusiveSum(__popc(word), ex, tot);
    int q = run + ex;
    for (uint32_t x = word; x; x &= x - 1) tcol[q++] = w * 32 + __ffs(x) - 1;
    run += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) total = run;
  __syncthreads();
  return total;
}

__device__ __forceinline__ void emit_items(const RowArgs& g, unsigned long long at, int m, int n,
                                           int cls, int64_t c_off, int64_t cin, int64_t p0,
                                           int np) {
  const int nr = row_tiles(m, cls, g.tall_rows), nc = col_tiles(n, cls);
  const int64_t tile_row = static_cast<int64_t>(tiles8(n)) * 64;
  for (int qr = 0; qr < nr; ++qr) {
    const int r0 = g.tall_rows * qr;
    for (int qc = 0; qc < nc; ++qc) {
      const int64_t o = (r0 >> 3) * tile_row + static_cast<int64_t>(qc) * 4 * 64;
      Item it;
      it.c_off = c_off + o;
      it.cin_off = cin >= 0 ? cin + o : -1;
      it.p0r8 = item_pack(p0, r0 >> 3, 4 * qc);
      it.np = np;
      it.rows = static_cast<int16_t>(nr > 1 ? min(g.tall_rows, m - r0) : m);
      it.n = static_cast<int16_t>(n);
      BT_DASSERT(static_cast<int64_t>(at) + qr * nc + qc < g.nitems_total, "work item slot");
      g.items[at + qr * nc + qc] = it;
    }
  }
}

// Pass 1: per C block-row i -- number of C_out blocks, products, T8 slab size,
// stored elements, per-class work items, useful flops.
template <int CH, bool SNAP = false>
__device__ __forceinline__ void row_count_one(const RowArgs& g, const int64_t i) {
  extern __shared__ uint32_t cnt[];
  uint32_t* bits = cnt + g.colw;
  int32_t* tcol = reinterpret_cast<int32_t*>(bits + ((g.colw + 31) >> 5));
  __shared__ unsigned long long cls_items[NSEG];
  __shared__ RowChunk<CH> rc;
  // empty C row (no A entries, no C_in blocks): sizes are zero, nothing else
  // (tensor-shaped operands such as c4 leave most matricized rows empty)
  if (g.a_rp[i] == g.a_rp[i + 1] && g.c_rp[i] == g.c_rp[i + 1]) {
    if (threadIdx.x == 0) {
      g.row_nnz[i] = 0;
      g.row_prod[i] = 0;
      g.row_vals[i] = 0;
      if (g.wflag) g.wflag[i] = 0;
    }
    return;
  }
  for (int t = threadIdx.x; t < NSEG; t += blockDim.x) cls_items[t] = 0;
  unsigned long long cand = 0, mnk = 0;
  const int m = g.m_sz[i];
  long long nnz = 0, prods = 0, vals = 0, elems = 0;
  // column chunks (one when the row fits the shared-memory counters)
  for (int64_t j0 = 0; j0 < g.ncols; j0 += g.colw) {
    const int64_t jw = min(g.colw, g.ncols - j0);
    if constexpr (SNAP)  // (candidates and flops were added by k_row_count_split)
      snap_counts(g, i, cnt, bits, nullptr, 0, true);
    else
      row_products(g, i, cnt, bits, rc, &cand, &mnk, j0, jw);
    const int ntouch = compact_touched<CH>(bits, static_cast<int>((jw + 31) >> 5), tcol);
    for (int q = threadIdx.x; q < ntouch; q += blockDim.x) {
      const int jl = tcol[q];
      const int64_t j = j0 + jl;
      const uint32_t v = cnt[jl];
      const int n = g.n_sz[j];
      ++nnz;
      prods += v & ~kCinFlag;
      vals += t8_size(m, n);
      elems += static_cast<long long>(m) * n;
      const int cls = shape_class(m, n, g.dmma_ok, g.tall_rows, g.tiny, g.wide);
      const int seg = cls * kMaxBands + band_of(j, g);
      tiles_add(&cls_items[seg], seg, n,
              static_cast<unsigned long long>(class_tiles(m, n, cls, g.tall_rows)));
    }
    __syncthreads();  // counters are cleared for the next chunk
  }
  // the six row sums in one reduction: shuffles within each warp, one
  // barrier, then thread 0 adds the per-warp partials (exact integer sums)
  constexpr int kW = CH / 32;
  __shared__ long long part[6][kW];
  long long r6[6] = {nnz, prods, vals, elems, static_cast<long long>(cand),
                     static_cast<long long>(mnk)};
#pragma unroll
  for (int q = 0; q < 6; ++q)
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) r6[q] += __shfl_xor_sync(0xffffffffu, r6[q], d);
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int q = 0; q < 6; ++q) part[q][threadIdx.x >> 5] = r6[q];
  }
  __syncthreads();
  long long tq[6] = {0, 0, 0, 0, 0, 0};
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
      for (int w = 0; w < kW; ++w) tq[q] += part[q][w];
  }
  const long long t_nnz = tq[0], t_prod = tq[1], t_vals = tq[2], t_el = tq[3], t_cand = tq[4],
                  t_mnk = tq[5];
  if (threadIdx.x == 0) {
    g.row_nnz[i] = static_cast<int32_t>(t_nnz);
    g.row_prod[i] = t_prod;
    g.row_vals[i] = t_vals;
    if (g.wflag) {  // does the row fit the warp-row fill?
      const bool over = g.a_rp[i + 1] - g.a_rp[i] > 64 || t_prod > g.wcap_k || t_nnz > g.wcap_d;
      g.wflag[i] = over ? 1 : 0;
      if (over) g.wlist[atomicAdd(g.wlist_n, 1ull)] = static_cast<int32_t>(i);
    }
    if (t_cand) atomicAdd(&g.totals[0], static_cast<unsigned long long>(t_cand));
    if (t_mnk) atomicAdd(&g.totals[1], static_cast<unsigned long long>(t_mnk) * m);
    if (t_el) atomicAdd(&g.totals[2], static_cast<unsigned long long>(t_el));
  }
  __syncthreads();
  for (int t = threadIdx.x; t < NSEG; t += blockDim.x)
    if (cls_items[t]) atomicAdd(&g.class_items[t], cls_items[t]);
}

// one CTA per row
template <int CH>
__global__ void __launch_bounds__(CH) k_row_count(const RowArgs g) {
  row_count_one<CH>(g, blockIdx.x);
}

// split-count mode, second step: the row sums from the per-range snapshots
// (its own instantiation: the common pass 1 carries none of it)
template <int CH>
__global__ void __launch_bounds__(CH) k_row_count_snap(const RowArgs g) {
  row_count_one<CH, true>(g, blockIdx.x);
}

// Split-count mode, first step: CTA (i, s) counts the kept pairs of its range
// of A chunks per C column (the fill's ranges) into snap[i][s][:], and adds
// its candidates and useful flops to the totals.  k_row_count then sums the
// ranges per row (snap_counts).  c3's 100 rows of ~2 000 A entries: one CTA
// per row left most SMs idle and every fill CTA recounted its whole row.
template <int CH>
__global__ void __launch_bounds__(CH) k_row_count_split(const RowArgs g) {
  extern __shared__ uint32_t cnt[];  // [ncols]
  __shared__ RowChunk<CH> rc;
  const int S = g.splits;
  const int64_t i = blockIdx.x / S;
  const int split = static_cast<int>(blockIdx.x % S);
  const int64_t N = g.ncols;
  const int32_t a0 = g.a_rp[i], a1 = g.a_rp[i + 1];
  for (int64_t j = threadIdx.x; j < N; j += CH) cnt[j] = 0u;
  __syncthreads();
  const int nch = (a1 - a0 + CH - 1) / CH;
  const int ch_lo = static_cast<int>((static_cast<int64_t>(split) * nch) / S);
  const int ch_hi = static_cast<int>((static_cast<int64_t>(split + 1) * nch) / S);
  unsigned long long cand = 0, mnk = 0;
  for (int ch = ch_lo; ch < ch_hi; ++ch) {
    const int32_t c0 = a0 + ch * CH;
    const int n = min(CH, a1 - c0);
    const int64_t T = stage_chunk<CH>(g, c0, a1, rc, 0, N);
    for (int64_t t = threadIdx.x; t < T; t += CH) {
      const int l = find_entry(rc, n, static_cast<int32_t>(t));
      const int32_t f = rc.b0[l] + static_cast<int32_t>(t - rc.pref[l]);
      ++cand;
      if (!keep_product(g.na, g.nb, c0 + l, f, g.eps)) continue;
      const int32_t j = g.b_col[f];
      atomicAdd(&cnt[j], 1u);
      mnk += static_cast<unsigned long long>(rc.ksz[l]) * g.n_sz[j];
    }
    __syncthreads();
  }
  int32_t* out = g.snap + (i * (S + 1) + split) * N;
  for (int64_t j = threadIdx.x; j < N; j += CH) out[j] = static_cast<int32_t>(cnt[j]);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    cand += __shfl_xor_sync(0xffffffffu, cand, d);
    mnk += __shfl_xor_sync(0xffffffffu, mnk, d);
  }
  if ((threadIdx.x & 31) == 0) {
    if (cand) atomicAdd(&g.totals[0], cand);
    if (mnk) atomicAdd(&g.totals[1], mnk * static_cast<unsigned long long>(g.m_sz[i]));
  }
}

// Pass 2: emit C_out row i (columns, T8 offsets, C_in slots, per-block product
// ranges) and the product descriptors, k ascending within every C block.
// Pairs of up to kPairCap are staged in shared memory by all threads in
// parallel; the ordered emission then walks the staged A entries one k at a
// time touching shared memory only.
// 4 resident CTAs per SM (64 registers, no spills): the fill is latency bound
// -- measured fill 50.8 -> 38.7 us (c1), 53 -> 45 (c2), 540 -> 318 (c4)
// against the unconstrained 111-register build (profiles/r02/fill_occupancy_ab.txt)
#ifndef BT_FILL_MINB
#define BT_FILL_MINB 4
#endif
template <int CH>
__device__ __forceinline__ void row_fill_one(const RowArgs& g, const int64_t i, const int split) {
  constexpr int kPairCap = pair_cap<CH>();
  constexpr int kPairPT = pair_pt<CH>();
  extern __shared__ uint32_t sm[];
  uint32_t* cnt = sm;                                        // counts -> C entry rank
  int32_t* cur = reinterpret_cast<int32_t*>(sm + g.colw);  // product cursor
  uint32_t* bits = sm + 2 * g.colw;                         // touched columns
  __shared__ RowChunk<CH> rc;
  // pair caches: static for 64/256 threads; for 512 at the end of the dynamic
  // block (g.pair_smem_off; static shared memory is capped at 48 KB)
  constexpr int kStatCap = CH >= 512 ? 1 : kPairCap;
  __shared__ int32_t s_bu_st[kStatCap];
  __shared__ int16_t s_l_st[kStatCap];
  __shared__ uint32_t s_key_st[kStatCap];
  uint32_t* s_key = s_key_st;   // sorted (column, slot) keys
  int32_t* s_bu = s_bu_st;      // B tile offset of staged pair
  int16_t* s_l = s_l_st;        // local A entry of staged pair
  if constexpr (CH >= 512) {
    char* dyn = reinterpret_cast<char*>(sm) + g.pair_smem_off;
    s_key = reinterpret_cast<uint32_t*>(dyn);
    s_bu = reinterpret_cast<int32_t*>(dyn + 4 * kPairCap);
    s_l = reinterpret_cast<int16_t*>(dyn + 8 * kPairCap);
  }
  using Sort = cub::BlockRadixSort<uint32_t, CH, kPairPT>;
  __shared__ typename Sort::TempStorage sort_tmp;
  __shared__ unsigned long long cls_n[NSEG], cls_at[NSEG];
  // long rows: `splits` CTAs per row, CTA s emitting the products of its range
  // of A chunks (its column cursors start after the earlier ranges' pairs);
  // the row's C index and work items are written by CTA 0
  if (g.out_rp[i] == g.out_rp[i + 1]) return;  // empty C row: nothing to emit
  const int32_t a0 = g.a_rp[i], a1 = g.a_rp[i + 1];
  const int nch = (a1 - a0 + CH - 1) / CH;
  const int ch_lo = static_cast<int>((static_cast<int64_t>(split) * nch) / g.splits);
  const int ch_hi = static_cast<int>((static_cast<int64_t>(split + 1) * nch) / g.splits);
  if (split > 0 && ch_lo == ch_hi) return;
  const int32_t e_lo = a0 + ch_lo * CH;
  const int32_t e_hi = min(a1, a0 + ch_hi * CH);
  uint32_t* before = nullptr;
  if (split > 0)
    before = sm + (g.colmask ? ((3 * g.colw + ((g.colw + 31) >> 5) + 1) & ~int64_t(1)) +
                                   2 * g.colw
                             : 3 * g.colw + ((g.colw + 31) >> 5));
  for (int t = threadIdx.x; t < NSEG; t += blockDim.x) cls_n[t] = 0;
  const int m = g.m_sz[i];
  const int32_t cbase = g.out_rp[i];
  const int64_t pbase = g.prod_base[i], vbase = g.val_base[i];
  int32_t* tcol = reinterpret_cast<int32_t*>(bits + ((g.colw + 31) >> 5));
  // C columns in chunks of colw (one chunk when the row fits the shared-memory
  // counters): C entries, ranks and product cursors continue across chunks
  long long run_prod = 0, run_val = 0;
  int run_q = 0;
  for (int64_t j0 = 0; j0 < g.ncols; j0 += g.colw) {
  const int64_t jw = min(g.colw, g.ncols - j0);
  // single-chunk rows: pair columns / B offsets cached, rc stays staged
  bool cached = false;
  if (g.snap)  // split-count mode: counts (and the earlier ranges') from pass 1
    snap_counts(g, i, cnt, bits, before, split, false);
  else
    cached = row_products(g, i, cnt, bits, rc, nullptr, nullptr, j0, jw, s_key, s_bu, s_l, before,
                          e_lo);
  const int ntouch = compact_touched<CH>(bits, static_cast<int>((jw + 31) >> 5), tcol);
  {
    // touched columns in ascending order, 256 at a time: ranks, product bases
    // and T8 offsets by block scans
    // both exclusive scans at once: warp shuffles, then the per-warp totals
    // through shared memory (2 barriers per 256 columns instead of two cub
    // block scans with their own barriers)
    constexpr int kW = CH / 32;
    __shared__ long long wt[2][kW];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int q0 = 0; q0 < ntouch; q0 += blockDim.x) {
      const int q = q0 + threadIdx.x;
      const bool ok = q < ntouch;
      const int j = ok ? tcol[q] : 0;  // chunk-local column
      const int64_t jg = j0 + j;
      const uint32_t cj = ok ? cnt[j] : 0u;
      const int n = ok ? g.n_sz[jg] : 0;
      const long long np = cj & ~kCinFlag, tv = ok ? t8_size(m, n) : 0;
      long long pi = np, vi = tv;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const long long py = __shfl_up_sync(0xffffffffu, pi, d);
        const long long vy = __shfl_up_sync(0xffffffffu, vi, d);
        if (lane >= d) {
          pi += py;
          vi += vy;
        }
      }
      if (lane == 31) {
        wt[0][wid] = pi;
        wt[1][wid] = vi;
      }
      __syncthreads();
      long long p_ex = pi - np, v_ex = vi - tv, p_tot = 0, v_tot = 0;
#pragma unroll
      for (int w = 0; w < kW; ++w) {
        const long long a = wt[0][w], b = wt[1][w];
        if (w < wid) {
          p_ex += a;
          v_ex += b;
        }
        p_tot += a;
        v_tot += b;
      }
      __syncthreads();
      if (ok && split > 0) cur[j] = static_cast<int32_t>(run_prod + p_ex + before[j]);
      if (ok && split == 0) {
        const int32_t c = cbase + run_q + q;
        g.out_col[c] = static_cast<int32_t>(jg);
        g.out_row[c] = static_cast<int32_t>(i);
        g.out_off[c] = vbase + run_val + v_ex;
        g.cin_map[c] = -1;
        g.out_np[c] = static_cast<int32_t>(np);
        g.out_p0[c] = pbase + run_prod + p_ex;
        cur[j] = static_cast<int32_t>(run_prod + p_ex);
        cnt[j] = static_cast<uint32_t>(run_q + q);  // rank of the C entry in the row
        const int cls = shape_class(m, n, g.dmma_ok, g.tall_rows, g.tiny, g.wide);
        const int seg = cls * kMaxBands + band_of(jg, g);
        tiles_add(&cls_n[seg], seg, static_cast<int>(n),
                static_cast<unsigned long long>(class_tiles(m, n, cls, g.tall_rows)));
      }
      run_prod += p_tot;
      run_val += v_tot;
    }
  }
  run_q += ntouch;
  __syncthreads();
  // C_in blocks of this chunk: slot of the matching C_out block
  if (split == 0)
    for (int32_t e = g.c_rp[i] + threadIdx.x; e < g.c_rp[i + 1]; e += blockDim.x) {
      const int64_t jl = g.c_col[e] - j0;
      if (jl >= 0 && jl < jw) g.cin_map[cbase + cnt[jl]] = g.c_off[e];
    }
  // ---- products of this column chunk, k ascending (this CTA's A chunks)
  for (int32_t c0 = e_lo; c0 < e_hi; c0 += CH) {
    const int n = min(CH, a1 - c0);
    const int64_t T = cached ? rc.pref[n] : stage_chunk<CH>(g, c0, a1, rc, j0, j0 + jw);
    if (cached && g.colmask && n <= 64) {
      // rank emission from the cached pairs (no global loads in the sweeps)
      unsigned long long* mask = reinterpret_cast<unsigned long long*>(
          sm + ((3 * g.colw + ((g.colw + 31) >> 5) + 1) & ~int64_t(1)));
      for (int q = threadIdx.x; q < ntouch; q += blockDim.x) mask[tcol[q]] = 0ull;
      __syncthreads();
      for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
        const uint32_t j = s_key[t];
        if (j == 0xffffffffu) continue;
        atomicOr(&mask[j], 1ull << s_l[t]);
      }
      __syncthreads();
      for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
        const uint32_t j = s_key[t];
        if (j == 0xffffffffu) continue;
        const int l = s_l[t];
        const int32_t p = cur[j] + __popcll(mask[j] & ((1ull << l) - 1ull));
        BT_DASSERT(p >= 0 && pbase + p < g.prod_base[i + 1], "descriptor slot");
        g.desc[pbase + p] = make_int4(rc.au[l], s_bu[t], (rc.ksz[l] + 3) >> 2, rc.k[l]);
      }
      __syncthreads();
      for (int q = threadIdx.x; q < ntouch; q += blockDim.x) {
        const int j = tcol[q];
        cur[j] += __popcll(mask[j]);
      }
      __syncthreads();
      continue;
    }
    if (g.colmask && n <= 64) {
      // Rank emission (chunks of <= 64 A entries): bit l of mask[j] marks the
      // pair (A entry l, column j); a pair's slot in its C block is cur[j] +
      // the number of lower entries l' < l in that column, i.e. k ascending,
      // in two parallel sweeps over the pairs -- no step per k.
      unsigned long long* mask = reinterpret_cast<unsigned long long*>(
          sm + ((3 * g.colw + ((g.colw + 31) >> 5) + 1) & ~int64_t(1)));
      for (int q = threadIdx.x; q < ntouch; q += blockDim.x) mask[tcol[q]] = 0ull;
      __syncthreads();
      for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
        const int l = find_entry(rc, n, static_cast<int32_t>(t));
        const int32_t f = rc.b0[l] + static_cast<int32_t>(t - rc.pref[l]);
        if (!keep_product(g.na, g.nb, c0 + l, f, g.eps)) continue;
        atomicOr(&mask[g.b_col[f] - j0], 1ull << l);
      }
      __syncthreads();
      for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
        const int l = find_entry(rc, n, static_cast<int32_t>(t));
        const int32_t f = rc.b0[l] + static_cast<int32_t>(t - rc.pref[l]);
        if (!keep_product(g.na, g.nb, c0 + l, f, g.eps)) continue;
        const int32_t j = static_cast<int32_t>(g.b_col[f] - j0);
        const int32_t p = cur[j] + __popcll(mask[j] & ((1ull << l) - 1ull));
        BT_DASSERT(p >= 0 && pbase + p < g.prod_base[i + 1], "descriptor slot");
        g.desc[pbase + p] = make_int4(rc.au[l], static_cast<int32_t>(g.b_off[f] >> 6),
                                      (rc.ksz[l] + 3) >> 2, rc.k[l]);
      }
      __syncthreads();
      for (int q = threadIdx.x; q < ntouch; q += blockDim.x) {
        const int j = tcol[q];
        cur[j] += __popcll(mask[j]);
      }
      __syncthreads();
      continue;
    }
    // Windows of <= kPairCap consecutive pairs (k ascending).  Inside a window
    // the kept pairs are sorted by (column, pair index) -- pair index order is
    // k order -- so every pair's slot is cur[j] + its rank in the column's run:
    // products stay in ascending k per C block without a step per k.
    if (n <= g.sort_min) {
      // few A entries (short rows): one k at a time, pairs staged per window
      for (int64_t w0 = 0; w0 < T; w0 += kPairCap) {
        const int64_t w1 = min(T, w0 + kPairCap);
        for (int64_t t = w0 + threadIdx.x; t < w1; t += blockDim.x) {
          const int slot = static_cast<int>(t - w0);
          const int l = find_entry(rc, n, static_cast<int32_t>(t));
          const int32_t f = rc.b0[l] + static_cast<int32_t>(t - rc.pref[l]);
          const bool keep = keep_product(g.na, g.nb, c0 + l, f, g.eps);
          s_key[slot] = keep ? static_cast<uint32_t>(g.b_col[f] - j0) : 0xffffffffu;
          s_bu[slot] = static_cast<int32_t>(g.b_off[f] >> 6);
        }
        __syncthreads();
        const int l_first = find_entry(rc, n, static_cast<int32_t>(w0));
        const int l_last = find_entry(rc, n, static_cast<int32_t>(w1 - 1));
        for (int l = l_first; l <= l_last; ++l) {
          const int kc = (rc.ksz[l] + 3) >> 2;
          const int au = rc.au[l];
          const int64_t t0 = max(w0, static_cast<int64_t>(rc.pref[l]));
          const int64_t t1 = min(w1, static_cast<int64_t>(rc.pref[l + 1]));
          for (int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
            const uint32_t j = s_key[t - w0];
            if (j == 0xffffffffu) continue;
            const int32_t p = cur[j]++;  // one pair per column per k: race free
            BT_DASSERT(p >= 0 && pbase + p < g.prod_base[i + 1], "descriptor slot");
        g.desc[pbase + p] = make_int4(au, s_bu[t - w0], kc, rc.k[l]);
          }
          __syncthreads();
        }
      }
      continue;
    }
    for (int64_t w0 = 0; w0 < T; w0 += kPairCap) {
      const int64_t w1 = min(T, w0 + kPairCap);
      uint32_t keys[kPairPT];
#pragma unroll
      for (int u = 0; u < kPairPT; ++u) {
        const int slot = threadIdx.x * kPairPT + u;
        const int64_t t = w0 + slot;
        keys[u] = 0xffffffffu;
        if (t < w1) {
          const int l = find_entry(rc, n, static_cast<int32_t>(t));
          const int32_t f = rc.b0[l] + static_cast<int32_t>(t - rc.pref[l]);
          if (keep_product(g.na, g.nb, c0 + l, f, g.eps)) {
            keys[u] = (static_cast<uint32_t>(g.b_col[f] - j0) << 11) | static_cast<uint32_t>(slot);
            s_bu[slot] = static_cast<int32_t>(g.b_off[f] >> 6);
            s_l[slot] = static_cast<int16_t>(l);
          }
        }
      }
      // blocked arrangement: thread owns ranks [tid*PT, ...); only the live
      // key bits are sorted (11 slot bits + the chunk's column bits; the
      // filtered-out key's low bits are all ones, above every real key)
      Sort(sort_tmp).Sort(keys, 0, 11 + (32 - __clz(static_cast<int>(jw))));
#pragma unroll
      for (int u = 0; u < kPairPT; ++u) s_key[threadIdx.x * kPairPT + u] = keys[u];
      __syncthreads();
      // run heads: the first rank of each column's run in this window goes to
      // run0[column] (cnt is free here: the C entry ranks were used above)
      uint32_t* run0 = cnt;
#pragma unroll
      for (int u = 0; u < kPairPT; ++u) {
        const uint32_t key = keys[u];
        const int q = threadIdx.x * kPairPT + u;
        if (key != 0xffffffffu && (q == 0 || (s_key[q - 1] >> 11) != (key >> 11)))
          run0[key >> 11] = static_cast<uint32_t>(q);
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < kPairPT; ++u) {
        const uint32_t key = keys[u];
        if (key == 0xffffffffu) continue;
        const int q = threadIdx.x * kPairPT + u;
        const uint32_t jkey = key >> 11;
        const int lo = static_cast<int>(run0[jkey]);  // first rank of this column's run
        const int slot = static_cast<int>(key & 0x7ffu);
        const int l = s_l[slot];
        const int kc = (rc.ksz[l] + 3) >> 2;
        const int32_t p = cur[jkey] + (q - lo);
        BT_DASSERT(p >= 0 && pbase + p < g.prod_base[i + 1], "descriptor slot");
        g.desc[pbase + p] = make_int4(rc.au[l], s_bu[slot], kc, rc.k[l]);
      }
      __syncthreads();
      // advance the column cursors by the run lengths (run ends do it)
#pragma unroll
      for (int u = 0; u < kPairPT; ++u) {
        const int q = threadIdx.x * kPairPT + u;
        const uint32_t key = s_key[q];
        if (key == 0xffffffffu) continue;
        const bool run_end = q + 1 == kPairCap || (s_key[q + 1] >> 11) != (key >> 11);
        if (run_end) cur[key >> 11] += q - static_cast<int>(run0[key >> 11]) + 1;
      }
      __syncthreads();
    }
  }
  __syncthreads();
  }  // column chunks
  if (split == 0) {
  // reserve this row's work items in every class segment (one atomic per class)
  for (int t = threadIdx.x; t < NSEG; t += blockDim.x) {
    const unsigned long long k = cls_n[t];
    cls_at[t] = k ? atomicAdd(&g.class_cursor[t], k) : 0ull;
  }
  __syncthreads();
  // work items of this row: tall blocks become 32-row tiles
  for (int32_t c = cbase + threadIdx.x; c < g.out_rp[i + 1]; c += blockDim.x) {
    const int j = g.out_col[c];
    const int n = g.n_sz[j];
    const int cls = shape_class(m, n, g.dmma_ok, g.tall_rows, g.tiny, g.wide);
    const int nt = class_tiles(m, n, cls, g.tall_rows);
    const int seg = cls * kMaxBands + band_of(j, g);
    const unsigned long long at = tiles_add(&cls_at[seg], seg, n, static_cast<unsigned long long>(nt));
    emit_items(g, at, m, n, cls, g.out_off[c], g.cin_map[c], g.out_p0[c], g.out_np[c]);
  }
  }  // split == 0
}

template <int CH>
__global__ void __launch_bounds__(CH, BT_FILL_MINB * 256 / CH) k_row_fill(const RowArgs g) {
  row_fill_one<CH>(g, blockIdx.x / g.splits, static_cast<int>(blockIdx.x % g.splits));
}

// list mode (rows left by the warp-row pass): one CTA per row, splits = 1
template <int CH>
__global__ void __launch_bounds__(CH, BT_FILL_MINB * 256 / CH) k_row_fill_list(const RowArgs g) {
  const unsigned long long n = *g.wlist_n;
  for (unsigned long long q = blockIdx.x; q < n; q += gridDim.x) {
    row_fill_one<CH>(g, g.wlist[q], 0);
    __syncthreads();
  }
}

// ---- warp-per-row fill (short rows: c2, c4) ---------------------------------
// One warp per C block-row, kWRows rows per CTA.  The row's distinct C columns
// live in a per-warp open-addressing hash table in shared memory (H slots)
// instead of the CTA fill's dense per-column arrays, whose 20 bytes per block
// column of C bound the rows an SM holds (c2: 1 463 columns -> 29 KB per row,
// 3 rows per SM with the pair caches; here 16-20 (H = 256) or 32+ (H = 128)
// rows per SM, no block-wide barriers inside a row).  Same outputs as
// k_row_fill: C columns ascending, products of a C block in ascending k (a
// pair's rank within its column = the number of lower A entries of the row in
// the column's 64-bit mask), so the numeric phase sees identical stacks.
// Pass 1 (k_row_count) flags the rows that do not fit (more than 64 A
// entries, more than 2H products, more than 3H/4 C blocks); k_row_fill_list
// emits those.  (A warp-row count pass was measured too: slower than the CTA
// count on c2 and c4 -- its per-row chain of pair batches is longer.)
constexpr int kWRows = 4;  // rows (warps) per CTA: more, smaller CTAs spread c2's 1 463 rows over all SMs
constexpr uint32_t kHEmpty = 0xffffffffu;

template <int H>
constexpr int hash_bits() { return H == 128 ? 7 : H == 256 ? 8 : 9; }

// insert `col`; returns whether it is new, `slot` its slot.  The callers keep
// the table below full occupancy (at most 3H/4 + 31 keys), so probing ends.
template <int H>
__device__ __forceinline__ bool hash_insert(uint32_t* hkey, uint32_t col, int& slot) {
  uint32_t s = (col * 2654435761u) >> (32 - hash_bits<H>());
  while (true) {
    const uint32_t prev = atomicCAS(&hkey[s], kHEmpty, col);
    if (prev == kHEmpty || prev == col) {
      slot = static_cast<int>(s);
      return prev == kHEmpty;
    }
    s = (s + 1) & (H - 1);
  }
}

// last A entry (lane) l < nac of the chunk with ex_l <= t (ex = exclusive
// prefix of the B-row lengths, one per lane)
__device__ __forceinline__ int warp_find_entry(int32_t ex, int nac, int32_t t) {
  int l = 0;
#pragma unroll
  for (int st = 16; st; st >>= 1) {
    const int c = l + st;
    const int32_t v = __shfl_sync(0xffffffffu, ex, c & 31);
    if (c < nac && v <= t) l = c;
  }
  return l;
}

// Per-warp shared memory of the fill pass (bytes): hmask u64[H], hkey u32[H],
// hcnt u32[H], pinfo u32[2H], pbu i32[2H], dl / ord / nbuf u32[3H/4] each,
// A-entry tables 3 x i32[64]
template <int H>
__host__ __device__ constexpr size_t wrow_fill_bytes() {
  return static_cast<size_t>(41 * H + 768);
}

// Candidate pairs are taken in groups of kWU x 32: every lane computes its kWU
// pairs' B entries and issues all their loads (norms, B column, B offset)
// before any hash work, so a group costs one memory round trip instead of kWU
// (the per-row chain of dependent DRAM round trips is what bounds these
// latency-bound passes).
constexpr int kWU = 4;

template <int H>
__global__ void __launch_bounds__(kWRows * 32) k_wrow_fill(const RowArgs g, const int64_t M) {
  constexpr int DMAX = 3 * H / 4, NR = (DMAX + 31) / 32;
  extern __shared__ __align__(16) unsigned char wfm[];
  __shared__ unsigned long long cls_n[NSEG], cls_at[NSEG];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  unsigned char* base = wfm + w * wrow_fill_bytes<H>();
  unsigned long long* hmask = reinterpret_cast<unsigned long long*>(base);
  uint32_t* hkey = reinterpret_cast<uint32_t*>(base + 8 * H);   // column, then product cursor
  uint32_t* hcnt = reinterpret_cast<uint32_t*>(base + 12 * H);  // products | (C_in index + 1) << 8
  uint32_t* pinfo = reinterpret_cast<uint32_t*>(base + 16 * H); // kept pair: slot << 8 | A entry
  int32_t* pbu = reinterpret_cast<int32_t*>(base + 24 * H);     // kept pair: B tile offset
  uint32_t* dl = reinterpret_cast<uint32_t*>(base + 32 * H);    // distinct keys, then item offsets
  uint32_t* ord = dl + DMAX;                                    // keys by ascending column
  int32_t* nbuf = reinterpret_cast<int32_t*>(ord + DMAX);       // n of ord[r]
  int32_t* a_au = reinterpret_cast<int32_t*>(base + 41 * H);    // per A entry of the row
  int32_t* a_k = a_au + 64;
  int32_t* a_kc = a_k + 64;
  for (int t = threadIdx.x; t < NSEG; t += blockDim.x) cls_n[t] = 0;
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kWRows + w;
  const bool act = i < M && !g.wflag[i] && g.out_rp[i] != g.out_rp[i + 1];
  int D = 0, m = 0;
  int32_t ci0 = 0;
  int64_t pbase = 0, vbase = 0;
  if (act) {
    const int32_t a0 = g.a_rp[i], a1 = g.a_rp[i + 1];
    ci0 = g.c_rp[i];
    const int32_t ci1 = g.c_rp[i + 1];
    m = g.m_sz[i];
    const int32_t cbase = g.out_rp[i];
    pbase = g.prod_base[i];
    vbase = g.val_base[i];
    for (int s = lane; s < H; s += 32) {
      hkey[s] = kHEmpty;
      hcnt[s] = 0u;
      hmask[s] = 0ull;
    }
    __syncwarp();
    for (int32_t e = ci0 + lane; e < ci1; e += 32) {  // C_in blocks (distinct columns)
      int s;
      hash_insert<H>(hkey, static_cast<uint32_t>(g.c_col[e]), s);
      hcnt[s] = static_cast<uint32_t>(e - ci0 + 1) << 8;
    }
    __syncwarp();
    int K = 0;
    for (int32_t cb = a0; cb < a1; cb += 32) {
      const int32_t e = cb + lane;
      const int nac = min(32, a1 - cb);
      int32_t b0 = 0, len = 0;
      if (e < a1) {
        const int32_t k = g.a_col[e];
        b0 = g.b_rp[k];
        len = g.b_rp[k + 1] - b0;
        const int lr = cb - a0 + lane;
        a_k[lr] = k;
        a_kc[lr] = (g.k_sz[k] + 3) >> 2;
        a_au[lr] = static_cast<int32_t>(g.a_off[e] >> 6);
      }
      int32_t incl = len;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
      }
      const int32_t ex = incl - len;
      const int32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      for (int32_t t0 = 0; t0 < tot; t0 += kWU * 32) {
        int32_t colv[kWU], buv[kWU];
        int lrv[kWU];
        bool keepv[kWU];
#pragma unroll
        for (int u = 0; u < kWU; ++u) {  // all loads of the group first
          const int32_t t = t0 + u * 32 + lane;
          const bool valid = t < tot;
          const int l = warp_find_entry(ex, nac, t);
          const int32_t f = __shfl_sync(0xffffffffu, b0, l) + t - __shfl_sync(0xffffffffu, ex, l);
          lrv[u] = cb - a0 + l;
          keepv[u] = valid && keep_product(g.na, g.nb, cb + l, f, g.eps);
          colv[u] = valid ? g.b_col[f] : 0;
          buv[u] = valid ? static_cast<int32_t>(g.b_off[f] >> 6) : 0;
        }
#pragma unroll
        for (int u = 0; u < kWU; ++u) {
          int s = 0;
          if (keepv[u]) {
            hash_insert<H>(hkey, static_cast<uint32_t>(colv[u]), s);
            atomicAdd(&hcnt[s], 1u);
            atomicOr(&hmask[s], 1ull << lrv[u]);
          }
          const unsigned kb = __ballot_sync(0xffffffffu, keepv[u]);
          if (keepv[u]) {
            const int kp = K + __popc(kb & lt);
            pinfo[kp] = (static_cast<uint32_t>(s) << 8) | static_cast<uint32_t>(lrv[u]);
            pbu[kp] = buv[u];
          }
          K += __popc(kb);
        }
      }
    }
    __syncwarp();
    // distinct columns -> dl (slot order), then ranked by column into ord
    for (int s0 = 0; s0 < H; s0 += 32) {
      const int s = s0 + lane;
      const uint32_t col = hkey[s];
      const bool occ = col != kHEmpty;
      const unsigned b = __ballot_sync(0xffffffffu, occ);
      if (occ) dl[D + __popc(b & lt)] = (col << 9) | static_cast<uint32_t>(s);
      D += __popc(b);
    }
    BT_DASSERT(D <= DMAX, "warp-row distinct columns");
    // rank of each key = number of smaller keys (keys are distinct), four per
    // 16-byte shared load (the list is padded with keys above every real one)
    const int D4 = (D + 3) & ~3;
    if (lane < D4 - D) dl[D + lane] = 0xffffffffu;
    __syncwarp();
    for (int d = lane; d < D; d += 32) {
      const uint32_t key = dl[d];
      int r = 0;
      const uint4* dl4 = reinterpret_cast<const uint4*>(dl);
      for (int x = 0; x < D4 / 4; ++x) {
        const uint4 v = dl4[x];
        r += (v.x < key) + (v.y < key) + (v.z < key) + (v.w < key);
      }
      ord[r] = key;
    }
    __syncwarp();
    {
      int nr[NR];  // column sizes of the C entries, all loads in flight
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const int r = q * 32 + lane;
        nr[q] = r < D ? g.n_sz[ord[r] >> 9] : 0;
      }
#pragma unroll
      for (int q = 0; q < NR; ++q)
        if (q * 32 + lane < D) nbuf[q * 32 + lane] = nr[q];
    }
    __syncwarp();
    // C entries in column order: C index, slab offsets, product ranges; the
    // column's product cursor replaces its key in hkey, the entry's offset
    // within its work-item segment goes to dl
    long long run_p = 0, run_v = 0;
    for (int r0 = 0; r0 < D; r0 += 32) {
      const int r = r0 + lane;
      const bool ok = r < D;
      const uint32_t key = ok ? ord[r] : 0u;
      const int32_t col = static_cast<int32_t>(key >> 9);
      const int s = static_cast<int>(key & 511u);
      const uint32_t hc = ok ? hcnt[s] : 0u;
      const int np = static_cast<int>(hc & 0xffu);
      const int cin_l = static_cast<int>(hc >> 8) - 1;
      const int n = ok ? nbuf[r] : 0;
      const long long tv = ok ? t8_size(m, n) : 0;
      long long pi = np, vi = tv;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const long long py = __shfl_up_sync(0xffffffffu, pi, d);
        const long long vy = __shfl_up_sync(0xffffffffu, vi, d);
        if (lane >= d) {
          pi += py;
          vi += vy;
        }
      }
      if (ok) {
        const int32_t c = cbase + r;
        const long long p_ex = run_p + pi - np;
        g.out_col[c] = col;
        g.out_row[c] = static_cast<int32_t>(i);
        g.out_off[c] = vbase + run_v + vi - tv;
        g.cin_map[c] = cin_l >= 0 ? g.c_off[ci0 + cin_l] : -1;
        g.out_np[c] = np;
        g.out_p0[c] = pbase + p_ex;
        hkey[s] = static_cast<uint32_t>(p_ex);
        const int cls = shape_class(m, n, g.dmma_ok, g.tall_rows, g.tiny, g.wide);
        const int seg = cls * kMaxBands + band_of(col, g);
        dl[r] = static_cast<uint32_t>(
            tiles_add(&cls_n[seg], seg, static_cast<int>(n), static_cast<unsigned long long>(class_tiles(m, n, cls, g.tall_rows))));
      }
      run_p += __shfl_sync(0xffffffffu, pi, 31);
      run_v += __shfl_sync(0xffffffffu, vi, 31);
    }
    __syncwarp();
    // product descriptors: slot = column cursor + rank of the A entry among
    // the column's entries (k ascending)
    for (int kp = lane; kp < K; kp += 32) {
      const uint32_t info = pinfo[kp];
      const int s = static_cast<int>(info >> 8), lr = static_cast<int>(info & 0xffu);
      const int32_t p = static_cast<int32_t>(hkey[s]) + __popcll(hmask[s] & ((1ull << lr) - 1ull));
      BT_DASSERT(p >= 0 && pbase + p < g.prod_base[i + 1], "warp-row descriptor slot");
      g.desc[pbase + p] = make_int4(a_au[lr], pbu[kp], a_kc[lr], a_k[lr]);
    }
  }
  __syncthreads();
  // one reservation per (class, band) segment for the CTA's rows
  for (int t = threadIdx.x; t < NSEG; t += blockDim.x) {
    const unsigned long long k = cls_n[t];
    cls_at[t] = k ? atomicAdd(&g.class_cursor[t], k) : 0ull;
  }
  __syncthreads();
  if (!act) return;
  // work items (tall blocks become tall_rows-row tiles)
  long long run_v = 0;
  for (int r0 = 0; r0 < D; r0 += 32) {
    const int r = r0 + lane;
    const bool ok = r < D;
    const uint32_t key = ok ? ord[r] : 0u;
    const int32_t col = static_cast<int32_t>(key >> 9);
    const int s = static_cast<int>(key & 511u);
    const int n = ok ? nbuf[r] : 0;
    const long long tv = ok ? t8_size(m, n) : 0;
    long long vi = tv;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long vy = __shfl_up_sync(0xffffffffu, vi, d);
      if (lane >= d) vi += vy;
    }
    if (ok) {
      const uint32_t hc = hcnt[s];
      const int cin_l = static_cast<int>(hc >> 8) - 1;
      const int64_t c_off = vbase + run_v + vi - tv;
      const int64_t cin = cin_l >= 0 ? g.c_off[ci0 + cin_l] : -1;
      const int cls = shape_class(m, n, g.dmma_ok, g.tall_rows, g.tiny, g.wide);
      const int seg = cls * kMaxBands + band_of(col, g);
      const unsigned long long at = cls_at[seg] + dl[r];
      emit_items(g, at, m, n, cls, c_off, cin, pbase + static_cast<int64_t>(hkey[s]),
                 static_cast<int>(hc & 0xffu));
    }
    run_v += __shfl_sync(0xffffffffu, vi, 31);
  }
}

// K-panel work items (L2 blocking of long product chains):
// item t of panel p covers the products of base item t whose k block lies in
// [kb[p], kb[p+1]) -- a sub-range, products being in ascending k.  Panel 0
// initialises C_out from C_in; later panels accumulate in place (cin = c_out);
// an in-place item without products is skipped by the kernel.
__global__ void k_panel_items(const Item* __restrict__ base, int64_t nitems,
                              const Desc* __restrict__ desc, const int32_t* __restrict__ kb,
                              int npanels, Item* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nitems) return;
  const Item it = base[t];
  const int64_t p0 = item_p0(it);
  const int r8 = item_r8(it), c8 = item_c8(it);
  int64_t lo = p0;
  for (int p = 0; p < npanels; ++p) {
    // first product with k >= kb[p+1]
    int64_t a = lo, b = p0 + it.np;
    while (a < b) {
      const int64_t mid = (a + b) >> 1;
      if (desc[mid].w < kb[p + 1]) a = mid + 1; else b = mid;
    }
    Item q = it;
    q.p0r8 = item_pack(lo, r8, c8);
    q.np = static_cast<int32_t>(a - lo);
    if (p > 0) q.cin_off = it.c_off;
    out[p * nitems + t] = q;
    lo = a;
  }
}

// Work-item segment bases (exclusive scan of the per-segment counts) and zeroed
// ticket counters, written on the device: no host round trip before the fill.
// Warp 0 scans: lane l owns NSEG/32 consecutive segments (all loads issued at
// once), then a shuffle scan of the lane sums -- instead of one thread walking
// NSEG dependent entries.  Needs blockDim.x >= 32.
__device__ void init_cursors(const unsigned long long* __restrict__ seg_items,
                             unsigned long long* __restrict__ cursor) {
  constexpr int kPer = (NSEG + 31) / 32;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x, q0 = lane * kPer;
    unsigned long long v[kPer], sum = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      v[j] = q0 + j < NSEG ? seg_items[q0 + j] : 0ull;
      sum += v[j];
    }
    unsigned long long incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    unsigned long long run = incl - sum;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      if (q0 + j < NSEG) cursor[q0 + j] = run;
      run += v[j];
    }
  }
  for (int q = threadIdx.x; q < NCLASS; q += blockDim.x) cursor[NSEG + q] = 0ull;
}

// Exclusive scans of the three per-row arrays in one single-CTA kernel (M <=
// 8192 rows); element M receives the totals.  Thread t owns the PER
// consecutive rows [t*PER, t*PER + PER): it sums them, the three sums are
// scanned across the CTA in one pass (warp shuffles, then the 32 warp totals
// by warp 0), and it writes its rows' prefixes -- two barriers in all (the
// three CUB block scans per 1 024 rows took 8-15 us, spilling).
// The sizes block lives in mapped page-locked memory; once all of it is
// written, thread 0 publishes `seq` in `ready` (system-scope fence first), so
// the host can poll that word instead of waiting for the stream.
__device__ __forceinline__ void publish_sizes(volatile unsigned long long* ready,
                                              unsigned long long seq) {
  __threadfence_system();  // every writer's sizes visible to the host ...
  __syncthreads();
  if (threadIdx.x == 0 && ready) *ready = seq;  // ... before the flag
}

__global__ void __launch_bounds__(1024) k_scan_rows(const int32_t* __restrict__ nnz,
                                                    const int64_t* __restrict__ prod,
                                                    const int64_t* __restrict__ vals, int64_t M,
                                                    int32_t* __restrict__ rp,
                                                    int64_t* __restrict__ pb,
                                                    int64_t* __restrict__ vb,
                                                    const unsigned long long* __restrict__ tot,
                                                    int ntot,
                                                    unsigned long long* __restrict__ sizes,
                                                    unsigned long long* __restrict__ cursor,
                                                    volatile unsigned long long* ready,
                                                    unsigned long long seq) {
  __shared__ long long wsum[3][32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int per = static_cast<int>((M + 1023) / 1024);
  const int64_t r0 = static_cast<int64_t>(t) * per;
  const int64_t r1 = M < r0 + per ? M : r0 + per;
  long long s0 = 0, s1 = 0, s2 = 0;
  for (int64_t i = r0; i < r1; ++i) {
    s0 += nnz[i];
    s1 += prod[i];
    s2 += vals[i];
  }
  long long x0 = s0, x1 = s1, x2 = s2;  // inclusive warp scan
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const long long y0 = __shfl_up_sync(0xffffffffu, x0, d);
    const long long y1 = __shfl_up_sync(0xffffffffu, x1, d);
    const long long y2 = __shfl_up_sync(0xffffffffu, x2, d);
    if (lane >= d) {
      x0 += y0;
      x1 += y1;
      x2 += y2;
    }
  }
  if (lane == 31) {
    wsum[0][wid] = x0;
    wsum[1][wid] = x1;
    wsum[2][wid] = x2;
  }
  __syncthreads();
  if (wid == 0) {  // exclusive scan of the 32 warp totals, in place
    long long w0 = wsum[0][lane], w1 = wsum[1][lane], w2 = wsum[2][lane];
    long long i0 = w0, i1 = w1, i2 = w2;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long y0 = __shfl_up_sync(0xffffffffu, i0, d);
      const long long y1 = __shfl_up_sync(0xffffffffu, i1, d);
      const long long y2 = __shfl_up_sync(0xffffffffu, i2, d);
      if (lane >= d) {
        i0 += y0;
        i1 += y1;
        i2 += y2;
      }
    }
    wsum[0][lane] = i0 - w0;
    wsum[1][lane] = i1 - w1;
    wsum[2][lane] = i2 - w2;
    if (lane == 31) {  // totals: row M of the scans and the host readback block
      rp[M] = static_cast<int32_t>(i0);
      pb[M] = i1;
      vb[M] = i2;
      sizes[0] = static_cast<unsigned long long>(i0);
      sizes[1] = static_cast<unsigned long long>(i1);
      sizes[2] = static_cast<unsigned long long>(i2);
    }
  }
  __syncthreads();
  long long e0 = wsum[0][wid] + x0 - s0, e1 = wsum[1][wid] + x1 - s1, e2 = wsum[2][wid] + x2 - s2;
  for (int64_t i = r0; i < r1; ++i) {
    rp[i] = static_cast<int32_t>(e0);
    pb[i] = e1;
    vb[i] = e2;
    e0 += nnz[i];
    e1 += prod[i];
    e2 += vals[i];
  }
  for (int q = t; q < ntot; q += blockDim.x) sizes[3 + q] = tot[q];
  init_cursors(tot + 3, cursor);
  publish_sizes(ready, seq);
}

// Large-M variant of the readback block (after the CUB scans).
__global__ void k_pack_sizes(const int32_t* __restrict__ rp, const int64_t* __restrict__ pb,
                             const int64_t* __restrict__ vb, int64_t M,
                             const unsigned long long* __restrict__ tot, int ntot,
                             unsigned long long* __restrict__ sizes,
                             unsigned long long* __restrict__ cursor,
                             volatile unsigned long long* ready, unsigned long long seq) {
  if (threadIdx.x == 0) {
    sizes[0] = static_cast<unsigned long long>(rp[M]);
    sizes[1] = static_cast<unsigned long long>(pb[M]);
    sizes[2] = static_cast<unsigned long long>(vb[M]);
  }
  for (int t = threadIdx.x; t < ntot; t += blockDim.x) sizes[3 + t] = tot[t];
  init_cursors(tot + 3, cursor);
  publish_sizes(ready, seq);
}

// ------------------------------------------------------------------- host
namespace {

template <class TIn, class TOut>
void exclusive_scan(Ctx& x, const TIn* in, TOut* out, int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, x.stream);
  void* tmp = x.ensure_scratch(bytes);
  cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, n, x.stream);
  count_launch(&x, 2);
}

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }


constexpr int kWarps = 4;
using KernelFn = void (*)(const NumArgs);


template <int S>
KernelFn dmma_kernel_s(int cls) {
  static const KernelFn table[16] = {
      k_smm_dmma<1, 1, kWarps, S>, k_smm_dmma<1, 2, kWarps, S>, k_smm_dmma<1, 3, kWarps, S>,
      k_smm_dmma<1, 4, kWarps, S>, k_smm_dmma<2, 1, kWarps, S>, k_smm_dmma<2, 2, kWarps, S>,
      k_smm_dmma<2, 3, kWarps, S>, k_smm_dmma<2, 4, kWarps, S>, k_smm_dmma<3, 1, kWarps, S>,
      k_smm_dmma<3, 2, kWarps, S>, k_smm_dmma<3, 3, kWarps, S>, k_smm_dmma<3, 4, kWarps, S>,
      k_smm_dmma<4, 1, kWarps, S>, k_smm_dmma<4, 2, kWarps, S>, k_smm_dmma<4, 3, kWarps, S>,
      k_smm_dmma<4, 4, kWarps, S>};
  return table[cls];
}

// one launch for all DMMA classes of a mixed-size multiply: the smallest
// instantiation whose largest tile (TM x TN tiles of 8) covers every class
KernelFn dmma_multi_kernel(int maxm, int maxn, int& plan_cls) {
  if (maxm <= 3 && maxn <= 3) {
    plan_cls = 10;
    return k_smm_dmma<3, 3, kWarps, 1, true>;
  }
  if (maxn <= 3) {
    plan_cls = 14;
    return k_smm_dmma<4, 3, kWarps, 1, true>;
  }
  if (maxm <= 3) {
    plan_cls = 11;
    return k_smm_dmma<3, 4, kWarps, 1, true>;
  }
  plan_cls = 15;
  return k_smm_dmma<4, 4, kWarps, 1, true>;
}

KernelFn dmma_kernel(int cls, int stages) {
  return stages >= 2 ? dmma_kernel_s<2>(cls) : dmma_kernel_s<1>(cls);
}

// the K-panels-in-one-launch variant of a class
template <int S>
KernelFn dmma_panel_kernel_s(int cls) {
  static const KernelFn table[16] = {
      k_smm_dmma<1, 1, kWarps, S, false, true>, k_smm_dmma<1, 2, kWarps, S, false, true>,
      k_smm_dmma<1, 3, kWarps, S, false, true>, k_smm_dmma<1, 4, kWarps, S, false, true>,
      k_smm_dmma<2, 1, kWarps, S, false, true>, k_smm_dmma<2, 2, kWarps, S, false, true>,
      k_smm_dmma<2, 3, kWarps, S, false, true>, k_smm_dmma<2, 4, kWarps, S, false, true>,
      k_smm_dmma<3, 1, kWarps, S, false, true>, k_smm_dmma<3, 2, kWarps, S, false, true>,
      k_smm_dmma<3, 3, kWarps, S, false, true>, k_smm_dmma<3, 4, kWarps, S, false, true>,
      k_smm_dmma<4, 1, kWarps, S, false, true>, k_smm_dmma<4, 2, kWarps, S, false, true>,
      k_smm_dmma<4, 3, kWarps, S, false, true>, k_smm_dmma<4, 4, kWarps, S, false, true>};
  return table[cls];
}
KernelFn dmma_panel_kernel(int cls, int stages) {
  return stages >= 2 ? dmma_panel_kernel_s<2>(cls) : dmma_panel_kernel_s<1>(cls);
}

// Dynamic shared-memory opt-in per (device, kernel): the largest size set so
// far, raised when a launch needs more.  Thread-safe (one context per host
// thread may drive its own device).
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, size_t> g_smem_set;
std::map<std::tuple<int, const void*, size_t>, int> g_occ;

void ensure_dyn_smem(const void* fn, size_t bytes) {
  int dev = 0;
  BT_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_attr_mu);
  size_t& cur = g_smem_set[{dev, fn}];
  if (bytes > cur) {
    BT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bytes)));
    cur = bytes;
  }
}

// opt-in + occupancy query of a numeric kernel, cached per (device, kernel, smem)
int dmma_occupancy(KernelFn fn, size_t smem) {
  ensure_dyn_smem(reinterpret_cast<const void*>(fn), smem);
  int dev = 0;
  BT_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = g_occ.find({dev, reinterpret_cast<const void*>(fn), smem});
    if (it != g_occ.end()) return it->second;
  }
  int per_sm = 0;
  BT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kWarps * 32, smem));
  std::lock_guard<std::mutex> lk(g_attr_mu);
  g_occ[{dev, reinterpret_cast<const void*>(fn), smem}] = per_sm;
  return per_sm;
}

// Tickets per atomic of the numeric kernels.  Short items (about one product
// per C tile: c2, c4) are bound by the single ticket counter -- batches of up
// to 8 (about 8 batches per warp, so the tail stays short): c2 numeric 0.121
// -> 0.109 ms, c4 3.12 -> 2.93 ms.  Longer product chains (c1, c3) lose with
// batches (c1 0.619 -> 0.684 ms at 8: neighbouring tiles move to one warp), so
// they keep one ticket per item.  BT_TICKET_BATCH overrides.
int ticket_batch(int64_t tickets, int64_t warps, double products_per_ticket) {
  int64_t b = 1;
  if (products_per_ticket < 2.0 && warps > 0)
    b = std::max<int64_t>(1, std::min<int64_t>(8, tickets / (warps * 8)));
  return std::max(1, std::min(64, env_int("BT_TICKET_BATCH", static_cast<int>(b))));
}

struct Plan {
  int stages = 1;
  int stage_doubles = 0;
  int a_region = 0;
  size_t smem = 0;
};

// Shared-memory plan for one DMMA class: per warp `stages` buffers holding one
// A slab (TMT x KT tiles) and one B block (KT x TNT tiles).  Measured on c1
// (profiles/): resident warps matter more than ring depth, so the default is
// the deepest ring that keeps 24 warps/SM, at least 1.
Plan plan_dmma(int cls, int ktmax) {
  Plan P;
  const int TMT = cls / 4 + 1, TNT = cls % 4 + 1;
  P.a_region = TMT * ktmax * 64;
  P.stage_doubles = P.a_region + ktmax * TNT * 64;
  const size_t per_stage = static_cast<size_t>(P.stage_doubles) * 8;
  const size_t budget = 220 * 1024;
  const int want_warps = env_int("BT_WARPS_PER_SM", 24);
  int s = env_int("BT_STAGES", 0);
  if (s <= 0) {
    s = 2;
    while (s > 1 && static_cast<size_t>(want_warps) * (s * per_stage + 1536) > budget) --s;
  }
  P.stages = std::max(1, std::min(s, 2));
  P.smem = kWarps * 1536 + static_cast<size_t>(kWarps) * P.stages * per_stage;
  return P;
}

}  // namespace

}  // namespace bt

using namespace bt;

// The local multiply C += A*B (one rank's stores); throws bt::Error.
void bt::local_multiply(Ctx& x, const Mat& A, const Mat& B, Mat& Cm, double eps, bt_stats* stats,
                        cudaEvent_t wait_numeric, cudaEvent_t numeric_start,
                        const std::function<void()>* after_sizes, bool sync_at_end,
                        bool poll_sizes) {
  {
    BT_REQUIRE(A.ctx == &x && B.ctx == &x && Cm.ctx == &x, BT_ERR_INVALID_ARGUMENT,
               "bt_multiply: matrices belong to another context");
    // conformity (multiply_cannon.hpp:70-73, multiply_rect.hpp:106-112)
    BT_REQUIRE(A.h_csz == B.h_rsz, BT_ERR_INVALID_ARGUMENT,
               "multiply: inner blockings of A and B differ");
    BT_REQUIRE(Cm.h_rsz == A.h_rsz && Cm.h_csz == B.h_csz, BT_ERR_INVALID_ARGUMENT,
               "multiply: C blockings do not conform");
    BT_REQUIRE(&Cm != &A && &Cm != &B, BT_ERR_INVALID_ARGUMENT,
               "multiply: C must not alias A or B");
    BT_CUDA(cudaSetDevice(x.device));
    Trace tr("multiply");
    cudaStream_t st = x.stream;
    const int64_t k0 = x.kernels;
    bt_stats S{};
    S.c_blocks_in = Cm.nblk;
    if (x.timing) BT_CUDA(cudaEventRecord(x.ev[0], st));
    const int64_t M = Cm.nbr, N = Cm.nbc;
    // Symbolic passes: per-column counters of one C row live in shared memory,
    // for a chunk of `colw` block columns at a time (rows wider than that are
    // swept chunk by chunk; any N works).  Fill pass: 3 ints per column
    // (counts, cursors, touched list) + bitmap, + 8 bytes per column for the
    // rank emission (colmask) on narrow matrices, + 4 for split CTAs.
    int64_t colw = N <= 14000 ? std::max<int64_t>(N, 1) : 8192;
    colw = std::max<int64_t>(1, std::min<int64_t>(colw, env_int("BT_COLW", 1 << 30)));
    const int64_t W = colw;
    size_t row_smem = static_cast<size_t>(W) * 12 + 4 * ((W + 31) / 32);
    const bool colmask = W <= 4096 && env_int("BT_COLMASK", 1);
    if (colmask) row_smem = 4 * ((3 * W + (W + 31) / 32 + 1) & ~int64_t(1)) + 8 * W;
    // few long C rows (c3: 100 rows of ~2000 A entries): several fill CTAs per
    // row, each emitting a range of A chunks (+4 bytes per column of counts)
    int fill_splits = 1;
    if (M > 0 && M < 2 * x.num_sms) {
      const int64_t chunks = (A.nblk / M + kChunkA - 1) / kChunkA;
      fill_splits = static_cast<int>(std::min<int64_t>(8, std::max<int64_t>(1, chunks / 2)));
    }
    fill_splits = std::min(64, std::max(1, env_int("BT_FILL_SPLITS", fill_splits)));
    // threads per row of the symbolic passes: 64 for many short rows (few A
    // entries, few pairs: c2, c4 -- four times the rows in flight), else 256
    const double a_per_row = M ? static_cast<double>(A.nblk) / static_cast<double>(M) : 0.0;
    const double b_per_row = A.nbc ? static_cast<double>(B.nblk) / static_cast<double>(A.nbc) : 0.0;
    // (and only while a row's column counters stay small: the 64-thread fill
    // pays off with >= ~10 resident CTAs per SM -- c4 pass 1 165 -> 83 us,
    // fill 229 -> 112 us; c2, whose 1 463-column counters take 29 KB, gains
    // nothing, profiles/r02/row_threads_ab.txt)
    int row_threads = (a_per_row <= 48.0 && a_per_row * b_per_row <= 384.0 &&
                       M >= 2 * x.num_sms && row_smem <= 12 * 1024) ? 64 : 256;
    {
      const int rt = env_int("BT_ROW_THREADS", row_threads);
      row_threads = rt == 64 ? 64 : rt == 512 ? 512 : 256;
    }
    if (row_threads == 64) fill_splits = 1;
    // warp-per-row fill for short rows (one warp per C row, a hash of the
    // row's columns instead of dense per-column arrays): H = 128 for ~<= 48
    // candidate pairs per row (c4), 256 up to ~120 (or ~240 with an eps
    // filter, which keeps a fraction of them: c2); pass 1 lists the rows that
    // do not fit for the CTA fill (BT_WARP_ROWS=0/128/256 overrides)
    int wrow_h = 0;
    {
      const double pairs = a_per_row * b_per_row;
      if (N < (int64_t(1) << 23) && a_per_row <= 24.0 && M >= x.num_sms) {
        if (pairs <= 48.0) wrow_h = 128;
        else if (pairs <= (eps > 0 ? 240.0 : 120.0)) wrow_h = 256;
      }
      const int e = env_int("BT_WARP_ROWS", -1);
      if (e == 0 || e == 128 || e == 256) wrow_h = e;
      if (N >= (int64_t(1) << 23)) wrow_h = 0;
    }
    if (wrow_h) fill_splits = 1;  // (the list fill takes one CTA per left-over row)
    BT_REQUIRE(row_smem <= 180 * 1024, BT_ERR_INTERNAL, "multiply: column chunk too wide");
    // split CTAs need 4 more bytes per column; if that does not fit, one CTA
    // per row
    if (fill_splits > 1 && row_smem + 4 * static_cast<size_t>(W) > 180 * 1024) fill_splits = 1;
    if (fill_splits > 1) row_smem += 4 * static_cast<size_t>(W);
    // split-count mode (few long rows, one column chunk): pass 1 counts each
    // fill CTA's range of A chunks in its own CTA and keeps the per-range
    // column counts, so the fill CTAs of a row do not recount the row
    const bool snap_mode = fill_splits > 1 && N <= colw && env_int("BT_SNAP", 1) != 0 &&
                           static_cast<double>(M) * (fill_splits + 1) * static_cast<double>(N) * 4.0 <= 64e6;
    if (snap_mode) row_threads = 256;
    // (the 512-thread fill's pair caches must fit beside the column arrays)
    if (row_threads == 512 && row_smem + 16 + 10 * static_cast<size_t>(pair_cap<512>()) > 180 * 1024)
      row_threads = 256;
    size_t pair_off = 0;
    if (row_threads == 512) {  // the 512-thread fill keeps its pair caches here
      pair_off = (row_smem + 15) & ~size_t(15);
      row_smem = pair_off + 10 * static_cast<size_t>(pair_cap<512>());
    }

    // ---- norms for the eps filter, cached with the stores: a
    // store's norms are computed once after it changes (both in one launch
    // when A and B are both stale)
    const double *na = nullptr, *nb = nullptr;
    if (eps > 0 && A.nblk && B.nblk) {
      if (!A.norms_ok && !B.norms_ok && &A != &B) {
        if (A.norm_cache.n < static_cast<size_t>(A.nblk)) A.norm_cache.alloc(A.nblk, st);
        if (B.norm_cache.n < static_cast<size_t>(B.nblk)) B.norm_cache.alloc(B.nblk, st);
        const NormSrc sa{A.vals.p, A.row_ptr.p, A.col.p, A.off.p, A.rsz.p, A.csz.p, A.nbr,
                         A.norm_cache.p, A.nblk};
        const NormSrc sb{B.vals.p, B.row_ptr.p, B.col.p, B.off.p, B.rsz.p, B.csz.p, B.nbr,
                         B.norm_cache.p, B.nblk};
        k_block_norms_pair<<<blocks_for((A.nblk + B.nblk) * 32, kNormThreads), kNormThreads, 0, st>>>(
            sa, sb);
        check_launch("block_norms");
        count_launch(&x);
        A.norms_ok = B.norms_ok = true;
      }
      na = A.norms(st);
      nb = B.norms(st);
    }

    // work items address row tiles of 8 in 13 bits (bt_smm.cuh Item)
    BT_REQUIRE(Cm.max_r <= 8 * kItemMaxR8, BT_ERR_INVALID_ARGUMENT,
               "multiply: blocks taller than 65 528 rows are not supported");
    const int kmax = A.max_c;
    // WIDE DMMA path: blocks wider than 32 columns as
    // 32-column tiles, k of any size in slices -- every block on the tensor
    // cores.  BT_WIDE=0 (or blocks beyond the item encoding) keeps the
    // CUDA-core generic kernel for n > 32 or k > 64.
    const bool wide = env_int("BT_WIDE", 1) != 0 && Cm.max_c <= 8 * kItemMaxC8 &&
                      Cm.max_r <= 8 * kItemMaxR8;
    const bool dmma_ok = wide || kmax <= 64;
    // the WIDE kernel is launched only when some block needs it
    const bool wide_k = wide && (Cm.max_c > 32 || kmax > 64);
    RowArgs ra{};
    ra.a_rp = A.row_ptr.p;
    ra.a_col = A.col.p;
    ra.b_rp = B.row_ptr.p;
    ra.b_col = B.col.p;
    ra.c_rp = Cm.row_ptr.p;
    ra.c_col = Cm.col.p;
    ra.a_off = A.off.p;
    ra.b_off = B.off.p;
    ra.c_off = Cm.off.p;
    ra.m_sz = Cm.rsz.p;
    ra.n_sz = Cm.csz.p;
    ra.k_sz = A.csz.p;
    ra.na = na;
    ra.nb = nb;
    ra.eps = eps;
    ra.ncols = N;
    ra.dmma_ok = dmma_ok;
    ra.wide = wide;
    ra.sort_min = env_int("BT_SORT_MIN", 48);
    ra.colmask = colmask;
    ra.tall_rows = env_int("BT_TALL_ROWS", 32) == 24 ? 24 : 32;
    // tiny C blocks (m, n <= 5) go to the DFMA kernel when every C block is
    // tiny; in a mixed basis they ride along in the MULTI DMMA launch, which
    // (with batched tickets) beats the DFMA kernel beside it: c2 numeric
    // 108 -> 102 us (the DFMA grid only gets SMs in the MULTI tail, and
    // launched first it slows the sweep to 145 us).  BT_DFMA=0/1 forces.
    {
      const bool all_tiny = Cm.max_r <= kTinyMax && Cm.max_c <= kTinyMax;
      ra.tiny = env_int("BT_DFMA", all_tiny ? 1 : 0) != 0;
    }
    ra.splits = fill_splits;
    ra.pair_smem_off = static_cast<int64_t>(pair_off);
    ra.snap = snap_mode ? x.ws<int32_t>(13, static_cast<size_t>(M) * (fill_splits + 1) * N) : nullptr;
    ra.colw = colw;
    {
      // column bands: when A and B together overflow a comfortable share of L2
      // (but are not in the K-panel regime below), sweep C in bands of B
      // columns so B(:, band) stays L2-resident; A is then streamed once per band
      const double a_bytes = 8.0 * static_cast<double>(A.nvals);
      const double b_bytes = 8.0 * static_cast<double>(B.nvals);
      int nb_ = 1;
      if (a_bytes + b_bytes > 96e6 && a_bytes + b_bytes <= 2.0 * 126e6)
        nb_ = static_cast<int>(std::ceil(b_bytes / 40e6));
      nb_ = env_int("BT_BANDS", nb_);
      ra.nbands = static_cast<int>(std::min<int64_t>(std::max(1, std::min(nb_, kMaxBands)),
                                                     std::max<int64_t>(N, 1)));
    }

    // ---- pass 1: sizes (the one host synchronisation)
    DBuf<int32_t> out_rp(M + 1, st);
    int32_t* row_nnz = x.ws<int32_t>(0, M + 1);
    int64_t* row_prod = x.ws<int64_t>(1, M + 1);
    int64_t* row_vals = x.ws<int64_t>(2, M + 1);
    int64_t* prod_base = x.ws<int64_t>(3, M + 1);
    int64_t* val_base = x.ws<int64_t>(4, M + 1);
    // [0..3) totals, [3, 3 + NSEG) work items per segment, [3 + NSEG] rows
    // the warp-row pass left to the CTA kernels
    constexpr int kTot = 4 + NSEG;
    unsigned long long* tot = x.ws<unsigned long long>(5, kTot);
    BT_CUDA(cudaMemsetAsync(tot, 0, sizeof(unsigned long long) * kTot, st));
    // sizes for the host: written by the scan kernel straight into mapped
    // page-locked memory (a copy-engine D2H would queue behind an
    // asynchronous export's transfer)
    unsigned long long* dsizes = reinterpret_cast<unsigned long long*>(x.pinned_dev);
    // the scan kernel publishes `seq` in this mapped word once the sizes are in
    // place: the host polls it (no stream-synchronize wake-up latency)
    volatile unsigned long long* ready_host = reinterpret_cast<volatile unsigned long long*>(
        static_cast<char*>(x.pinned) + Ctx::kPinnedFlag);
    volatile unsigned long long* ready_dev = reinterpret_cast<volatile unsigned long long*>(
        static_cast<char*>(x.pinned_dev) + Ctx::kPinnedFlag);
    const unsigned long long seq = ++x.size_seq;
    unsigned long long* cursor = x.ws<unsigned long long>(18, NSEG + NCLASS);
    ra.row_nnz = row_nnz;
    ra.row_prod = row_prod;
    ra.row_vals = row_vals;
    ra.totals = tot;
    ra.class_items = tot + 3;
    ra.wflag = wrow_h ? x.ws<int32_t>(11, M) : nullptr;
    ra.wlist = x.ws<int32_t>(12, M);
    ra.wlist_n = tot + 3 + NSEG;
    ra.wcap_k = 2 * wrow_h;
    ra.wcap_d = 3 * wrow_h / 4;
    const size_t sm1 = static_cast<size_t>(W) * 8 + 4 * ((W + 31) / 32);
    if (M > 0) {
      // static + dynamic shared memory may exceed the 48 KB default: always opt in
      // pass 1's CTA width: the fill's, except 128 for short rows that 256-thread
      // CTAs would spread over more than one wave (c2: 1 463 rows of ~215
      // pairs, pass 1 + scan 37 -> 29 us; c1's 1 600-pair rows keep 256, c4 64)
      int ct = row_threads;
      if (row_threads == 256 && a_per_row * b_per_row <= 512.0 && M >= 6 * x.num_sms) ct = 128;
      ct = env_int("BT_COUNT_THREADS", ct);
      if (ra.snap) ct = 256;
      auto count_fn = ra.snap     ? k_row_count_snap<256>
                      : ct == 64  ? k_row_count<64>
                      : ct == 128 ? k_row_count<128>
                      : ct == 512 ? k_row_count<512>
                                  : k_row_count<256>;
      const int count_threads = (ct == 64 || ct == 128 || ct == 512) ? ct : 256;
      ensure_dyn_smem(reinterpret_cast<const void*>(count_fn), sm1);
      if (ra.snap) {
        const size_t smn = 4 * static_cast<size_t>(N);
        ensure_dyn_smem(reinterpret_cast<const void*>(k_row_count_split<256>), smn);
        k_row_count_split<256><<<static_cast<unsigned>(M * fill_splits), 256, smn, st>>>(ra);
        check_launch("row_count_split");
        count_launch(&x);
      }
      count_fn<<<static_cast<unsigned>(M), count_threads, sm1, st>>>(ra);
      check_launch("row_count");
      count_launch(&x);
    }
    if (M <= 8192) {
      k_scan_rows<<<1, 1024, 0, st>>>(row_nnz, row_prod, row_vals, M, out_rp.p, prod_base,
                                      val_base, tot, kTot, dsizes, cursor, ready_dev, seq);
      check_launch("scan_rows");
      count_launch(&x);
    } else {
      BT_CUDA(cudaMemsetAsync(row_nnz + M, 0, sizeof(int32_t), st));
      BT_CUDA(cudaMemsetAsync(row_prod + M, 0, sizeof(int64_t), st));
      BT_CUDA(cudaMemsetAsync(row_vals + M, 0, sizeof(int64_t), st));
      exclusive_scan(x, row_nnz, out_rp.p, M + 1);
      exclusive_scan(x, row_prod, prod_base, M + 1);
      exclusive_scan(x, row_vals, val_base, M + 1);
      k_pack_sizes<<<1, 256, 0, st>>>(out_rp.p, prod_base, val_base, M, tot, kTot, dsizes,
                                      cursor, ready_dev, seq);
      check_launch("pack_sizes");
      count_launch(&x);
    }
    struct Sizes {
      unsigned long long nout, nprod, nvals;
      unsigned long long tot[kTot];
    };
    static_assert(sizeof(Sizes) <= 2048, "pinned staging");
    // the scan kernel wrote the sizes into mapped pinned memory (no D2H copy)
    Sizes& h = *reinterpret_cast<Sizes*>(x.pinned);
    const bool phases = x.timing && env_int("BT_PHASES", 0);
    if (phases) BT_CUDA(cudaEventRecord(x.ev[4], st));
    tr.mark("pass1 enqueued");
    const int poll_mode = env_int("BT_POLL_SIZES", 1);  // 0 off, 1 single-GPU calls, 2 all
    if (M > 0 && ((poll_sizes && poll_mode == 1) || poll_mode == 2)) {
      // poll the flag; after 20 ms fall back to the stream wait (which also
      // reports a failed kernel)
      const double t_start = Trace::now();
      unsigned spins = 0;
      while (*ready_host != seq) {
        if ((++spins & 4095u) == 0 && Trace::now() - t_start > 20.0) break;
      }
      if (*ready_host != seq) BT_CUDA(cudaStreamSynchronize(st));
      std::atomic_thread_fence(std::memory_order_acquire);
    } else {
      BT_CUDA(cudaStreamSynchronize(st));
    }
    tr.mark("pass1 sync");
    // caller's check between the sizes and any use of B's values (the
    // speculative case-2 gather confirms its segments here, or throws)
    if (after_sizes) (*after_sizes)();
    const int64_t nout = static_cast<int64_t>(h.nout), nprod = static_cast<int64_t>(h.nprod),
                  nvals = static_cast<int64_t>(h.nvals);
    S.candidates = static_cast<int64_t>(h.tot[0]);
    S.flops = 2.0 * static_cast<double>(h.tot[1]);
    S.products = nprod;
    const int64_t nelems = static_cast<int64_t>(h.tot[2]);
    BT_REQUIRE(nprod < (int64_t(1) << kItemP0Bits), BT_ERR_INVALID_ARGUMENT, "too many products");
    BT_REQUIRE(A.nvals / 64 < (int64_t(1) << 31) && B.nvals / 64 < (int64_t(1) << 31),
               BT_ERR_INVALID_ARGUMENT, "multiply: operand slab exceeds 2^31 tiles");

    // ---- pass 2: C_out pattern, product stacks (descriptors)
    // An empty C (no C_in blocks: nothing reads its col/off/vals) hands its
    // buffers over as the outputs when they are large enough -- a repeated
    // clear + multiply then allocates nothing
    const bool reuse_c = Cm.nblk == 0;
    DBuf<int32_t> out_col;
    DBuf<int64_t> out_off;
    if (reuse_c && Cm.col.n >= static_cast<size_t>(std::max<int64_t>(nout, 1)) &&
        Cm.off.n >= static_cast<size_t>(std::max<int64_t>(nout, 1))) {
      out_col = std::move(Cm.col);
      out_off = std::move(Cm.off);
    } else {
      out_col.alloc(std::max<int64_t>(nout, 1), st);
      out_off.alloc(std::max<int64_t>(nout, 1), st);
    }
    int32_t* out_row = x.ws<int32_t>(6, nout);
    int32_t* out_np = x.ws<int32_t>(7, nout);
    int64_t* cin_map = x.ws<int64_t>(8, nout);
    int64_t* out_p0 = x.ws<int64_t>(9, nout);
    Desc* desc = x.ws<Desc>(10, nprod);
    ra.out_rp = out_rp.p;
    ra.prod_base = prod_base;
    ra.val_base = val_base;
    ra.out_col = out_col.p;
    ra.out_row = out_row;
    ra.out_off = out_off.p;
    ra.cin_map = cin_map;
    ra.out_np = out_np;
    ra.out_p0 = out_p0;
    ra.desc = desc;
    // work-item segments per tile class (sizes from pass 1)
    std::array<int64_t, NSEG + 1> sbound{};
    for (int q = 0; q < NSEG; ++q) sbound[q + 1] = sbound[q] + static_cast<int64_t>(h.tot[3 + q]);
    std::array<int64_t, NCLASS + 1> ibound{};
    for (int q = 0; q <= NCLASS; ++q) ibound[q] = sbound[q * kMaxBands];
    const int64_t nitems = ibound[NCLASS];
    Item* items = x.ws<Item>(17, nitems);
    ra.class_cursor = cursor;
    ra.items = items;
    ra.nprod_total = nprod;
    ra.nitems_total = nitems;
    if (phases) BT_CUDA(cudaEventRecord(x.ev[5], st));
    const int64_t nleft = wrow_h ? static_cast<int64_t>(h.tot[3 + NSEG]) : 0;
    if (env_int("BT_TRACE", 0) && wrow_h)
      fprintf(stderr, "[bt] warp-row fill (H=%d): %lld of %lld rows left to the CTA fill\n",
              wrow_h, static_cast<long long>(nleft), static_cast<long long>(M));
    if (nout > 0 && wrow_h) {
      const unsigned grid = static_cast<unsigned>((M + kWRows - 1) / kWRows);
      const size_t smw = static_cast<size_t>(kWRows) *
                         (wrow_h == 128 ? wrow_fill_bytes<128>() : wrow_fill_bytes<256>());
      auto wfn = wrow_h == 128 ? k_wrow_fill<128> : k_wrow_fill<256>;
      ensure_dyn_smem(reinterpret_cast<const void*>(wfn), smw);
      wfn<<<grid, kWRows * 32, smw, st>>>(ra, M);
      check_launch("wrow_fill");
      count_launch(&x);
      if (nleft > 0) {
        ensure_dyn_smem(reinterpret_cast<const void*>(k_row_fill_list<256>), row_smem);
        k_row_fill_list<256><<<static_cast<unsigned>(std::min<int64_t>(nleft, 4 * x.num_sms)), 256, row_smem,
                          st>>>(ra);
        check_launch("row_fill_list");
        count_launch(&x);
      }
    } else if (nout > 0) {
      auto fill_fn = row_threads == 64    ? k_row_fill<64>
                     : row_threads == 512 ? k_row_fill<512>
                                          : k_row_fill<256>;
      ensure_dyn_smem(reinterpret_cast<const void*>(fill_fn), row_smem);
      fill_fn<<<static_cast<unsigned>(M * fill_splits), row_threads, row_smem, st>>>(ra);
      check_launch("row_fill");
      count_launch(&x);
    }

    tr.mark("pass2 enqueued");
    // ---- numeric phase: one kernel per tile class, classes run concurrently
    DBuf<double> new_vals;
    if (reuse_c && Cm.vals.n >= static_cast<size_t>(std::max<int64_t>(nvals, 64)))
      new_vals = std::move(Cm.vals);
    else
      new_vals.alloc(std::max<int64_t>(nvals, 64), st);
    tr.mark("C slab");
    if (nout > 0) {
      NumArgs g{};
      g.npanels = 1;
      g.items = items;
      g.desc = desc;
      g.at = A.vals.p;
      g.bt = B.vals.p;
      g.cin = Cm.vals.p;
      g.cout = new_vals.p;
      g.a_len = A.nvals;
      g.b_len = B.nvals;
      g.cin_len = Cm.nvals;
      g.cout_len = nvals;
      unsigned long long* counters = cursor + NSEG;
      // K panels: when the operands are far larger than L2, C is comparatively
      // small and product chains are long (the case-1 regime: S_C << S_A, S_B),
      // the numeric phase walks K in panels whose A/B slices fit L2 and
      // accumulates C in place between panels
      const double ab_bytes = 8.0 * static_cast<double>(A.nvals + B.nvals);
      const double c_bytes = 8.0 * static_cast<double>(nvals);
      int npanels = 1;
      if (ab_bytes > 2.0 * 126e6 && nitems > 0) {
        // one DMMA class: all panels in one launch (no per-panel tail), so
        // panels of ~100 MB of A/B (c3 sweep: 10 % best at 12-20 panels, 50 %
        // at 64); several classes: one launch per panel, fewer and larger
        int present = 0;
        for (int q = 0; q < NCLASS; ++q) present += ibound[q + 1] > ibound[q];
        const bool one = present == 1 && ibound[GENERIC] > ibound[0];
        const double per_tile = static_cast<double>(nprod) / static_cast<double>(nitems);
        int p = static_cast<int>(std::ceil(ab_bytes / (one ? 100e6 : 60e6)));
        p = std::min(p, static_cast<int>(per_tile / 4));          // >= ~4 products/panel
        p = std::min(p, static_cast<int>((one ? 0.5 : 0.25) * ab_bytes / c_bytes));  // C traffic
        p = std::min(p, one ? 64 : 32);
        npanels = std::max(1, p);
      }
      if (nitems > 0) npanels = std::min(64, std::max(1, env_int("BT_KPANELS", npanels)));
      if (env_int("BT_TRACE", 0))
        fprintf(stderr, "[bt] numeric: %lld items, %lld products, %d K panel(s)\n",
                static_cast<long long>(nitems), static_cast<long long>(nprod), npanels);
      Item* pitems = items;
      if (npanels > 1) {
        std::vector<int32_t> kb(npanels + 1);
        for (int q = 0; q <= npanels; ++q)
          kb[q] = static_cast<int32_t>((A.nbc * q) / npanels);
        kb[npanels] = INT32_MAX;
        int32_t* d_kb = x.ws<int32_t>(20, npanels + 1);
        BT_CUDA(cudaMemcpyAsync(d_kb, kb.data(), 4 * (npanels + 1), cudaMemcpyHostToDevice, st));
        pitems = x.ws<Item>(19, static_cast<size_t>(npanels) * nitems);
        k_panel_items<<<blocks_for(nitems, 256), 256, 0, st>>>(items, nitems, desc, d_kb, npanels,
                                                               pitems);
        check_launch("panel_items");
        count_launch(&x);
      }
      if (phases) BT_CUDA(cudaEventRecord(x.ev[6], st));
      if (wait_numeric) BT_CUDA(cudaStreamWaitEvent(st, wait_numeric, 0));
      if (numeric_start) BT_CUDA(cudaEventRecord(numeric_start, st));
      if (x.timing) BT_CUDA(cudaEventRecord(x.ev[1], st));
      // panels of a single DMMA class run as ONE launch (per-tile flags order
      // the in-place accumulation; one tail instead of one per panel)
      int only = -1, present = 0;
      for (int q = 0; q < NCLASS; ++q)
        if (ibound[q + 1] > ibound[q]) {
          only = q;
          ++present;
        }
      const bool fused = npanels > 1 && present == 1 && only < GENERIC && !wide_k &&
                         env_int("BT_PANEL_FUSE", 1) != 0;
      if (fused) {
        const int q = only;
        const int64_t lo = ibound[q], hi = ibound[q + 1];
        const int ktmax = std::max(1, tiles8(kmax));
        const Plan P = plan_dmma(q, ktmax);
        g.stages = P.stages;
        g.stage_doubles = P.stage_doubles;
        g.a_region = P.a_region;
        g.items = pitems;
        g.item_lo = lo;
        g.nitems = hi - lo;
        g.npanels = npanels;
        g.panel_stride = nitems;
        g.tile_flag = x.ws<int>(21, nitems) + lo;
        BT_CUDA(cudaMemsetAsync(x.ws<int>(21, nitems), 0, 4 * nitems, st));
        g.counter = counters + q;
        KernelFn fn = dmma_panel_kernel(q, P.stages);
        const int per_sm = dmma_occupancy(fn, P.smem);
        BT_REQUIRE(per_sm >= 1, BT_ERR_INTERNAL, "smm_dmma: kernel does not fit on an SM");
        const int64_t grid = std::min<int64_t>(static_cast<int64_t>(x.num_sms) * per_sm,
                                               (hi - lo + kWarps - 1) / kWarps);
        // K panels in one launch: one ticket per atomic -- batches let a warp
        // hold tickets of a later panel while it waits on the earlier one
        // (c3 10 %: 1.73 -> 2.81 ms with batches of 6)
        g.ticket_batch = 1;
        fn<<<static_cast<unsigned>(grid), kWarps * 32, P.smem, st>>>(g);
        check_launch("smm_dmma_panels");
        count_launch(&x);
      }
      for (int panel = 0; panel < (fused ? 0 : npanels); ++panel) {
      g.items = pitems + static_cast<int64_t>(panel) * nitems;
      if (panel > 0) {  // later panels accumulate into C_out in place
        g.cin = g.cout;
        BT_CUDA(cudaMemsetAsync(counters, 0, sizeof(unsigned long long) * NCLASS, st));
      }
      const int ktmax = std::max(1, tiles8(kmax));
      int nclasses = 0;
      for (int q = 0; q < NCLASS; ++q) nclasses += ibound[q + 1] > ibound[q];
      // several classes (mixed block sizes): all DMMA classes in ONE launch of
      // the MULTI kernel (per-item tile dispatch; BT_MULTI=0: one kernel per
      // class on side streams); the generic class beside it
      int maxm = 0, maxn = 0;
      for (int q = 0; q < GENERIC; ++q)
        if (ibound[q + 1] > ibound[q]) {
          maxm = std::max(maxm, q / 4 + 1);
          maxn = std::max(maxn, q % 4 + 1);
        }
      // (wide_k: every DMMA class in one WIDE launch, even a single class)
      const bool multi = maxm > 0 && (wide_k || (nclasses > 1 && env_int("BT_MULTI", 1) != 0));
      const bool fork = nclasses > 1;
      const int nstreams = std::min(nclasses, Ctx::kAux);
      if (fork) {
        BT_CUDA(cudaEventRecord(x.ev_fork, st));
        for (int a = 0; a < nstreams; ++a) BT_CUDA(cudaStreamWaitEvent(x.aux[a], x.ev_fork, 0));
      }
      if (multi) {
        int pcls = 15;
        KernelFn fn = wide_k ? k_smm_dmma<4, 4, kWarps, 1, true, false, true>
                             : dmma_multi_kernel(maxm, maxn, pcls);
        // stage plan of the largest tile (WIDE: k slices of <= kKTCap tiles)
        const Plan P = plan_dmma(pcls, wide_k ? std::min(ktmax, kKTCap) : ktmax);
        g.stages = 1;
        g.stage_doubles = P.stage_doubles;
        g.a_region = P.a_region;
        const size_t smem = kWarps * 1536 + static_cast<size_t>(kWarps) * P.stage_doubles * 8;
        g.item_lo = ibound[0];
        g.nitems = ibound[GENERIC] - ibound[0];
        g.counter = counters;  // class 0's ticket counter serves the single launch
        const int per_sm = dmma_occupancy(fn, smem);
        BT_REQUIRE(per_sm >= 1, BT_ERR_INTERNAL, "smm_dmma: kernel does not fit on an SM");
        const int64_t grid = std::min<int64_t>(static_cast<int64_t>(x.num_sms) * per_sm,
                                               (g.nitems + kWarps - 1) / kWarps);
        g.ticket_batch = ticket_batch(g.nitems, grid * kWarps,
                                      static_cast<double>(nprod) / std::max<int64_t>(nitems, 1));
        fn<<<static_cast<unsigned>(grid), kWarps * 32, smem, fork ? x.aux[0] : st>>>(g);
        check_launch("smm_dmma_multi");
        count_launch(&x);
      }
      int launched = multi ? 1 : 0;
      for (int q = 0; q < NCLASS; ++q) {
        const int64_t lo = ibound[q], hi = ibound[q + 1];
        if (hi <= lo) continue;
        if (multi && q < GENERIC) continue;  // (the MULTI launch covers every DMMA class)
        cudaStream_t ks = fork ? x.aux[launched % nstreams] : st;
        ++launched;
        g.item_lo = lo;
        g.nitems = hi - lo;
        g.counter = counters + q;
        if (q == GENERIC) {
          k_smm_generic<<<static_cast<unsigned>(hi - lo), 256, 0, ks>>>(g, A.csz.p);
          check_launch("smm_generic");
          count_launch(&x);
          continue;
        }
        if (q == TINY) {  // CUDA-core DFMA, one thread per C block
          const bool four = A.max_r <= 4 && B.max_c <= 4;
          (four ? k_smm_dfma<4, 4> : k_smm_dfma<kTinyMax, kTinyMax>)
              <<<blocks_for(hi - lo, 128), 128, 0, ks>>>(g, A.csz.p);
          check_launch("smm_dfma");
          count_launch(&x);
          continue;
        }
        const Plan P = plan_dmma(q, ktmax);
        g.stages = P.stages;
        g.stage_doubles = P.stage_doubles;
        g.a_region = P.a_region;
        KernelFn fn = dmma_kernel(q, P.stages);
        const int per_sm = dmma_occupancy(fn, P.smem);
        BT_REQUIRE(per_sm >= 1, BT_ERR_INTERNAL, "smm_dmma: kernel does not fit on an SM");
        const int64_t grid = std::min<int64_t>(static_cast<int64_t>(x.num_sms) * per_sm,
                                               (hi - lo + kWarps - 1) / kWarps);
        g.ticket_batch = ticket_batch(g.nitems, grid * kWarps,
                                      static_cast<double>(nprod) / std::max<int64_t>(nitems, 1));
        fn<<<static_cast<unsigned>(grid), kWarps * 32, P.smem, ks>>>(g);
        check_launch("smm_dmma");
        count_launch(&x);
      }
      if (fork)
        for (int a = 0; a < nstreams; ++a) {
          BT_CUDA(cudaEventRecord(x.ev_join[a], x.aux[a]));
          BT_CUDA(cudaStreamWaitEvent(st, x.ev_join[a], 0));
        }
      }  // panels
      if (x.timing) BT_CUDA(cudaEventRecord(x.ev[2], st));
    }

    // ---- install C_out
    Cm.vals = std::move(new_vals);
    Cm.row_ptr = std::move(out_rp);
    Cm.col = std::move(out_col);
    Cm.off = std::move(out_off);
    Cm.nblk = nout;
    Cm.norms_ok = false;
    Cm.nvals = nvals;
    Cm.nelems = nelems;
    if (x.timing) BT_CUDA(cudaEventRecord(x.ev[3], st));
    tr.mark("numeric enqueued");
    x.last_had_numeric = nout > 0;
    if (sync_at_end || x.timing == 1) BT_CUDA(cudaStreamSynchronize(st));
    tr.mark("final sync");
    if (x.timing == 1) {
      float ms = 0;
      if (nout > 0) {
        BT_CUDA(cudaEventElapsedTime(&ms, x.ev[1], x.ev[2]));
        S.ms_numeric = ms;
      }
      BT_CUDA(cudaEventElapsedTime(&ms, x.ev[0], x.ev[3]));
      S.ms_total = ms;
      if (phases && nout > 0) {
        float a, b, c, d;
        BT_CUDA(cudaEventElapsedTime(&a, x.ev[0], x.ev[4]));
        BT_CUDA(cudaEventElapsedTime(&b, x.ev[4], x.ev[5]));
        BT_CUDA(cudaEventElapsedTime(&c, x.ev[5], x.ev[6]));
        BT_CUDA(cudaEventElapsedTime(&d, x.ev[6], x.ev[1]));
        fprintf(stderr, "[bt-phases] pass1+scan %.1f us | host sync gap %.1f us | fill %.1f us | "
                        "pre-numeric %.1f us | numeric %.1f us | total %.1f us\n",
                1e3 * a, 1e3 * b, 1e3 * c, 1e3 * d, 1e3 * S.ms_numeric, 1e3 * ms);
      }
    }
    S.c_blocks_out = nout;
    S.kernels = static_cast<int32_t>(x.kernels - k0);
    if (stats) *stats = S;
  }
}

extern "C" int bt_multiply(bt_ctx* ctx, const bt_mat* ah, const bt_mat* bh, bt_mat* ch,
                           double eps, bt_stats* stats) {
  return guard([&] {
    BT_REQUIRE(ctx && ah && bh && ch, BT_ERR_INVALID_ARGUMENT, "null argument");
    local_multiply(ctx->impl, ah->impl, bh->impl, ch->impl, eps, stats, nullptr, nullptr, nullptr,
                   false, ctx->impl.nranks == 1);
  });
}

extern "C" int bt_ctx_last_timing(bt_ctx* ctx, double* ms_numeric, double* ms_total) {
  return guard([&] {
    BT_REQUIRE(ctx, BT_ERR_INVALID_ARGUMENT, "null context");
    Ctx& x = ctx->impl;
    BT_REQUIRE(x.timing != 0, BT_ERR_INVALID_ARGUMENT,
               "bt_ctx_last_timing: timing is off (bt_ctx_set_timing)");
    BT_CUDA(cudaEventSynchronize(x.ev[3]));
    float ms = 0;
    if (ms_numeric) {
      *ms_numeric = 0;
      if (x.last_had_numeric) {
        BT_CUDA(cudaEventElapsedTime(&ms, x.ev[1], x.ev[2]));
        *ms_numeric = ms;
      }
    }
    if (ms_total) {
      BT_CUDA(cudaEventElapsedTime(&ms, x.ev[0], x.ev[3]));
      *ms_total = ms;
    }
  });
}
