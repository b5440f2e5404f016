/*
 * bt_oracle.c -- CPU restatement of the reference block-sparse multiply path.
 * TEST INFRASTRUCTURE ONLY (see bt_oracle.h).  Build: oracle/Makefile
 * (-O2 -ffp-contract=off, no -march: bit-compatible with the reference's
 * CMake Release build).
 */
#include "bt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ Rng */
/* std::mt19937_64 as specified by the C++ standard ([rand.eng.mers]); the
 * reference relies on its bit-exact output (random.hpp:14-16). */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x7FFFFFFFULL

void bto_rng_seed(bto_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
}

static void mt_twist(bto_rng* r) {
  for (int i = 0; i < MT_N; ++i) {
    uint64_t x = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->idx = 0;
}

uint64_t bto_rng_next(bto_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* random.hpp:24-27 */
int64_t bto_rng_uniform_int(bto_rng* r, int64_t lo, int64_t hi) {
  uint64_t span = (uint64_t)(hi - lo) + 1;
  return lo + (int64_t)(bto_rng_next(r) % span);
}

/* random.hpp:30-32 */
double bto_rng_uniform(bto_rng* r) { return (double)(bto_rng_next(r) >> 11) * 0x1.0p-53; }

/* random.hpp:34 */
int bto_rng_bernoulli(bto_rng* r, double p) { return bto_rng_uniform(r) < p; }

/* random.hpp:37-43 (Box-Muller, one value per call, no cached spare) */
double bto_rng_normal(bto_rng* r) {
  double u1 = bto_rng_uniform(r);
  while (u1 == 0.0) u1 = bto_rng_uniform(r);
  double u2 = bto_rng_uniform(r);
  const double two_pi = 6.283185307179586476925286766559;
  return sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
}

/* ------------------------------------------------------------- matrices */
void bto_mat_free(bto_mat* m) {
  free(m->rsz);
  free(m->csz);
  free(m->row_ptr);
  free(m->col);
  free(m->off);
  free(m->vals);
  memset(m, 0, sizeof(*m));
}

int bto_mat_empty(bto_mat* m, int64_t nbr, const int32_t* rsz, int64_t nbc, const int32_t* csz) {
  memset(m, 0, sizeof(*m));
  m->nbr = nbr;
  m->nbc = nbc;
  m->rsz = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nbr > 0 ? nbr : 1));
  m->csz = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nbc > 0 ? nbc : 1));
  m->row_ptr = (int64_t*)calloc((size_t)nbr + 1, sizeof(int64_t));
  if (!m->rsz || !m->csz || !m->row_ptr) return -1;
  for (int64_t t = 0; t < nbr; ++t) {
    if (rsz[t] < 1) return -2; /* Blocking: block sizes must be positive (block.hpp:77) */
    m->rsz[t] = rsz[t];
  }
  for (int64_t t = 0; t < nbc; ++t) {
    if (csz[t] < 1) return -2;
    m->csz[t] = csz[t];
  }
  return 0;
}

int bto_mat_from_blocks(bto_mat* m, int64_t nbr, const int32_t* rsz, int64_t nbc,
                        const int32_t* csz, int64_t nblk, const int64_t* bi, const int64_t* bj,
                        const double* vals) {
  int rc = bto_mat_empty(m, nbr, rsz, nbc, csz);
  if (rc) return rc;
  m->nblk = nblk;
  m->col = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nblk > 0 ? nblk : 1));
  m->off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nblk > 0 ? nblk : 1));
  int64_t nv = 0;
  for (int64_t t = 0; t < nblk; ++t) {
    if (bi[t] < 0 || bi[t] >= nbr || bj[t] < 0 || bj[t] >= nbc) return -3;
    if (t > 0 && (bi[t] < bi[t - 1] || (bi[t] == bi[t - 1] && bj[t] <= bj[t - 1]))) return -4;
    m->col[t] = bj[t];
    m->off[t] = nv;
    nv += (int64_t)rsz[bi[t]] * csz[bj[t]];
    m->row_ptr[bi[t] + 1]++;
  }
  for (int64_t r = 0; r < nbr; ++r) m->row_ptr[r + 1] += m->row_ptr[r];
  m->nvals = nv;
  m->vals = (double*)malloc(sizeof(double) * (size_t)(nv > 0 ? nv : 1));
  if (nv) memcpy(m->vals, vals, sizeof(double) * (size_t)nv);
  return 0;
}

/* oracles.hpp:74-85: for i, for j: if (!bernoulli(occ)) continue; values = normal() */
int bto_random_matrix(bto_mat* m, uint64_t seed, int64_t nbr, const int32_t* rsz, int64_t nbc,
                      const int32_t* csz, double occ, double scale_exp) {
  int rc = bto_mat_empty(m, nbr, rsz, nbc, csz);
  if (rc) return rc;
  bto_rng r;
  bto_rng_seed(&r, seed);
  int64_t cap_b = 1024, cap_v = 1 << 16;
  m->col = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap_b);
  m->off = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap_b);
  m->vals = (double*)malloc(sizeof(double) * (size_t)cap_v);
  int64_t nb = 0, nv = 0;
  for (int64_t i = 0; i < nbr; ++i) {
    for (int64_t j = 0; j < nbc; ++j) {
      if (!bto_rng_bernoulli(&r, occ)) continue;
      double scale = 1.0;
      if (scale_exp > 0) scale = pow(10.0, -scale_exp * bto_rng_uniform(&r));
      int64_t sz = (int64_t)rsz[i] * csz[j];
      if (nb == cap_b) {
        cap_b *= 2;
        m->col = (int64_t*)realloc(m->col, sizeof(int64_t) * (size_t)cap_b);
        m->off = (int64_t*)realloc(m->off, sizeof(int64_t) * (size_t)cap_b);
      }
      while (nv + sz > cap_v) {
        cap_v *= 2;
        m->vals = (double*)realloc(m->vals, sizeof(double) * (size_t)cap_v);
      }
      m->col[nb] = j;
      m->off[nb] = nv;
      for (int64_t t = 0; t < sz; ++t) {
        double v = bto_rng_normal(&r);
        m->vals[nv + t] = scale_exp > 0 ? v * scale : v;
      }
      nv += sz;
      nb++;
      m->row_ptr[i + 1]++;
    }
  }
  for (int64_t i = 0; i < nbr; ++i) m->row_ptr[i + 1] += m->row_ptr[i];
  m->nblk = nb;
  m->nvals = nv;
  return 0;
}

/* oracles.hpp:60-70 */
int64_t bto_random_blocking(uint64_t seed, int64_t total, int bmin, int bmax, int32_t* out,
                            int64_t cap) {
  bto_rng r;
  bto_rng_seed(&r, seed);
  int64_t left = total, n = 0;
  while (left > 0) {
    int s = (int)bto_rng_uniform_int(&r, bmin, bmax);
    if (s > left) s = (int)left;
    if (n < cap) out[n] = s;
    n++;
    left -= s;
  }
  return n;
}

/* ---------------------------------------------------------------- kernel */
/* block.hpp:45-60 */
void bto_block_gemm_acc(double* c, const double* a, const double* b, int m, int n, int k) {
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) {
      double acc = c[(size_t)i * n + j];
      for (int p = 0; p < k; ++p) acc += a[(size_t)i * k + p] * b[(size_t)p * n + j];
      c[(size_t)i * n + j] = acc;
    }
}

/* Block Frobenius norm (the build-defined eps filter): squares
   summed along each row first, then the row sums in row order; unfused
   (-ffp-contract=off).  The GPU (k_block_norms) adds in the same order. */
double bto_block_norm(const double* a, int m, int n) {
  double s = 0.0;
  for (int r = 0; r < m; ++r) {
    double rs = 0.0;
    for (int c = 0; c < n; ++c) rs += a[(size_t)r * n + c] * a[(size_t)r * n + c];
    s += rs;
  }
  return sqrt(s);
}

/* ------------------------------------------------------------- multiply */
typedef struct {
  int64_t j, k, ai, bi;
} prod_t;

static int cmp_prod_j(const void* x, const void* y) {
  const prod_t* p = (const prod_t*)x;
  const prod_t* q = (const prod_t*)y;
  if (p->j != q->j) return p->j < q->j ? -1 : 1;
  if (p->k != q->k) return p->k < q->k ? -1 : 1; /* (row, col, k): block.hpp:112-118 */
  return 0;
}

/* multiply_tiles_into (multiply_cannon.hpp:24-44) on whole local stores:
 * batch = {A(i,k) x B(k,j)}, ordered by (i, j, k), each item applied to
 * get_or_create(i, j) with block_gemm_acc. */
int bto_multiply(const bto_mat* a, const bto_mat* b, bto_mat* c, double eps, int64_t* nprod_out,
                 double* flops_out) {
  if (a->nbc != b->nbr || c->nbr != a->nbr || c->nbc != b->nbc) return -1;
  for (int64_t t = 0; t < a->nbc; ++t)
    if (a->csz[t] != b->rsz[t]) return -1;
  for (int64_t t = 0; t < a->nbr; ++t)
    if (a->rsz[t] != c->rsz[t]) return -1;
  for (int64_t t = 0; t < b->nbc; ++t)
    if (b->csz[t] != c->csz[t]) return -1;

  double* na = NULL;
  double* nb = NULL;
  if (eps > 0) {
    na = (double*)malloc(sizeof(double) * (size_t)(a->nblk + 1));
    nb = (double*)malloc(sizeof(double) * (size_t)(b->nblk + 1));
    for (int64_t r = 0; r < a->nbr; ++r)
      for (int64_t e = a->row_ptr[r]; e < a->row_ptr[r + 1]; ++e)
        na[e] = bto_block_norm(a->vals + a->off[e], a->rsz[r], a->csz[a->col[e]]);
    for (int64_t r = 0; r < b->nbr; ++r)
      for (int64_t e = b->row_ptr[r]; e < b->row_ptr[r + 1]; ++e)
        nb[e] = bto_block_norm(b->vals + b->off[e], b->rsz[r], b->csz[b->col[e]]);
  }

  bto_mat out;
  memset(&out, 0, sizeof(out));
  bto_mat_empty(&out, c->nbr, c->rsz, c->nbc, c->csz);
  int64_t cap_b = c->nblk + 1024, cap_v = c->nvals + 65536;
  out.col = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap_b);
  out.off = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap_b);
  out.vals = (double*)malloc(sizeof(double) * (size_t)cap_v);
  int64_t nbo = 0, nvo = 0, nprod = 0;
  double flops = 0;
  int64_t pcap = 1024;
  prod_t* prods = (prod_t*)malloc(sizeof(prod_t) * (size_t)pcap);

  for (int64_t i = 0; i < a->nbr; ++i) {
    int64_t np = 0;
    for (int64_t e = a->row_ptr[i]; e < a->row_ptr[i + 1]; ++e) {
      int64_t k = a->col[e];
      for (int64_t f = b->row_ptr[k]; f < b->row_ptr[k + 1]; ++f) {
        if (eps > 0 && na[e] * nb[f] < eps) continue;
        if (np == pcap) {
          pcap *= 2;
          prods = (prod_t*)realloc(prods, sizeof(prod_t) * (size_t)pcap);
        }
        prods[np].j = b->col[f];
        prods[np].k = k;
        prods[np].ai = e;
        prods[np].bi = f;
        np++;
      }
    }
    qsort(prods, (size_t)np, sizeof(prod_t), cmp_prod_j);
    /* merge C_in row i with product columns */
    int64_t ce = c->row_ptr[i], ce_end = c->row_ptr[i + 1];
    int64_t p = 0;
    const int m = a->rsz[i];
    while (ce < ce_end || p < np) {
      int64_t j;
      if (ce < ce_end && (p >= np || c->col[ce] <= prods[p].j))
        j = c->col[ce];
      else
        j = prods[p].j;
      const int n = c->csz[j];
      int64_t sz = (int64_t)m * n;
      if (nbo == cap_b) {
        cap_b *= 2;
        out.col = (int64_t*)realloc(out.col, sizeof(int64_t) * (size_t)cap_b);
        out.off = (int64_t*)realloc(out.off, sizeof(int64_t) * (size_t)cap_b);
      }
      while (nvo + sz > cap_v) {
        cap_v *= 2;
        out.vals = (double*)realloc(out.vals, sizeof(double) * (size_t)cap_v);
      }
      double* dst = out.vals + nvo;
      if (ce < ce_end && c->col[ce] == j) {
        memcpy(dst, c->vals + c->off[ce], sizeof(double) * (size_t)sz);
        ce++;
      } else {
        memset(dst, 0, sizeof(double) * (size_t)sz); /* get_or_create: zero block */
      }
      while (p < np && prods[p].j == j) {
        const int k = a->csz[prods[p].k];
        bto_block_gemm_acc(dst, a->vals + a->off[prods[p].ai], b->vals + b->off[prods[p].bi], m, n,
                           k);
        nprod++;
        flops += 2.0 * m * n * k;
        p++;
      }
      out.col[nbo] = j;
      out.off[nbo] = nvo;
      nbo++;
      nvo += sz;
      out.row_ptr[i + 1]++;
    }
  }
  for (int64_t i = 0; i < out.nbr; ++i) out.row_ptr[i + 1] += out.row_ptr[i];
  out.nblk = nbo;
  out.nvals = nvo;
  free(prods);
  free(na);
  free(nb);
  bto_mat_free(c);
  *c = out;
  if (nprod_out) *nprod_out = nprod;
  if (flops_out) *flops_out = flops;
  return 0;
}

int bto_filter(bto_mat* c, double eps) {
  int64_t nb = 0, nv = 0;
  for (int64_t i = 0; i < c->nbr; ++i) {
    int64_t start = nb;
    for (int64_t e = c->row_ptr[i]; e < c->row_ptr[i + 1]; ++e) {
      int64_t sz = (int64_t)c->rsz[i] * c->csz[c->col[e]];
      double nrm = bto_block_norm(c->vals + c->off[e], c->rsz[i], c->csz[c->col[e]]);
      if (nrm < eps) continue;
      memmove(c->vals + nv, c->vals + c->off[e], sizeof(double) * (size_t)sz);
      c->col[nb] = c->col[e];
      c->off[nb] = nv;
      nb++;
      nv += sz;
    }
    c->row_ptr[i] = start;
  }
  c->row_ptr[c->nbr] = nb;
  /* row_ptr[i] was overwritten with the new start of row i; restore CSR form */
  c->nblk = nb;
  c->nvals = nv;
  return 0;
}

/* oracles.hpp:27-37 */
void bto_dense_gemm_acc(double* c, const double* a, const double* b, int64_t m, int64_t n,
                        int64_t k) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = c[i * n + j];
      for (int64_t p = 0; p < k; ++p) acc += a[i * k + p] * b[p * n + j];
      c[i * n + j] = acc;
    }
}

/* matrix.hpp:458-470 */
int bto_to_dense(const bto_mat* m, double* out) {
  int64_t rows = 0, cols = 0;
  int64_t* roff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m->nbr + 1));
  int64_t* coff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m->nbc + 1));
  roff[0] = 0;
  for (int64_t t = 0; t < m->nbr; ++t) roff[t + 1] = roff[t] + m->rsz[t];
  coff[0] = 0;
  for (int64_t t = 0; t < m->nbc; ++t) coff[t + 1] = coff[t] + m->csz[t];
  rows = roff[m->nbr];
  cols = coff[m->nbc];
  memset(out, 0, sizeof(double) * (size_t)(rows * cols));
  for (int64_t i = 0; i < m->nbr; ++i)
    for (int64_t e = m->row_ptr[i]; e < m->row_ptr[i + 1]; ++e) {
      int64_t j = m->col[e];
      const double* blk = m->vals + m->off[e];
      for (int r = 0; r < m->rsz[i]; ++r)
        for (int q = 0; q < m->csz[j]; ++q)
          out[(roff[i] + r) * cols + coff[j] + q] = blk[(int64_t)r * m->csz[j] + q];
    }
  free(roff);
  free(coff);
  return 0;
}

/* oracles.hpp:49-57 */
double bto_frobenius_rel_error(const double* a, const double* b, int64_t n) {
  double diff = 0.0, ref = 0.0;
  for (int64_t t = 0; t < n; ++t) {
    diff += (a[t] - b[t]) * (a[t] - b[t]);
    ref += b[t] * b[t];
  }
  if (ref == 0.0) return sqrt(diff);
  return sqrt(diff / ref);
}

/* later-listed dimensions vary fastest */
int64_t bto_mixed_radix(const int64_t* coords, const int64_t* extents, int n) {
  int64_t idx = 0;
  for (int d = 0; d < n; ++d) idx = idx * extents[d] + coords[d];
  return idx;
}

void bto_mixed_radix_inv(int64_t idx, const int64_t* extents, int n, int64_t* coords) {
  for (int d = n - 1; d >= 0; --d) {
    coords[d] = idx % extents[d];
    idx /= extents[d];
  }
}
