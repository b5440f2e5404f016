/*
 * bt_oracle.h -- CPU restatement of the reference block-sparse multiply path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it, and only as the checker.  The product path (libbtcuda.so) never
 * links or calls it.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj/).  Compiled with -O2 -ffp-contract=off so block_gemm_acc
 * reproduces the reference's unfused mul+add bits (CMake Release, no -march;
 * SURVEY.md 8c).
 *
 * Parity pinning: the restatement is checked against (1) the reference's own
 * known-answer tests (tests/test_blocks.cpp:33-76) and (2) the compiled
 * reference itself (oracle/_ref/libbtref.so built from /root/reference by
 * oracle/Makefile) on seeded random instances -- see tests/test_oracle.py.
 * The eps filter and the tensor index remap have no reference code
 * (SPEC.md:249): those two parts are "parity unpinned" and
 * follow the written definitions in DESIGN.md section 3.
 */
#ifndef BT_ORACLE_H
#define BT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- Rng: random.hpp:17-47 (mt19937_64 + explicit transforms) ---- */
typedef struct {
  uint64_t mt[312];
  int idx;
} bto_rng;

void bto_rng_seed(bto_rng* r, uint64_t seed);
uint64_t bto_rng_next(bto_rng* r);
int64_t bto_rng_uniform_int(bto_rng* r, int64_t lo, int64_t hi);
double bto_rng_uniform(bto_rng* r);
int bto_rng_bernoulli(bto_rng* r, double p);
double bto_rng_normal(bto_rng* r);

/* ---- block-CSR matrix in canonical (row, col) order ---- */
typedef struct {
  int64_t nbr, nbc;
  int32_t* rsz;     /* [nbr] block row sizes  (block.hpp:70-97 Blocking) */
  int32_t* csz;     /* [nbc] block col sizes */
  int64_t nblk;
  int64_t* row_ptr; /* [nbr+1] */
  int64_t* col;     /* [nblk] */
  int64_t* off;     /* [nblk] element offset of each block, compact row-major */
  double* vals;     /* [nvals] */
  int64_t nvals;
} bto_mat;

void bto_mat_free(bto_mat* m);
/* empty matrix with the given blockings */
int bto_mat_empty(bto_mat* m, int64_t nbr, const int32_t* rsz, int64_t nbc, const int32_t* csz);
/* from (i,j,values) triples in canonical order; values concatenated compact */
int bto_mat_from_blocks(bto_mat* m, int64_t nbr, const int32_t* rsz, int64_t nbc,
                        const int32_t* csz, int64_t nblk, const int64_t* bi, const int64_t* bj,
                        const double* vals);

/* random_matrix: tests/support/oracles.hpp:74-85.  Blocks present with
 * probability occ in (i,j) row-major order; values Rng::normal row-major.
 * If scale_exp > 0, right after each presence draw one extra uniform u is drawn
 * and every value of the block is multiplied by 10^(-scale_exp*u)
 * (BASELINE config 2's per-block norm spread; scale_exp == 0 is exactly the
 * reference semantics). */
int bto_random_matrix(bto_mat* m, uint64_t seed, int64_t nbr, const int32_t* rsz, int64_t nbc,
                      const int32_t* csz, double occ, double scale_exp);

/* random_blocking: oracles.hpp:60-70 */
int64_t bto_random_blocking(uint64_t seed, int64_t total, int bmin, int bmax, int32_t* out,
                            int64_t cap);

/* block_gemm_acc: block.hpp:45-60.  c(m x n) += a(m x k) * b(k x n), row-major,
 * k innermost, unfused mul+add. */
void bto_block_gemm_acc(double* c, const double* a, const double* b, int m, int n, int k);

/* Frobenius norm of a block: sequential sum of squares (no FMA), sqrt. */
double bto_block_norm(const double* a, int m, int n);

/* Local multiply C += A*B with reference semantics: multiply_tiles_into
 * (multiply_cannon.hpp:24-44) + order_batches (block.hpp:112-118) +
 * get_or_create (matrix.hpp:191-196).  C_out pattern = C_in U {(i,j): some
 * product survives}.  eps > 0 applies the build-defined product filter:
 * product (i,k,j) executes iff ||A_ik||_F * ||B_kj||_F >= eps.
 * c is replaced by the result.  Reports executed products and useful flops. */
int bto_multiply(const bto_mat* a, const bto_mat* b, bto_mat* c, double eps, int64_t* nprod,
                 double* flops);

/* Post-filter: drop C blocks with ||C_ij||_F < eps. */
int bto_filter(bto_mat* c, double eps);

/* dense_gemm_acc: oracles.hpp:27-37 */
void bto_dense_gemm_acc(double* c, const double* a, const double* b, int64_t m, int64_t n,
                        int64_t k);
/* to_dense: matrix.hpp:458-470 */
int bto_to_dense(const bto_mat* m, double* out);
/* frobenius_rel_error: oracles.hpp:49-57 */
double bto_frobenius_rel_error(const double* a, const double* b, int64_t n);

/* Mixed-radix tensor<->matrix block index (within a
 * dimension group later dimensions vary fastest). */
int64_t bto_mixed_radix(const int64_t* coords, const int64_t* extents, int n);
void bto_mixed_radix_inv(int64_t idx, const int64_t* extents, int n, int64_t* coords);

#ifdef __cplusplus
}
#endif
#endif
