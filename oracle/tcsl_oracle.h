/* CPU oracle for the Tiled-CSL hot path — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference lab's codec and LSCD engine
 * (/root/reference/proj, see tcsl_oracle.c for per-function file:line
 * citations). Only tests/, __graft_entry__.smoke() and bench.py's CPU
 * baseline leg may load this library, and only as the checker. The product
 * path (paper_2309_10285_b200/) never links or calls it.
 *
 * Pinning: tests/test_oracle.py checks this port against the reference's own
 * golden FNV-1a hashes (proj/tests/acceptance.cpp:60-64), its unit-test KATs
 * (proj/tests/test_codec.cpp, test_engine.cpp, test_gemm.cpp) and, when
 * oracle/_ref/libtcsl_ref.so was built, against the reference itself.
 *
 * Status codes: 0 = ok, otherwise (tcsl::Errc ordinal + 1), matching
 * proj/include/tcsl/errors.hpp:10-22.
 */
#ifndef TCSL_ORACLE_H
#define TCSL_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_BAD_MAGIC = 1,
  ORC_BAD_VERSION = 2,
  ORC_BAD_HEADER = 3,
  ORC_BAD_DTYPE = 4,
  ORC_TRUNCATED = 5,
  ORC_TRAILING_DATA = 6,
  ORC_INCONSISTENT_OFFSETS = 7,
  ORC_LOCATION_OUT_OF_RANGE = 8,
  ORC_DIMENSION_MISMATCH = 9,
  ORC_INVALID_ARGUMENT = 10,
  ORC_IO_FAILURE = 11,
  ORC_NO_MEMORY = 100
};

/* Tiled-CSL matrix owned by the oracle (free with orc_tcsl_free). */
typedef struct orc_tcsl {
  uint32_t m, k;
  int32_t m_tb, k_tb;
  int32_t reordered;
  uint32_t num_tiles;
  uint32_t *offsets;  /* num_tiles + 1 */
  uint32_t *entries;  /* n_entries */
  uint64_t n_entries;
} orc_tcsl;

/* binary16 <-> binary32 */
float orc_f32_from_f16(uint16_t b);
uint16_t orc_f16_from_f32(float v);

/* std::mt19937_64 */
typedef struct orc_mt64 {
  uint64_t s[312];
  int i;
} orc_mt64;
void orc_mt64_seed(orc_mt64 *g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64 *g);

int orc_gen_random_sparse(int rows, int cols, double beta, uint64_t seed, uint16_t *out);
int orc_tile_validate(int m_tb, int k_tb, int threads);
/* prune_magnitude: floor(beta*n) smallest |v| -> +0 (ties: larger index first). */
int orc_prune_magnitude(const uint16_t *a, int64_t n, double beta, uint16_t *out);

int orc_encode(const uint16_t *a, int rows, int cols, int m_tb, int k_tb, int reorder, orc_tcsl **out);
void orc_tcsl_free(orc_tcsl *t);
/* Wrap caller-owned arrays into a borrowed view (no copy, do not free). */
orc_tcsl orc_tcsl_view(uint32_t m, uint32_t k, int m_tb, int k_tb, int reordered,
                       uint32_t *offsets, uint32_t *entries, uint64_t n_entries);

int orc_decode(const orc_tcsl *t, uint16_t *out /* m*k */);
int orc_extract_tile(const orc_tcsl *t, uint32_t tile, uint16_t *buf /* m_tb*k_tb */);
int orc_reg_pressure(const orc_tcsl *t, int threads_per_block, int *out);

/* Y[m x n] = spmm(t, B[k x n]); bit-exact with tcsl::spmm. nthreads > 1 splits
 * row blocks across pthreads (row blocks are independent, so the bits do not
 * change). */
int orc_spmm(const orc_tcsl *t, const uint16_t *b, int n, float *y, int nthreads);
/* Y = dense_gemm_ref(A, B, cfg) */
int orc_dense_gemm(const uint16_t *a, int m, int k, const uint16_t *b, int n, int m_tb, int k_tb,
                   float *y);

/* TCSL container: returns malloc'ed buffer in *buf (free with orc_free). */
int orc_serialize(const orc_tcsl *t, uint8_t **buf, size_t *size);
int orc_deserialize(const uint8_t *data, size_t size, orc_tcsl **out);
int orc_check_offsets(const orc_tcsl *t);
uint64_t orc_fnv1a(const uint8_t *data, size_t size);
void orc_free(void *p);

#ifdef __cplusplus
}
#endif
#endif
