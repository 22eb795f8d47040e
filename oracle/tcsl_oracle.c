/* CPU oracle for the Tiled-CSL hot path — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference lab's algorithms; every function cites
 * the reference file:line it restates (paths relative to /root/reference/proj).
 * Build with -ffp-contract=off (proj/CMakeLists.txt:12-13): the spmm/gemm
 * bit-exactness contract needs every multiply and add to round separately.
 * See tcsl_oracle.h for who may use this file.
 */
#include "tcsl_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* binary16 <-> binary32: src/half.cpp:10-66                                 */

uint16_t orc_f16_from_f32(float v) { /* src/half.cpp:10-40 */
  uint32_t f;
  memcpy(&f, &v, 4);
  const uint32_t sign = (f >> 16) & 0x8000u;
  const uint32_t mag = f & 0x7FFFFFFFu;
  if (mag > 0x7F800000u) return 0x7E00u;
  if (mag >= 0x47800000u) return (uint16_t)(sign | 0x7C00u);
  if (mag >= 0x38800000u) {
    uint32_t h = (mag - 0x38000000u) >> 13;
    const uint32_t rem = (mag - 0x38000000u) & 0x1FFFu;
    h += (rem > 0x1000u) || (rem == 0x1000u && (h & 1u));
    return (uint16_t)(sign | h);
  }
  const int e = (int)(mag >> 23);
  const int shift = 126 - e;
  if (mag == 0 || shift > 24) return (uint16_t)sign;
  const uint32_t sig = 0x800000u | (mag & 0x7FFFFFu);
  uint32_t q = sig >> shift;
  const uint32_t rem = sig & ((1u << shift) - 1u);
  const uint32_t halfway = 1u << (shift - 1);
  q += (rem > halfway) || (rem == halfway && (q & 1u));
  return (uint16_t)(sign | q);
}

float orc_f32_from_f16(uint16_t b) { /* src/half.cpp:42-66 */
  const uint32_t sign = (uint32_t)(b & 0x8000u) << 16;
  const uint32_t e = (b >> 10) & 0x1Fu;
  uint32_t man = b & 0x3FFu;
  uint32_t out;
  if (e == 0) {
    if (man == 0) {
      out = sign;
    } else {
      int e32 = 113;
      while (!(man & 0x400u)) {
        man <<= 1;
        --e32;
      }
      out = sign | ((uint32_t)e32 << 23) | ((man & 0x3FFu) << 13);
    }
  } else if (e == 0x1Fu) {
    out = sign | 0x7F800000u | (man << 13);
  } else {
    out = sign | ((e + 112u) << 23) | (man << 13);
  }
  float f;
  memcpy(&f, &out, 4);
  return f;
}

static int f16_is_zero(uint16_t b) { return (b & 0x7FFFu) == 0; } /* include/tcsl/half.hpp:20 */
static uint16_t f16_norm_zero(uint16_t b) { return f16_is_zero(b) ? 0 : b; } /* half.hpp:27 */

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 (C++ [rand.eng.mers], parameters of [rand.predef])       */

void orc_mt64_seed(orc_mt64 *g, uint64_t seed) {
  g->s[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->s[i] = 6364136223846793005ull * (g->s[i - 1] ^ (g->s[i - 1] >> 62)) + (uint64_t)i;
  g->i = 312;
}

uint64_t orc_mt64_next(orc_mt64 *g) {
  const uint64_t upper = 0xFFFFFFFF80000000ull, lower = 0x7FFFFFFFull;
  if (g->i >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (g->s[i] & upper) | (g->s[(i + 1) % 312] & lower);
      uint64_t v = g->s[(i + 156) % 312] ^ (y >> 1);
      if (y & 1u) v ^= 0xB5026F5AA96619E9ull;
      g->s[i] = v;
    }
    g->i = 0;
  }
  uint64_t x = g->s[g->i++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}

/* src/matrix.cpp:35-67 — selection sampling of exactly round(beta*n) zeros. */
int orc_gen_random_sparse(int rows, int cols, double beta, uint64_t seed, uint16_t *out) {
  if (rows <= 0 || cols <= 0) return ORC_INVALID_ARGUMENT;
  if (!(beta >= 0.0 && beta <= 1.0)) return ORC_INVALID_ARGUMENT;
  const int64_t n = (int64_t)rows * cols;
  int64_t needed = llround(beta * (double)n);
  if (needed < 0) needed = 0;
  if (needed > n) needed = n;
  orc_mt64 *g = (orc_mt64 *)malloc(sizeof(orc_mt64));
  if (!g) return ORC_NO_MEMORY;
  orc_mt64_seed(g, seed);
  int64_t remaining = n;
  for (int64_t i = 0; i < n; ++i, --remaining) {
    if (orc_mt64_next(g) % (uint64_t)remaining < (uint64_t)needed) {
      out[i] = 0x0000;
      --needed;
    } else {
      const uint64_t r = orc_mt64_next(g);
      const uint16_t man = (uint16_t)(r & 0x3FFu);
      const uint16_t expf = (uint16_t)(13 + (r >> 10) % 5);
      const uint16_t sign = (uint16_t)(((r >> 63) & 1u) << 15);
      out[i] = (uint16_t)(sign | (expf << 10) | man);
    }
  }
  free(g);
  return ORC_OK;
}

/* src/matrix.cpp:69-100 — the ordering is a strict total order (|v| ascending,
   NaN as +inf, then index descending), so a full sort selects exactly the same
   set as the reference's nth_element. */
typedef struct {
  float r;
  int64_t i;
} prune_key;

static int prune_cmp(const void *pa, const void *pb) {
  const prune_key *a = (const prune_key *)pa, *b = (const prune_key *)pb;
  if (a->r != b->r) return a->r < b->r ? -1 : 1;
  return a->i > b->i ? -1 : (a->i < b->i ? 1 : 0);
}

int orc_prune_magnitude(const uint16_t *a, int64_t n, double beta, uint16_t *out) {
  if (!(beta >= 0.0 && beta <= 1.0)) return ORC_INVALID_ARGUMENT;
  memcpy(out, a, (size_t)n * 2);
  int64_t cut = (int64_t)floor(beta * (double)n);
  if (cut < 0) cut = 0;
  if (cut > n) cut = n;
  if (cut == 0 || n == 0) return ORC_OK;
  prune_key *keys = (prune_key *)malloc((size_t)n * sizeof(prune_key));
  if (!keys) return ORC_NO_MEMORY;
  for (int64_t i = 0; i < n; ++i) {
    const float m = fabsf(orc_f32_from_f16(a[i]));
    keys[i].r = isnan(m) ? HUGE_VALF : m;
    keys[i].i = i;
  }
  qsort(keys, (size_t)n, sizeof(prune_key), prune_cmp);
  for (int64_t i = 0; i < cut; ++i) out[keys[i].i] = 0;
  free(keys);
  return ORC_OK;
}

/* src/matrix.cpp:11-18 */
int orc_tile_validate(int m_tb, int k_tb, int threads) {
  if (m_tb <= 0 || k_tb <= 0) return ORC_INVALID_ARGUMENT;
  if (m_tb % 8 != 0 || k_tb % 8 != 0) return ORC_INVALID_ARGUMENT;
  if ((int64_t)m_tb * k_tb > 65536) return ORC_INVALID_ARGUMENT;
  if (threads <= 0) return ORC_INVALID_ARGUMENT;
  return ORC_OK;
}

static int div_up(int64_t a, int64_t b) { return (int)((a + b - 1) / b); } /* matrix.hpp:34 */

static uint32_t tcsl_tiles(const orc_tcsl *t) {
  return (uint32_t)div_up(t->m, t->m_tb) * (uint32_t)div_up(t->k, t->k_tb);
}

/* ------------------------------------------------------------------------ */
/* encode: src/tcsl_format.cpp:36-124                                        */

typedef struct {
  uint32_t *v;
  size_t n, cap;
} u32vec;

static int vpush(u32vec *v, uint32_t x) {
  if (v->n == v->cap) {
    size_t nc = v->cap ? v->cap * 2 : 1024;
    uint32_t *p = (uint32_t *)realloc(v->v, nc * sizeof(uint32_t));
    if (!p) return ORC_NO_MEMORY;
    v->v = p;
    v->cap = nc;
  }
  v->v[v->n++] = x;
  return ORC_OK;
}

static int bank_id(int x, int y) { return (x % 8) * 4 + (y % 8) / 2; } /* tcsl_format.hpp:18 */

int orc_encode(const uint16_t *a, int rows, int cols, int m_tb, int k_tb, int reorder, orc_tcsl **out) {
  int st = orc_tile_validate(m_tb, k_tb, 1);
  if (st) return st;
  if (rows <= 0 || cols <= 0) return ORC_INVALID_ARGUMENT;
  const int tm = div_up(rows, m_tb), tk = div_up(cols, k_tb);
  const uint32_t nt = (uint32_t)tm * (uint32_t)tk;
  orc_tcsl *t = (orc_tcsl *)calloc(1, sizeof(orc_tcsl));
  if (!t) return ORC_NO_MEMORY;
  t->m = (uint32_t)rows;
  t->k = (uint32_t)cols;
  t->m_tb = m_tb;
  t->k_tb = k_tb;
  t->reordered = reorder ? 1 : 0;
  t->num_tiles = nt;
  t->offsets = (uint32_t *)malloc(((size_t)nt + 1) * sizeof(uint32_t));
  /* 32 FIFO buckets, each at most m_tb*k_tb/32 long per tile. */
  const int bcap = m_tb * k_tb / 32 + 1;
  uint32_t *buckets = (uint32_t *)malloc((size_t)32 * bcap * sizeof(uint32_t));
  int bsize[32], head[32];
  u32vec ent = {0, 0, 0};
  if (!t->offsets || !buckets) {
    free(buckets);
    orc_tcsl_free(t);
    return ORC_NO_MEMORY;
  }
  t->offsets[0] = 0;
  uint32_t tile = 0;
  for (int ti = 0; ti < tm; ++ti) {
    for (int tj = 0; tj < tk; ++tj, ++tile) {
      const int r0 = ti * m_tb, c0 = tj * k_tb;
      const int x_end = (m_tb < rows - r0) ? m_tb : rows - r0;
      const int y_end = (k_tb < cols - c0) ? k_tb : cols - c0;
      memset(bsize, 0, sizeof(bsize));
      size_t nnz = 0;
      /* gather in row-major scan order, dropping +-0 (tcsl_format.cpp:67-78) */
      for (int x = 0; x < x_end; ++x) {
        const uint16_t *row = a + (int64_t)(r0 + x) * cols + c0;
        for (int y = 0; y < y_end; ++y) {
          const uint16_t v = row[y];
          if (f16_is_zero(v)) continue;
          const uint32_t e = ((uint32_t)v << 16) | (uint32_t)(uint16_t)(x * k_tb + y);
          if (reorder) {
            const int b = bank_id(x, y);
            buckets[(size_t)b * bcap + bsize[b]++] = e;
          } else {
            st = vpush(&ent, e);
            if (st) goto fail;
          }
          ++nnz;
        }
      }
      if (reorder) {
        /* greedy: fullest bucket, smallest id on ties, FIFO (tcsl_format.cpp:81-97) */
        memset(head, 0, sizeof(head));
        for (size_t left = nnz; left > 0; --left) {
          int best = 0;
          int best_left = bsize[0] - head[0];
          for (int bk = 1; bk < 32; ++bk) {
            const int l = bsize[bk] - head[bk];
            if (l > best_left) {
              best = bk;
              best_left = l;
            }
          }
          st = vpush(&ent, buckets[(size_t)best * bcap + head[best]++]);
          if (st) goto fail;
        }
      }
      /* pad to 32 with +0.0 at the first zero positions of the full tile,
         fringe included (tcsl_format.cpp:103-119) */
      const size_t rem = nnz % 32;
      if (rem != 0) {
        size_t need = 32 - rem;
        for (int x = 0; x < m_tb && need > 0; ++x) {
          for (int y = 0; y < k_tb && need > 0; ++y) {
            const int inside = x < x_end && y < y_end;
            if (inside && !f16_is_zero(a[(int64_t)(r0 + x) * cols + c0 + y])) continue;
            st = vpush(&ent, (uint32_t)(uint16_t)(x * k_tb + y));
            if (st) goto fail;
            --need;
          }
        }
      }
      t->offsets[tile + 1] = (uint32_t)ent.n; /* u32 wrap like tcsl_format.cpp:120 */
    }
  }
  free(buckets);
  t->entries = ent.v ? ent.v : (uint32_t *)malloc(4);
  t->n_entries = ent.n;
  *out = t;
  return ORC_OK;
fail:
  free(buckets);
  free(ent.v);
  orc_tcsl_free(t);
  return st;
}

void orc_tcsl_free(orc_tcsl *t) {
  if (!t) return;
  free(t->offsets);
  free(t->entries);
  free(t);
}

orc_tcsl orc_tcsl_view(uint32_t m, uint32_t k, int m_tb, int k_tb, int reordered, uint32_t *offsets,
                       uint32_t *entries, uint64_t n_entries) {
  orc_tcsl t;
  t.m = m;
  t.k = k;
  t.m_tb = m_tb;
  t.k_tb = k_tb;
  t.reordered = reordered;
  t.offsets = offsets;
  t.entries = entries;
  t.n_entries = n_entries;
  t.num_tiles = tcsl_tiles(&t);
  return t;
}

/* src/tcsl_format.cpp:19-32 */
int orc_check_offsets(const orc_tcsl *t) {
  const uint32_t nt = tcsl_tiles(t);
  if (t->offsets[0] != 0) return ORC_INCONSISTENT_OFFSETS;
  for (uint32_t i = 0; i < nt; ++i) {
    if (t->offsets[i + 1] < t->offsets[i]) return ORC_INCONSISTENT_OFFSETS;
    if ((t->offsets[i + 1] - t->offsets[i]) % 32 != 0) return ORC_INCONSISTENT_OFFSETS;
  }
  if (t->offsets[nt] != t->n_entries) return ORC_INCONSISTENT_OFFSETS;
  return ORC_OK;
}

/* src/tcsl_format.cpp:126-155 */
int orc_decode(const orc_tcsl *t, uint16_t *out) {
  int st = orc_tile_validate(t->m_tb, t->k_tb, 1);
  if (st) return st;
  if (t->m == 0 || t->k == 0) return ORC_BAD_HEADER;
  st = orc_check_offsets(t);
  if (st) return st;
  const int tk = div_up(t->k, t->k_tb);
  const int tile_elems = t->m_tb * t->k_tb;
  memset(out, 0, (size_t)t->m * t->k * 2);
  const uint32_t nt = tcsl_tiles(t);
  for (uint32_t tile = 0; tile < nt; ++tile) {
    const int r0 = (int)tile / tk * t->m_tb;
    const int c0 = (int)tile % tk * t->k_tb;
    for (uint32_t e = t->offsets[tile]; e < t->offsets[tile + 1]; ++e) {
      const uint32_t entry = t->entries[e];
      const int loc = (int)(entry & 0xFFFFu);
      if (loc >= tile_elems) return ORC_LOCATION_OUT_OF_RANGE;
      const int r = r0 + loc / t->k_tb, c = c0 + loc % t->k_tb;
      const uint16_t v = f16_norm_zero((uint16_t)(entry >> 16));
      if (r >= (int)t->m || c >= (int)t->k) {
        if (!f16_is_zero(v)) return ORC_LOCATION_OUT_OF_RANGE;
        continue;
      }
      out[(size_t)r * t->k + c] = v;
    }
  }
  return ORC_OK;
}

/* src/engine.cpp:8-25 */
int orc_extract_tile(const orc_tcsl *t, uint32_t tile, uint16_t *buf) {
  int st = orc_tile_validate(t->m_tb, t->k_tb, 1);
  if (st) return st;
  if (tile >= tcsl_tiles(t)) return ORC_INVALID_ARGUMENT;
  if (t->offsets[tile + 1] < t->offsets[tile] || t->offsets[tile + 1] > t->n_entries)
    return ORC_INCONSISTENT_OFFSETS;
  const int tile_elems = t->m_tb * t->k_tb;
  memset(buf, 0, (size_t)tile_elems * 2);
  for (uint32_t e = t->offsets[tile]; e < t->offsets[tile + 1]; ++e) {
    const uint32_t entry = t->entries[e];
    const int loc = (int)(entry & 0xFFFFu);
    if (loc >= tile_elems) return ORC_LOCATION_OUT_OF_RANGE;
    buf[loc] = f16_norm_zero((uint16_t)(entry >> 16));
  }
  return ORC_OK;
}

/* src/engine.cpp:80-91 */
int orc_reg_pressure(const orc_tcsl *t, int threads_per_block, int *out) {
  int st = orc_tile_validate(t->m_tb, t->k_tb, threads_per_block);
  if (st) return st;
  int worst = 0;
  for (uint32_t tile = 0; tile < tcsl_tiles(t); ++tile) {
    const uint32_t count = t->offsets[tile + 1] - t->offsets[tile];
    const int need = div_up(count, threads_per_block);
    if (need > worst) worst = need;
  }
  *out = worst;
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* spmm: src/engine.cpp:27-78                                                */

typedef struct {
  const orc_tcsl *t;
  const float *bf; /* widened, K-padded B */
  int n;
  float *y;
  int rb0, rb1;
  int status;
} spmm_job;

static void *spmm_rows(void *arg) {
  spmm_job *j = (spmm_job *)arg;
  const orc_tcsl *t = j->t;
  const int m_tb = t->m_tb, k_tb = t->k_tb, n = j->n;
  const int tiles_k = div_up(t->k, k_tb);
  uint16_t *tile = (uint16_t *)malloc((size_t)m_tb * k_tb * 2);
  float *at = (float *)malloc((size_t)m_tb * k_tb * 4);
  float *acc = (float *)malloc((size_t)m_tb * n * 4);
  if (!tile || !at || !acc) {
    j->status = ORC_NO_MEMORY;
    goto done;
  }
  for (int rb = j->rb0; rb < j->rb1; ++rb) {
    memset(acc, 0, (size_t)m_tb * n * 4);
    for (int tj = 0; tj < tiles_k; ++tj) {
      int st = orc_extract_tile(t, (uint32_t)rb * tiles_k + tj, tile);
      if (st) {
        j->status = st;
        goto done;
      }
      for (int i = 0; i < m_tb * k_tb; ++i) at[i] = orc_f32_from_f16(tile[i]);
      /* per output (x, j): kk ascending inside the tile, tiles ascending */
      for (int x = 0; x < m_tb; ++x) {
        float *arow = acc + (size_t)x * n;
        const float *trow = at + (size_t)x * k_tb;
        for (int kk = 0; kk < k_tb; ++kk) {
          const float av = trow[kk];
          const float *brow = j->bf + ((size_t)tj * k_tb + kk) * n;
          for (int c = 0; c < n; ++c) arow[c] += av * brow[c];
        }
      }
    }
    const int x_end = (m_tb < (int)t->m - rb * m_tb) ? m_tb : (int)t->m - rb * m_tb;
    memcpy(j->y + (size_t)rb * m_tb * n, acc, (size_t)x_end * n * 4);
  }
done:
  free(tile);
  free(at);
  free(acc);
  return NULL;
}

int orc_spmm(const orc_tcsl *t, const uint16_t *b, int n, float *y, int nthreads) {
  int st = orc_tile_validate(t->m_tb, t->k_tb, 1);
  if (st) return st;
  if (n <= 0) return ORC_INVALID_ARGUMENT;
  const int tiles_m = div_up(t->m, t->m_tb), tiles_k = div_up(t->k, t->k_tb);
  const size_t k_pad = (size_t)tiles_k * t->k_tb;
  float *bf = (float *)calloc(k_pad * n, 4);
  if (!bf) return ORC_NO_MEMORY;
  for (size_t kk = 0; kk < t->k; ++kk)
    for (int c = 0; c < n; ++c) bf[kk * n + c] = orc_f32_from_f16(b[kk * n + c]);
  if (nthreads < 1) nthreads = 1;
  if (nthreads > tiles_m) nthreads = tiles_m;
  spmm_job *jobs = (spmm_job *)calloc((size_t)nthreads, sizeof(spmm_job));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int i = 0; i < nthreads; ++i) {
    jobs[i].t = t;
    jobs[i].bf = bf;
    jobs[i].n = n;
    jobs[i].y = y;
    jobs[i].rb0 = (int)((int64_t)tiles_m * i / nthreads);
    jobs[i].rb1 = (int)((int64_t)tiles_m * (i + 1) / nthreads);
  }
  if (nthreads == 1) {
    spmm_rows(&jobs[0]);
  } else {
    for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, spmm_rows, &jobs[i]);
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  }
  st = ORC_OK;
  for (int i = 0; i < nthreads; ++i)
    if (jobs[i].status && !st) st = jobs[i].status;
  free(jobs);
  free(th);
  free(bf);
  return st;
}

/* src/gemm.cpp:7-44 */
int orc_dense_gemm(const uint16_t *a, int m, int k, const uint16_t *b, int n, int m_tb, int k_tb,
                   float *y) {
  int st = orc_tile_validate(m_tb, k_tb, 1);
  if (st) return st;
  if (m <= 0 || k <= 0 || n <= 0) return ORC_INVALID_ARGUMENT;
  const int k_pad = div_up(k, k_tb) * k_tb;
  float *bf = (float *)calloc((size_t)k_pad * n, 4);
  float *af = (float *)calloc((size_t)k_pad, 4);
  float *acc = (float *)malloc((size_t)n * 4);
  if (!bf || !af || !acc) {
    free(bf);
    free(af);
    free(acc);
    return ORC_NO_MEMORY;
  }
  for (int kk = 0; kk < k; ++kk)
    for (int c = 0; c < n; ++c) bf[(size_t)kk * n + c] = orc_f32_from_f16(b[(size_t)kk * n + c]);
  for (int i = 0; i < m; ++i) {
    for (int kk = 0; kk < k; ++kk) af[kk] = orc_f32_from_f16(a[(size_t)i * k + kk]);
    for (int c = 0; c < n; ++c) acc[c] = 0.0f;
    for (int kk = 0; kk < k_pad; ++kk) {
      const float av = af[kk];
      const float *brow = bf + (size_t)kk * n;
      for (int c = 0; c < n; ++c) acc[c] += av * brow[c];
    }
    memcpy(y + (size_t)i * n, acc, (size_t)n * 4);
  }
  free(bf);
  free(af);
  free(acc);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* TCSL container: src/tcsl_format.cpp:157-222, include/tcsl/tcsl_format.hpp:68-71 */

static void put32(uint8_t *p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static uint32_t get32(const uint8_t *p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

int orc_serialize(const orc_tcsl *t, uint8_t **buf, size_t *size) {
  int st = orc_tile_validate(t->m_tb, t->k_tb, 1);
  if (st) return st;
  if (t->m == 0 || t->k == 0) return ORC_BAD_HEADER;
  st = orc_check_offsets(t);
  if (st) return st;
  const uint32_t nt = tcsl_tiles(t);
  const size_t sz = 28 + 4 * ((size_t)nt + 1) + 4 * (size_t)t->n_entries;
  uint8_t *b = (uint8_t *)malloc(sz);
  if (!b) return ORC_NO_MEMORY;
  memcpy(b, "TCSL", 4);
  b[4] = 1;
  b[5] = 0;
  b[6] = t->reordered ? 1 : 0;
  b[7] = 0;
  put32(b + 8, t->m);
  put32(b + 12, t->k);
  put32(b + 16, (uint32_t)t->m_tb);
  put32(b + 20, (uint32_t)t->k_tb);
  put32(b + 24, nt);
  memcpy(b + 28, t->offsets, 4 * ((size_t)nt + 1));
  memcpy(b + 28 + 4 * ((size_t)nt + 1), t->entries, 4 * (size_t)t->n_entries);
  *buf = b;
  *size = sz;
  return ORC_OK;
}

int orc_deserialize(const uint8_t *d, size_t size, orc_tcsl **out) {
  if (size < 4) return ORC_TRUNCATED;
  if (memcmp(d, "TCSL", 4) != 0) return ORC_BAD_MAGIC;
  if (size < 6) return ORC_TRUNCATED;
  if ((d[4] | (d[5] << 8)) != 1) return ORC_BAD_VERSION;
  if (size < 8) return ORC_TRUNCATED;
  const uint16_t flags = (uint16_t)(d[6] | (d[7] << 8));
  if (flags & ~1u) return ORC_BAD_VERSION;
  if (size < 24) return ORC_TRUNCATED;
  const uint32_t m = get32(d + 8), k = get32(d + 12), m_tb = get32(d + 16), k_tb = get32(d + 20);
  if (m == 0 || k == 0) return ORC_BAD_HEADER;
  if (m_tb == 0 || k_tb == 0 || m_tb > 65536 || k_tb > 65536) return ORC_BAD_HEADER;
  if (orc_tile_validate((int)m_tb, (int)k_tb, 1)) return ORC_BAD_HEADER;
  if (size < 28) return ORC_TRUNCATED;
  const uint32_t nt = get32(d + 24);
  orc_tcsl probe = orc_tcsl_view(m, k, (int)m_tb, (int)k_tb, 0, NULL, NULL, 0);
  if (nt != probe.num_tiles) return ORC_BAD_HEADER;
  const size_t off_bytes = 4 * ((size_t)nt + 1);
  if (size < 28 + off_bytes) return ORC_TRUNCATED;
  const uint8_t *po = d + 28;
  if (get32(po) != 0) return ORC_INCONSISTENT_OFFSETS;
  for (uint32_t i = 0; i < nt; ++i) {
    const uint32_t a = get32(po + 4 * i), b = get32(po + 4 * (i + 1));
    if (b < a) return ORC_INCONSISTENT_OFFSETS;
    if ((b - a) % 32 != 0) return ORC_INCONSISTENT_OFFSETS;
  }
  const uint32_t ne = get32(po + 4 * (size_t)nt);
  if (size < 28 + off_bytes + 4 * (size_t)ne) return ORC_TRUNCATED;
  if (size != 28 + off_bytes + 4 * (size_t)ne) return ORC_TRAILING_DATA;
  orc_tcsl *t = (orc_tcsl *)calloc(1, sizeof(orc_tcsl));
  if (!t) return ORC_NO_MEMORY;
  *t = probe;
  t->reordered = flags & 1u;
  t->offsets = (uint32_t *)malloc(off_bytes);
  t->entries = (uint32_t *)malloc(4 * (size_t)ne + 4);
  if (!t->offsets || !t->entries) {
    orc_tcsl_free(t);
    return ORC_NO_MEMORY;
  }
  memcpy(t->offsets, po, off_bytes);
  memcpy(t->entries, po + off_bytes, 4 * (size_t)ne);
  t->n_entries = ne;
  *out = t;
  return ORC_OK;
}

/* proj/tests/acceptance.cpp:25-32 */
uint64_t orc_fnv1a(const uint8_t *data, size_t size) {
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < size; ++i) {
    h ^= data[i];
    h *= 1099511628211ull;
  }
  return h;
}

void orc_free(void *p) { free(p); }
