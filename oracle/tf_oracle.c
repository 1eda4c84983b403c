/*
 * tf_oracle.c -- CPU restatement of the reference tile-fusion inspector and
 * executors, written in plain C from the reference's behaviour.
 *
 * TEST INFRASTRUCTURE ONLY (see tf_oracle.h).  The product path never links
 * this file.  Parity is pinned against the reference's known-answer tests
 * and against golden vectors dumped from the reference itself (oracle/_ref).
 *
 * Build without -march and with -ffp-contract=off: the reference is built
 * with -O3 and no -march (CMakeLists.txt:8-10), so its x86-64 code performs
 * every product and sum as a separately rounded mul then add
 * (kernels.hpp:54-55).  Keeping the same order makes the oracle bit-exact.
 */
#include "tf_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* error plumbing                                                       */
/* ------------------------------------------------------------------ */
static _Thread_local char g_err[512];

const char *tfo_last_error(void) { return g_err; }

static int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}
#define INVALID 1

/* ------------------------------------------------------------------ */
/* small containers                                                     */
/* ------------------------------------------------------------------ */
typedef struct {
  int32_t *d;
  int64_t n, cap;
} ivec;

static void iv_push(ivec *v, int32_t x) {
  if (v->n == v->cap) {
    v->cap = v->cap ? v->cap * 2 : 16;
    v->d = (int32_t *)realloc(v->d, (size_t)v->cap * sizeof(int32_t));
  }
  v->d[v->n++] = x;
}
static void iv_free(ivec *v) {
  free(v->d);
  v->d = NULL;
  v->n = v->cap = 0;
}

typedef struct {
  int32_t lo, hi;
  ivec j;
  double cost;
} otile;

typedef struct {
  otile *d;
  int64_t n, cap;
} tvec;

static void tv_push(tvec *v, otile t) {
  if (v->n == v->cap) {
    v->cap = v->cap ? v->cap * 2 : 16;
    v->d = (otile *)realloc(v->d, (size_t)v->cap * sizeof(otile));
  }
  v->d[v->n++] = t;
}

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* Pattern view: the scheduler reads only row_ptr / col_idx
 * (SparsityView, csr.hpp:118-140). */
typedef struct {
  int32_t n_rows, n_cols;
  const int32_t *rp, *ci;
} pview;

static inline int32_t rnnz(const pview *a, int32_t r) {
  return a->rp[r + 1] - a->rp[r];
}

/* ------------------------------------------------------------------ */
/* inspector                                                            */
/* ------------------------------------------------------------------ */

/* choose_tile_size -- scheduler.cpp:124-129 */
int tfo_choose_tile_size(int32_t n, int32_t p, int32_t ct, int32_t *out) {
  if (n < 1 || p < 1 || ct < 1)
    return fail(INVALID, "choose_tile_size: all inputs must be >= 1");
  int32_t tiles = (n + ct - 1) / ct;
  *out = tiles >= p ? ct : (n + p - 1) / p;
  return 0;
}

/* Epoch-marked distinct-column scratch -- scheduler.cpp:19-27 */
typedef struct {
  int64_t *mark;
  int64_t epoch;
} scratch_t;

/* tile_cost_ws -- scheduler.cpp:29-64.  Integer counts are exact in double,
 * so counting in int64 and converting reproduces the reference's doubles. */
static double tile_cost_ws(const pview *a, int32_t lo, int32_t hi,
                           const int32_t *j, int64_t nj, const tfo_config *cfg,
                           scratch_t *s) {
  const double t = (double)(hi - lo);
  const double jc = (double)nj;
  int64_t nnzj = 0, uc = 0;
  const int64_t ep = ++s->epoch;
  for (int64_t q = 0; q < nj; ++q) {
    const int32_t r = j[q];
    for (int32_t k = a->rp[r]; k < a->rp[r + 1]; ++k) {
      ++nnzj;
      const int32_t col = a->ci[k];
      if (s->mark[col] != ep) {
        s->mark[col] = ep;
        ++uc;
      }
    }
  }
  const double dn = (double)nnzj, du = (double)uc;
  const double cc = (double)cfg->c_cols, bc = (double)cfg->b_cols;
  if (cfg->b_is_dense) {
    const double first = cfg->whole_b_cost ? (double)a->n_rows : t;
    const double idx = ceil((dn + jc + 1.0) * cfg->index_to_scalar_ratio);
    return (du + t + jc) * cc + first * bc + idx;
  }
  int64_t nb = 0;
  for (int32_t i = lo; i < hi; ++i) nb += rnnz(a, i);
  const double db = (double)nb;
  const double idx =
      ceil((dn + jc + 1.0 + db + t + 1.0) * cfg->index_to_scalar_ratio);
  return (db + dn + du + t + jc) * cc + idx;
}

/* split_rec -- scheduler.cpp:66-93: emit when under budget or width 1,
 * else bisect at lo + w/2; straddling rows are demoted; left then right. */
static void split_rec(const pview *a, otile tile, const tfo_config *cfg,
                      scratch_t *s, tvec *pieces, ivec *demoted) {
  tile.cost = tile_cost_ws(a, tile.lo, tile.hi, tile.j.d, tile.j.n, cfg, s);
  if (tile.cost <= (double)cfg->cache_size_words || tile.hi - tile.lo <= 1) {
    tv_push(pieces, tile);
    return;
  }
  const int32_t mid = tile.lo + (tile.hi - tile.lo) / 2;
  otile left = {tile.lo, mid, {0}, 0.0};
  otile right = {mid, tile.hi, {0}, 0.0};
  for (int64_t q = 0; q < tile.j.n; ++q) {
    const int32_t r = tile.j.d[q];
    const int32_t b = a->rp[r], e = a->rp[r + 1];
    if (b == e) {
      iv_push(r < mid ? &left.j : &right.j, r);
    } else if (a->ci[e - 1] < mid) {
      iv_push(&left.j, r);
    } else if (a->ci[b] >= mid) {
      iv_push(&right.j, r);
    } else {
      iv_push(demoted, r);
    }
  }
  iv_free(&tile.j);
  split_rec(a, left, cfg, s, pieces, demoted);
  split_rec(a, right, cfg, s, pieces, demoted);
}

/* bisect_by_count -- scheduler.cpp:95-113 */
static void bisect_by_count(const pview *a, otile tile, const tfo_config *cfg,
                            scratch_t *s, tvec *out) {
  tile.cost = tile_cost_ws(a, tile.lo, tile.hi, tile.j.d, tile.j.n, cfg, s);
  if (tile.cost <= (double)cfg->cache_size_words || tile.j.n <= 1) {
    tv_push(out, tile);
    return;
  }
  const int64_t half = tile.j.n / 2;
  otile left = {0, 0, {0}, 0.0}, right = {0, 0, {0}, 0.0};
  for (int64_t q = 0; q < half; ++q) iv_push(&left.j, tile.j.d[q]);
  for (int64_t q = half; q < tile.j.n; ++q) iv_push(&right.j, tile.j.d[q]);
  iv_free(&tile.j);
  bisect_by_count(a, left, cfg, s, out);
  bisect_by_count(a, right, cfg, s, out);
}

static int require_square(const pview *a, const char *who) {
  if (a->n_rows != a->n_cols)
    return fail(INVALID, "%s: matrix must be square", who);
  if (a->n_rows < 1) return fail(INVALID, "%s: matrix must be nonempty", who);
  return 0;
}

/* step1_coarse_fuse -- scheduler.cpp:131-161 (tiles as a vector) */
static int step1_tiles(const pview *a, int32_t t, tvec *tiles, ivec *unfused) {
  int rc = require_square(a, "step1_coarse_fuse");
  if (rc) return rc;
  if (t < 1) return fail(INVALID, "step1_coarse_fuse: tile_size must be >= 1");
  const int32_t n = a->n_rows;
  const int32_t nt = (int32_t)(((int64_t)n + t - 1) / t);
  for (int32_t v = 0; v < nt; ++v) {
    otile o = {(int32_t)((int64_t)v * t), 0, {0}, 0.0};
    int64_t hi = (int64_t)(v + 1) * t;
    o.hi = (int32_t)(hi < n ? hi : n);
    tv_push(tiles, o);
  }
  for (int32_t j = 0; j < n; ++j) {
    const int32_t b = a->rp[j], e = a->rp[j + 1];
    if (b == e) {
      iv_push(&tiles->d[j / t].j, j);
      continue;
    }
    const int32_t v = a->ci[b] / t;
    if (a->ci[e - 1] < tiles->d[v].hi)
      iv_push(&tiles->d[v].j, j);
    else
      iv_push(unfused, j);
  }
  return 0;
}

int tfo_step1(int32_t n_rows, int32_t n_cols, const int32_t *row_ptr,
              const int32_t *col_idx, int32_t t, int64_t *tile_j_off,
              int32_t *tile_j_rows, int32_t *unfused, int64_t *n_unfused) {
  pview a = {n_rows, n_cols, row_ptr, col_idx};
  tvec tiles = {0};
  ivec un = {0};
  int rc = step1_tiles(&a, t, &tiles, &un);
  if (rc) return rc;
  int64_t off = 0;
  for (int64_t v = 0; v < tiles.n; ++v) {
    tile_j_off[v] = off;
    memcpy(tile_j_rows + off, tiles.d[v].j.d,
           (size_t)tiles.d[v].j.n * sizeof(int32_t));
    off += tiles.d[v].j.n;
    iv_free(&tiles.d[v].j);
  }
  tile_j_off[tiles.n] = off;
  if (un.n) memcpy(unfused, un.d, (size_t)un.n * sizeof(int32_t));
  *n_unfused = un.n;
  iv_free(&un);
  free(tiles.d);
  return 0;
}

/* balance -- scheduler.cpp:163-194: greedy fill to the running ideal
 * ceil(rem/rem_chunks), keeping one row in reserve per remaining chunk. */
int tfo_balance(const int32_t *rows, int64_t m, const int32_t *w,
                int64_t num_chunks, int64_t *chunk_off) {
  if (num_chunks < 1) return fail(INVALID, "balance: num_chunks must be >= 1");
  int64_t rem = 0;
  for (int64_t q = 0; q < m; ++q) rem += w[rows[q]];
  int64_t i = 0;
  int64_t c = 0;
  for (; c < num_chunks && i < m; ++c) {
    chunk_off[c] = i;
    const int64_t rc = num_chunks - c;
    const int64_t ideal = (rem + rc - 1) / rc;
    int64_t acc = w[rows[i++]];
    while (i < m && m - i > rc - 1) {
      const int64_t nx = w[rows[i]];
      if (acc + nx > ideal) break;
      acc += nx;
      ++i;
    }
    rem -= acc;
  }
  for (; c <= num_chunks; ++c) chunk_off[c] = i;
  return 0;
}

int tfo_tile_cost(int32_t n_rows, const int32_t *row_ptr,
                  const int32_t *col_idx, int32_t i_lo, int32_t i_hi,
                  const int32_t *j_rows, int64_t nj, const tfo_config *cfg,
                  double *out) {
  pview a = {n_rows, n_rows, row_ptr, col_idx};
  scratch_t s = {(int64_t *)calloc((size_t)n_rows + 1, sizeof(int64_t)), 0};
  *out = tile_cost_ws(&a, i_lo, i_hi, j_rows, nj, cfg, &s);
  free(s.mark);
  return 0;
}

static void flatten_wave(const tvec *tv, tfo_schedule *out, int w) {
  out->n_tiles[w] = tv->n;
  int64_t total = 0;
  for (int64_t v = 0; v < tv->n; ++v) total += tv->d[v].j.n;
  out->i_lo[w] = (int32_t *)malloc((size_t)(tv->n + 1) * sizeof(int32_t));
  out->i_hi[w] = (int32_t *)malloc((size_t)(tv->n + 1) * sizeof(int32_t));
  out->cost[w] = (double *)malloc((size_t)(tv->n + 1) * sizeof(double));
  out->j_off[w] = (int64_t *)malloc((size_t)(tv->n + 1) * sizeof(int64_t));
  out->j_rows[w] = (int32_t *)malloc((size_t)(total + 1) * sizeof(int32_t));
  int64_t off = 0;
  for (int64_t v = 0; v < tv->n; ++v) {
    const otile *t = &tv->d[v];
    out->i_lo[w][v] = t->lo;
    out->i_hi[w][v] = t->hi;
    out->cost[w][v] = t->cost;
    out->j_off[w][v] = off;
    if (t->j.n) memcpy(out->j_rows[w] + off, t->j.d, (size_t)t->j.n * 4);
    off += t->j.n;
  }
  out->j_off[w][tv->n] = off;
}

static void free_tvec(tvec *tv) {
  for (int64_t v = 0; v < tv->n; ++v) iv_free(&tv->d[v].j);
  free(tv->d);
  tv->d = NULL;
  tv->n = tv->cap = 0;
}

/* split_tile -- scheduler.cpp:202-210 */
int tfo_split_tile(int32_t n_rows, const int32_t *row_ptr,
                   const int32_t *col_idx, int32_t i_lo, int32_t i_hi,
                   const int32_t *j_rows, int64_t nj, const tfo_config *cfg,
                   tfo_schedule *pieces, int32_t **demoted,
                   int64_t *n_demoted) {
  pview a = {n_rows, n_rows, row_ptr, col_idx};
  scratch_t s = {(int64_t *)calloc((size_t)n_rows + 1, sizeof(int64_t)), 0};
  otile t = {i_lo, i_hi, {0}, 0.0};
  for (int64_t q = 0; q < nj; ++q) iv_push(&t.j, j_rows[q]);
  tvec out = {0};
  ivec dem = {0};
  split_rec(&a, t, cfg, &s, &out, &dem);
  if (dem.n) qsort(dem.d, (size_t)dem.n, sizeof(int32_t), cmp_i32);
  memset(pieces, 0, sizeof *pieces);
  pieces->n = n_rows;
  flatten_wave(&out, pieces, 0);
  tvec none = {0};
  flatten_wave(&none, pieces, 1);
  *demoted = (int32_t *)malloc((size_t)(dem.n + 1) * sizeof(int32_t));
  if (dem.n) memcpy(*demoted, dem.d, (size_t)dem.n * 4);
  *n_demoted = dem.n;
  free_tvec(&out);
  iv_free(&dem);
  free(s.mark);
  return 0;
}

/* build_schedule -- scheduler.cpp:212-245 */
int tfo_build_schedule(int32_t n_rows, int32_t n_cols, const int32_t *row_ptr,
                       const int32_t *col_idx, const tfo_config *cfg,
                       tfo_schedule *out) {
  pview a = {n_rows, n_cols, row_ptr, col_idx};
  memset(out, 0, sizeof *out);
  int rc = require_square(&a, "build_schedule");
  if (rc) return rc;
  const int32_t n = n_rows;
  int32_t t;
  rc = tfo_choose_tile_size(n, cfg->num_workers, cfg->ct_size, &t);
  if (rc) return rc;
  tvec tiles = {0};
  ivec unfused = {0};
  rc = step1_tiles(&a, t, &tiles, &unfused);
  if (rc) return rc;

  scratch_t s = {(int64_t *)calloc((size_t)n + 1, sizeof(int64_t)), 0};
  tvec w0 = {0}, w1 = {0};
  for (int64_t v = 0; v < tiles.n; ++v)
    split_rec(&a, tiles.d[v], cfg, &s, &w0, &unfused);
  free(tiles.d);

  if (unfused.n) {
    qsort(unfused.d, (size_t)unfused.n, sizeof(int32_t), cmp_i32);
    int32_t *wts = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    for (int32_t j = 0; j < n; ++j) wts[j] = rnnz(&a, j);
    const int64_t by_ct = (unfused.n + cfg->ct_size - 1) / cfg->ct_size;
    const int64_t chunks =
        (int64_t)cfg->num_workers > by_ct ? (int64_t)cfg->num_workers : by_ct;
    int64_t *off = (int64_t *)malloc((size_t)(chunks + 1) * sizeof(int64_t));
    tfo_balance(unfused.d, unfused.n, wts, chunks, off);
    for (int64_t c = 0; c < chunks; ++c) {
      if (off[c + 1] == off[c]) continue;
      otile o = {0, 0, {0}, 0.0};
      for (int64_t q = off[c]; q < off[c + 1]; ++q) iv_push(&o.j, unfused.d[q]);
      bisect_by_count(&a, o, cfg, &s, &w1);
    }
    free(off);
    free(wts);
  }
  iv_free(&unfused);
  free(s.mark);

  out->n = n;
  out->tile_size = t;
  flatten_wave(&w0, out, 0);
  flatten_wave(&w1, out, 1);
  free_tvec(&w0);
  free_tvec(&w1);
  return 0;
}

void tfo_schedule_free(tfo_schedule *s) {
  for (int w = 0; w < 2; ++w) {
    free(s->i_lo[w]);
    free(s->i_hi[w]);
    free(s->cost[w]);
    free(s->j_off[w]);
    free(s->j_rows[w]);
  }
  memset(s, 0, sizeof *s);
}

void tfo_free(void *p) { free(p); }

/* fused_ratio -- scheduler.cpp:247-252 (Eq. 2) */
double tfo_fused_ratio(const tfo_schedule *s) {
  if (s->n < 1) return 0.0;
  const int64_t fused = s->j_off[0] ? s->j_off[0][s->n_tiles[0]] : 0;
  return (double)fused / (2.0 * (double)s->n);
}

/* ------------------------------------------------------------------ */
/* validate_schedule -- scheduler.cpp:254-390                           */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t count;
  char *buf;
  size_t len, cap;
} vlog;

static void vfail(vlog *l, const char *fmt, ...) {
  char tmp[256];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(tmp, sizeof tmp, fmt, ap);
  va_end(ap);
  size_t k = strlen(tmp);
  if (l->len + k + 2 > l->cap) {
    l->cap = (l->len + k + 2) * 2;
    l->buf = (char *)realloc(l->buf, l->cap);
  }
  memcpy(l->buf + l->len, tmp, k);
  l->len += k;
  l->buf[l->len++] = '\n';
  l->buf[l->len] = 0;
  l->count++;
}

typedef struct {
  int32_t lo, hi;
} rng2;
static int cmp_rng(const void *a, const void *b) {
  const rng2 *x = (const rng2 *)a, *y = (const rng2 *)b;
  if (x->lo != y->lo) return (x->lo > y->lo) - (x->lo < y->lo);
  return (x->hi > y->hi) - (x->hi < y->hi);
}

static int64_t validate_core(const pview *a, const tfo_schedule *s,
                             const tfo_config *cfg, int64_t *ob1, vlog *l) {
  const int square = a->n_rows == a->n_cols;
  if (!square) vfail(l, "matrix is not square");
  const int32_t n = a->n_rows;
  if (s->n != n) vfail(l, "schedule n does not match matrix");
  if (!square || s->n != n) return l->count;

  /* wavefront-0 i_ranges partition [0, n) */
  const int64_t n0 = s->n_tiles[0], n1 = s->n_tiles[1];
  rng2 *rs = (rng2 *)malloc((size_t)(n0 + 1) * sizeof(rng2));
  int64_t nr = 0;
  for (int64_t v = 0; v < n0; ++v) {
    const int32_t lo = s->i_lo[0][v], hi = s->i_hi[0][v];
    if (lo >= hi) {
      vfail(l, "wavefront-0 tile with empty i_range [%d,%d)", lo, hi);
      continue;
    }
    if (lo < 0 || hi > n) {
      vfail(l, "i_range out of bounds");
      continue;
    }
    rs[nr].lo = lo;
    rs[nr].hi = hi;
    ++nr;
  }
  qsort(rs, (size_t)nr, sizeof(rng2), cmp_rng);
  int32_t expect = 0;
  int contiguous = 1;
  for (int64_t q = 0; q < nr; ++q) {
    if (rs[q].lo != expect) {
      vfail(l, "i coverage gap or overlap at %d (expected %d)", rs[q].lo,
            expect);
      contiguous = 0;
      break;
    }
    expect = rs[q].hi;
  }
  if (contiguous && nr > 0 && expect != n)
    vfail(l, "i coverage stops at %d", expect);
  if (nr == 0 && n > 0) vfail(l, "wavefront 0 covers nothing");
  free(rs);

  for (int64_t v = 0; v < n1; ++v)
    if (s->i_lo[1][v] != s->i_hi[1][v]) {
      vfail(l, "wavefront-1 tile carries a nonempty i_range");
      break;
    }

  /* j lists partition [0, n) */
  char *seen = (char *)calloc((size_t)n + 1, 1);
  int64_t seen_count = 0;
  for (int w = 0; w < 2; ++w) {
    for (int64_t v = 0; v < s->n_tiles[w]; ++v) {
      int32_t prev = -1;
      for (int64_t q = s->j_off[w][v]; q < s->j_off[w][v + 1]; ++q) {
        const int32_t j = s->j_rows[w][q];
        if (j < 0 || j >= n) {
          vfail(l, "j out of range: %d", j);
          continue;
        }
        if (j <= prev) vfail(l, "j_list not strictly ascending");
        prev = j;
        if (seen[j]) {
          vfail(l, "j appears twice: %d", j);
        } else {
          seen[j] = 1;
          ++seen_count;
        }
      }
    }
  }
  if (seen_count != n)
    vfail(l, "j coverage incomplete: %lld of %d", (long long)seen_count, n);
  free(seen);

  /* dependence closure for fused rows */
  for (int64_t v = 0; v < n0; ++v) {
    const int32_t lo = s->i_lo[0][v], hi = s->i_hi[0][v];
    int ok = 1;
    for (int64_t q = s->j_off[0][v]; q < s->j_off[0][v + 1] && ok; ++q) {
      const int32_t j = s->j_rows[0][q];
      if (j < 0 || j >= n) continue;
      for (int32_t k = a->rp[j]; k < a->rp[j + 1]; ++k) {
        const int32_t col = a->ci[k];
        if (col < lo || col >= hi) {
          vfail(l, "row %d fused into [%d,%d) but depends on %d", j, lo, hi,
                col);
          ok = 0;
          break;
        }
      }
    }
  }

  /* cost bound, width-1 / single-row tiles exempt */
  {
    scratch_t sc = {(int64_t *)calloc((size_t)n + 1, sizeof(int64_t)), 0};
    const double budget = (double)cfg->cache_size_words;
    for (int w = 0; w < 2; ++w) {
      for (int64_t v = 0; v < s->n_tiles[w]; ++v) {
        const int64_t b = s->j_off[w][v], e = s->j_off[w][v + 1];
        int bad = 0;
        for (int64_t q = b; q < e; ++q)
          if (s->j_rows[w][q] < 0 || s->j_rows[w][q] >= n) bad = 1;
        if (bad) continue;
        const double cost = tile_cost_ws(a, s->i_lo[w][v], s->i_hi[w][v],
                                         s->j_rows[w] + b, e - b, cfg, &sc);
        if (cost <= budget) continue;
        const int irreducible = w == 0
                                    ? (s->i_hi[w][v] - s->i_lo[w][v]) <= 1
                                    : (e - b) <= 1;
        if (irreducible)
          ++*ob1;
        else
          vfail(l, "splittable tile exceeds cache budget (cost %f)", cost);
      }
    }
    free(sc.mark);
  }

  /* wavefront balance */
  const int64_t p = cfg->num_workers;
  if (s->tile_size < 1) {
    vfail(l, "tile_size must be >= 1");
  } else {
    const int64_t avail0 = ((int64_t)n + s->tile_size - 1) / s->tile_size;
    const int64_t need = p < avail0 ? p : avail0;
    if (n0 < need)
      vfail(l, "wavefront 0 has too few tiles for %lld workers", (long long)p);
  }
  const int64_t w1_rows = n1 ? s->j_off[1][n1] : 0;
  const int64_t need1 = p < w1_rows ? p : w1_rows;
  if (n1 < need1)
    vfail(l, "wavefront 1 has too few tiles for %lld workers", (long long)p);
  return l->count;
}

int tfo_validate_schedule(int32_t n_rows, int32_t n_cols,
                          const int32_t *row_ptr, const int32_t *col_idx,
                          const tfo_schedule *s, const tfo_config *cfg,
                          int64_t *n_violations, int64_t *over_budget_width1,
                          char *first_msg, size_t msg_cap) {
  pview a = {n_rows, n_cols, row_ptr, col_idx};
  vlog l = {0};
  int64_t ob1 = 0;
  validate_core(&a, s, cfg, &ob1, &l);
  *n_violations = l.count;
  *over_budget_width1 = ob1;
  if (first_msg && msg_cap) {
    first_msg[0] = 0;
    if (l.buf) {
      size_t k = strcspn(l.buf, "\n");
      if (k >= msg_cap) k = msg_cap - 1;
      memcpy(first_msg, l.buf, k);
      first_msg[k] = 0;
    }
  }
  free(l.buf);
  return l.count == 0;
}

int tfo_validate_schedule_all(int32_t n_rows, int32_t n_cols,
                              const int32_t *row_ptr, const int32_t *col_idx,
                              const tfo_schedule *s, const tfo_config *cfg,
                              char **messages) {
  pview a = {n_rows, n_cols, row_ptr, col_idx};
  vlog l = {0};
  int64_t ob1 = 0;
  validate_core(&a, s, cfg, &ob1, &l);
  if (!l.buf) l.buf = (char *)calloc(1, 1);
  *messages = l.buf;
  return l.count == 0;
}

/* ------------------------------------------------------------------ */
/* executors -- kernels.hpp:54-155                                      */
/* ------------------------------------------------------------------ */
/* gemm_row (kernels.hpp:57-67): out[k] = sum_j B[i,j]*C[j,k], j ascending,
 * separately rounded products and sums.
 * spmm_row (kernels.hpp:71-80): out[q] = sum_k A.val[k]*X[A.col[k],q]. */
#define DEFINE_EXEC(T, SFX)                                                   \
  static void first_row_##SFX(int32_t i, const int32_t *brp,                  \
                              const int32_t *bci, const T *bv,                \
                              const T *bdense, int32_t bc, const T *c,        \
                              int32_t cc, T *out) {                           \
    for (int32_t k = 0; k < cc; ++k) out[k] = (T)0;                           \
    if (!brp) {                                                               \
      const T *brow = bdense + (size_t)i * bc;                                \
      for (int32_t j = 0; j < bc; ++j) {                                      \
        const T bij = brow[j];                                                \
        const T *crow = c + (size_t)j * cc;                                   \
        for (int32_t k = 0; k < cc; ++k) {                                    \
          T prod = bij * crow[k];                                             \
          out[k] = out[k] + prod;                                             \
        }                                                                     \
      }                                                                       \
    } else {                                                                  \
      for (int32_t e = brp[i]; e < brp[i + 1]; ++e) {                         \
        const T v = bv[e];                                                    \
        const T *crow = c + (size_t)bci[e] * cc;                              \
        for (int32_t k = 0; k < cc; ++k) {                                    \
          T prod = v * crow[k];                                               \
          out[k] = out[k] + prod;                                             \
        }                                                                     \
      }                                                                       \
    }                                                                         \
  }                                                                           \
  static void spmm_row_##SFX(int32_t r, const int32_t *arp,                   \
                             const int32_t *aci, const T *av, const T *x,     \
                             int32_t cc, T *out) {                            \
    for (int32_t q = 0; q < cc; ++q) out[q] = (T)0;                           \
    for (int32_t e = arp[r]; e < arp[r + 1]; ++e) {                           \
      const T v = av[e];                                                      \
      const T *xrow = x + (size_t)aci[e] * cc;                                \
      for (int32_t q = 0; q < cc; ++q) {                                      \
        T prod = v * xrow[q];                                                 \
        out[q] = out[q] + prod;                                               \
      }                                                                       \
    }                                                                         \
  }                                                                           \
  int tfo_run_##SFX(int32_t n, const int32_t *arp, const int32_t *aci,        \
                    const T *av, const int32_t *brp, const int32_t *bci,      \
                    const T *bv, const T *bdense, int32_t bc, const T *c,     \
                    int32_t cc, const tfo_schedule *sched, T *d,              \
                    int64_t *stats) {                                         \
    if (sched && sched->n != n)                                               \
      return fail(INVALID, "schedule and problem disagree on n");             \
    T *d1 = (T *)calloc((size_t)n * cc + 1, sizeof(T));                       \
    memset(d, 0, (size_t)n * cc * sizeof(T));                                 \
    int64_t fr = 0, sr = 0;                                                   \
    if (sched) {                                                              \
      for (int w = 0; w < 2; ++w) {                                           \
        for (int64_t v = 0; v < sched->n_tiles[w]; ++v) {                     \
          for (int32_t i = sched->i_lo[w][v]; i < sched->i_hi[w][v]; ++i) {   \
            first_row_##SFX(i, brp, bci, bv, bdense, bc, c, cc,               \
                            d1 + (size_t)i * cc);                             \
            ++fr;                                                             \
          }                                                                   \
          for (int64_t q = sched->j_off[w][v]; q < sched->j_off[w][v + 1];    \
               ++q) {                                                         \
            const int32_t j = sched->j_rows[w][q];                            \
            spmm_row_##SFX(j, arp, aci, av, d1, cc, d + (size_t)j * cc);      \
            ++sr;                                                             \
          }                                                                   \
        }                                                                     \
      }                                                                       \
    } else {                                                                  \
      for (int32_t i = 0; i < n; ++i, ++fr)                                   \
        first_row_##SFX(i, brp, bci, bv, bdense, bc, c, cc,                   \
                        d1 + (size_t)i * cc);                                 \
      for (int32_t j = 0; j < n; ++j, ++sr)                                   \
        spmm_row_##SFX(j, arp, aci, av, d1, cc, d + (size_t)j * cc);          \
    }                                                                         \
    free(d1);                                                                 \
    if (stats) {                                                              \
      stats[0] += fr;                                                         \
      stats[1] += sr;                                                         \
    }                                                                         \
    return 0;                                                                 \
  }                                                                           \
  int tfo_run_##SFX##_mt(int32_t n, const int32_t *arp, const int32_t *aci,   \
                         const T *av, const int32_t *brp, const int32_t *bci, \
                         const T *bv, const T *bdense, int32_t bc,            \
                         const T *c, int32_t cc, const tfo_schedule *sched,   \
                         T *d, int workers) {                                 \
    if (workers < 1) return fail(INVALID, "workers must be >= 1");            \
    if (sched && sched->n != n)                                               \
      return fail(INVALID, "schedule and problem disagree on n");             \
    T *d1 = (T *)calloc((size_t)n * cc + 1, sizeof(T));                       \
    if (sched) {                                                              \
      for (int w = 0; w < 2; ++w) {                                           \
        const int64_t nt = sched->n_tiles[w];                                 \
        if (!nt) continue;                                                    \
        _Pragma("omp parallel for schedule(dynamic, 1) num_threads(workers)") \
        for (int64_t v = 0; v < nt; ++v) {                                    \
          for (int32_t i = sched->i_lo[w][v]; i < sched->i_hi[w][v]; ++i)     \
            first_row_##SFX(i, brp, bci, bv, bdense, bc, c, cc,               \
                            d1 + (size_t)i * cc);                             \
          for (int64_t q = sched->j_off[w][v]; q < sched->j_off[w][v + 1];    \
               ++q) {                                                         \
            const int32_t j = sched->j_rows[w][q];                            \
            spmm_row_##SFX(j, arp, aci, av, d1, cc, d + (size_t)j * cc);      \
          }                                                                   \
        }                                                                     \
      }                                                                       \
    } else {                                                                  \
      _Pragma("omp parallel for schedule(static) num_threads(workers)")       \
      for (int32_t i = 0; i < n; ++i)                                         \
        first_row_##SFX(i, brp, bci, bv, bdense, bc, c, cc,                   \
                        d1 + (size_t)i * cc);                                 \
      _Pragma("omp parallel for schedule(static) num_threads(workers)")       \
      for (int32_t j = 0; j < n; ++j)                                         \
        spmm_row_##SFX(j, arp, aci, av, d1, cc, d + (size_t)j * cc);          \
    }                                                                         \
    free(d1);                                                                 \
    return 0;                                                                 \
  }

DEFINE_EXEC(double, f64)
DEFINE_EXEC(float, f32)

/* ------------------------------------------------------------------ */
/* generators                                                           */
/* ------------------------------------------------------------------ */
/* std::mt19937_64 (the standard's parameters). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64 *g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) +
               (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64 *g) {
  if (g->idx >= 312) {
    static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

void tfo_mt64_stream(uint64_t seed, uint64_t *out, int64_t count) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = mt64_next(&g);
}

/* libstdc++ generate_canonical<double,53> over a 64-bit engine: one draw
 * scaled by 2^-64, clamped below 1. */
static double canon(mt64 *g) {
  double r = (double)mt64_next(g) * 1.0;
  r = r / 18446744073709551616.0;
  if (r >= 1.0) r = nextafter(1.0, 0.0);
  return r;
}
/* uniform_real_distribution<double>(a,b): canon*(b-a)+a */
static double uniform(mt64 *g, double a, double b) {
  double x = canon(g) * (b - a);
  return x + a;
}

typedef struct {
  ivec rp, ci;
  double *v;
  int64_t nv, cv;
} csrb;

static void cb_val(csrb *m, double x) {
  if (m->nv == m->cv) {
    m->cv = m->cv ? m->cv * 2 : 64;
    m->v = (double *)realloc(m->v, (size_t)m->cv * sizeof(double));
  }
  m->v[m->nv++] = x;
}

/* gen_random_sparse -- generate.hpp:15-63: geometric skipping with
 * 53-bit draws; empty rows get their diagonal. */
int tfo_gen_random_sparse(int32_t n, double density, uint64_t seed,
                          int32_t **row_ptr, int32_t **col_idx,
                          double **values) {
  if (n < 1) return fail(INVALID, "gen_random_sparse: n must be >= 1");
  if (!(density > 0.0) || density > 1.0)
    return fail(INVALID, "gen_random_sparse: density must be in (0,1]");
  mt64 g;
  mt64_seed(&g, seed);
  csrb m = {0};
  iv_push(&m.rp, 0);
  const int full = density >= 1.0;
  const double log_skip = full ? 0.0 : log1p(-density);
  for (int32_t r = 0; r < n; ++r) {
    const int64_t start = m.ci.n;
    if (full) {
      for (int32_t c = 0; c < n; ++c) {
        iv_push(&m.ci, c);
        double x = (double)(mt64_next(&g) >> 11);
        cb_val(&m, 0.1 + 0.9 * x * 0x1.0p-53);
      }
    } else {
      int64_t c = -1;
      for (;;) {
        const double u = ((double)(mt64_next(&g) >> 11) + 0.5) * 0x1.0p-53;
        c += 1 + (int64_t)floor(log(u) / log_skip);
        if (c >= n) break;
        iv_push(&m.ci, (int32_t)c);
        double x = (double)(mt64_next(&g) >> 11);
        cb_val(&m, 0.1 + 0.9 * x * 0x1.0p-53);
      }
    }
    if (m.ci.n == start) {
      iv_push(&m.ci, r);
      double x = (double)(mt64_next(&g) >> 11);
      cb_val(&m, 0.1 + 0.9 * x * 0x1.0p-53);
    }
    iv_push(&m.rp, (int32_t)m.ci.n);
  }
  *row_ptr = m.rp.d;
  *col_idx = m.ci.d ? m.ci.d : (int32_t *)malloc(4);
  *values = m.v ? m.v : (double *)malloc(8);
  return 0;
}

/* gen_banded -- generate.hpp:66-94 */
int tfo_gen_banded(int32_t n, int32_t hb, int32_t **row_ptr,
                   int32_t **col_idx, double **values) {
  if (n < 1) return fail(INVALID, "gen_banded: n must be >= 1");
  if (hb < 0 || hb >= n)
    return fail(INVALID, "gen_banded: need 0 <= half_bandwidth < n");
  csrb m = {0};
  iv_push(&m.rp, 0);
  for (int32_t r = 0; r < n; ++r) {
    const int32_t lo = r - hb > 0 ? r - hb : 0;
    const int32_t hi = r + hb < n - 1 ? r + hb : n - 1;
    for (int32_t c = lo; c <= hi; ++c) {
      iv_push(&m.ci, c);
      cb_val(&m, 1.0);
    }
    iv_push(&m.rp, (int32_t)m.ci.n);
  }
  *row_ptr = m.rp.d;
  *col_idx = m.ci.d;
  *values = m.v;
  return 0;
}

/* tests/support.hpp:68-75 */
void tfo_random_dense(int32_t rows, int32_t cols, uint64_t seed, double *out) {
  mt64 g;
  mt64_seed(&g, seed);
  const int64_t total = (int64_t)rows * cols;
  for (int64_t k = 0; k < total; ++k) out[k] = uniform(&g, -1.0, 1.0);
}

/* tests/support.hpp:50-66 */
int tfo_gen_rect_random(int32_t rows, int32_t cols, double density,
                        uint64_t seed, int32_t **row_ptr, int32_t **col_idx,
                        double **values) {
  mt64 g;
  mt64_seed(&g, seed);
  csrb m = {0};
  iv_push(&m.rp, 0);
  for (int32_t r = 0; r < rows; ++r) {
    int any = 0;
    for (int32_t c = 0; c < cols; ++c) {
      if (uniform(&g, 0.0, 1.0) < density) {
        iv_push(&m.ci, c);
        cb_val(&m, uniform(&g, 0.1, 1.0));
        any = 1;
      }
    }
    if (!any) {
      iv_push(&m.ci, r % cols);
      cb_val(&m, uniform(&g, 0.1, 1.0));
    }
    iv_push(&m.rp, (int32_t)m.ci.n);
  }
  *row_ptr = m.rp.d;
  *col_idx = m.ci.d;
  *values = m.v;
  return 0;
}
