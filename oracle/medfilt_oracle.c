/*
 * medfilt_oracle.c -- TEST INFRASTRUCTURE ONLY (the CPU checker, never the product).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  The CUDA product path never links it.
 *
 * A plain-C restatement of the reference's sorting-based median filter
 * (arXiv 1406.1717; /root/reference/proj/include/medfilt), written from the
 * algorithm, not copied.  Every function cites the reference lines it follows.
 * Pinned by tests/test_oracle.py against (a) the SPEC golden vectors,
 * (b) the reference library itself compiled into oracle/_ref/ (see
 * oracle/Makefile) and (c) the golden checksums in tests/golden/configs.json
 * that the reference produced on the five BASELINE configs.
 *
 * Values are carried as int64 "keys"; int32 inputs widen losslessly and the
 * float inputs go through the order-preserving bit-key map,
 * so one code path serves all four dtypes.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* status codes mirror include/medfilt_gpu.h (mf_status) */
enum { ORC_OK = 0, ORC_EMPTY_INPUT = 1, ORC_K_ZERO = 2, ORC_K_EVEN = 3, ORC_K_TOO_LARGE = 4,
       ORC_BAD_ARG = 5, ORC_NO_MEMORY = 7 };

/* ---- window arithmetic: make_window_spec, core.hpp:62-76; output_size core.hpp:58 ---- */
int orc_window_spec(uint64_t n, uint64_t k, uint64_t *h, uint64_t *b, uint64_t *out_len) {
  if (n == 0) return ORC_EMPTY_INPUT;            /* core.hpp:63 */
  if (k == 0) return ORC_K_ZERO;                 /* core.hpp:64 */
  if (k % 2 == 0) return ORC_K_EVEN;             /* core.hpp:65-67 */
  if (k >= 0xFFFFFFFFull) return ORC_K_TOO_LARGE; /* core.hpp:68-69, index_t = uint32 */
  if (h) *h = (k - 1) / 2;                       /* core.hpp:73 */
  if (b) *b = (n + k - 1) / k;                   /* core.hpp:74 */
  if (out_len) *out_len = n < k ? 0 : n - k + 1; /* core.hpp:58 */
  return ORC_OK;
}

/* ---- key map: IEEE bits -> signed key realising totalOrder; involution ---- */
void orc_keymap_f32(const uint32_t *bits, int32_t *key, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    int32_t s = (int32_t)bits[i];
    key[i] = s >= 0 ? s : (int32_t)(s ^ 0x7FFFFFFF);
  }
}
void orc_keymap_f64(const uint64_t *bits, int64_t *key, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    int64_t s = (int64_t)bits[i];
    key[i] = s >= 0 ? s : (int64_t)(s ^ 0x7FFFFFFFFFFFFFFFll);
  }
}

/* ---- Sample order: sample_less core.hpp:34-38, indexed_less core.hpp:42-47 ----
 * A sample is (value, sentinel).  The +INF sentinel (core.hpp:26-28) pads the
 * tail of the last block (filter.hpp:28-36). */
typedef struct { int64_t v; int inf; } orc_sample;

static inline int s_less(orc_sample a, orc_sample b) {
  if (a.inf != b.inf) return b.inf;
  return a.v < b.v;
}
static inline int s_iless(orc_sample a, uint32_t ia, orc_sample b, uint32_t ib) {
  if (a.inf != b.inf) return b.inf;
  if (a.v != b.v) return a.v < b.v;
  return ia < ib;
}

/* ---- piecewise_sort, filter.hpp:41-54: stable sort of (value, index) pairs per block ---- */
typedef struct { int64_t v; uint32_t i; } orc_pair;
static int pair_cmp(const void *pa, const void *pb) {
  const orc_pair *a = (const orc_pair *)pa, *b = (const orc_pair *)pb;
  if (a->v != b->v) return a->v < b->v ? -1 : 1;
  return a->i < b->i ? -1 : (a->i > b->i);
}

/* Sort one block of padded samples; sentinels carry v = INT64_MAX and sit at
 * the tail (filter.hpp:46-47 sorts plain (value,index) pairs for this reason). */
static void sort_block(const orc_sample *blk, uint32_t k, orc_pair *tmp, uint32_t *perm) {
  for (uint32_t i = 0; i < k; ++i) { tmp[i].v = blk[i].v; tmp[i].i = i; }
  qsort(tmp, k, sizeof(orc_pair), pair_cmp);
  for (uint32_t t = 0; t < k; ++t) perm[t] = tmp[t].i;
}

/* ---- Block<T>, block.hpp:24-146: dancing-links sorted list over one block ---- */
typedef struct {
  uint32_t k, h, m;   /* node k is the head/tail sentinel; m = median cursor */
  uint64_t s;         /* number of small elements */
  orc_sample *alpha;  /* k+1 samples, alpha[k] = +INF (block.hpp:31) */
  uint32_t *prev, *next;
} orc_block;

static int block_init(orc_block *B, uint32_t k, uint32_t h) {
  B->k = k; B->h = h; B->m = k; B->s = 0;
  B->alpha = (orc_sample *)malloc(sizeof(orc_sample) * (k + 1));
  B->prev = (uint32_t *)malloc(sizeof(uint32_t) * (k + 1));
  B->next = (uint32_t *)malloc(sizeof(uint32_t) * (k + 1));
  if (!B->alpha || !B->prev || !B->next) return ORC_NO_MEMORY;
  for (uint32_t i = 0; i <= k; ++i) { B->alpha[i].v = INT64_MAX; B->alpha[i].inf = 1; }
  return ORC_OK;
}
static void block_free(orc_block *B) { free(B->alpha); free(B->prev); free(B->next); }

/* construct, block.hpp:36-55: link the whole sorted list, s = h, m = pi[h] */
static void block_construct(orc_block *B, const orc_sample *alpha, const uint32_t *pi) {
  uint32_t k = B->k, p = k;
  memcpy(B->alpha, alpha, sizeof(orc_sample) * k);
  for (uint32_t t = 0; t < k; ++t) { uint32_t q = pi[t]; B->next[p] = q; B->prev[q] = p; p = q; }
  B->next[p] = k; B->prev[k] = p;
  B->s = B->h; B->m = pi[B->h];
}
/* unwind, block.hpp:60-69: delete k-1..0, leaving the stale links undelete needs */
static void block_unwind(orc_block *B) {
  for (uint32_t i = B->k; i-- > 0;) {
    uint32_t p = B->prev[i], q = B->next[i];
    B->next[p] = q; B->prev[q] = p;
  }
  B->m = B->k; B->s = 0;
}
/* below_cursor, block.hpp:129-132 */
static inline int block_below(const orc_block *B, uint32_t i) {
  return s_iless(B->alpha[i], i, B->alpha[B->m], B->m);
}
/* del, block.hpp:71-87 */
static void block_del(orc_block *B, uint32_t i) {
  uint32_t p = B->prev[i], q = B->next[i];
  B->next[p] = q; B->prev[q] = p;
  if (block_below(B, i)) { B->s--; return; }
  if (B->m == i) B->m = q;
  if (B->s > 0) { B->m = B->prev[B->m]; B->s--; }
}
/* undelete, block.hpp:89-98 */
static void block_undel(orc_block *B, uint32_t i) {
  uint32_t p = B->prev[i], q = B->next[i];
  B->next[p] = i; B->prev[q] = i;
  if (block_below(B, i)) B->m = B->prev[B->m];
}
/* advance block.hpp:100-104; peek block.hpp:108-111 */
static inline void block_advance(orc_block *B) { B->m = B->next[B->m]; B->s++; }
static inline orc_sample block_peek(const orc_block *B) { return B->alpha[B->m]; }

/* Optional per-step state trace (for phase-level parity of the GPU walk). */
typedef struct { uint32_t mA, mB; uint32_t sA, sB; } orc_state;

/* ---- median_filter, filter.hpp:149-155 = pad_to_blocks (:28-36) -> piecewise_sort (:41-54)
 *      -> run_postprocess (:64-106).  y gets max(0, n-k+1) values. ---- */
static int median_filter_core(const int64_t *x, uint64_t n, uint64_t k, int64_t *y,
                              orc_state *trace) {
  uint64_t h, b, keep;
  int st = orc_window_spec(n, k, &h, &b, &keep);
  if (st) return st;
  uint32_t K = (uint32_t)k;
  /* pad_to_blocks: b*k samples with a +INF tail (filter.hpp:28-36) */
  orc_sample *pad = (orc_sample *)malloc(sizeof(orc_sample) * b * k);
  uint32_t *pa = (uint32_t *)malloc(sizeof(uint32_t) * k), *pb = (uint32_t *)malloc(sizeof(uint32_t) * k);
  orc_pair *tmp = (orc_pair *)malloc(sizeof(orc_pair) * k);
  orc_block A, B;
  int okA = block_init(&A, K, (uint32_t)h), okB = block_init(&B, K, (uint32_t)h);
  if (!pad || !pa || !pb || !tmp || okA || okB) { st = ORC_NO_MEMORY; goto out; }
  for (uint64_t i = 0; i < b * k; ++i) {
    if (i < n) { pad[i].v = x[i]; pad[i].inf = 0; } else { pad[i].v = INT64_MAX; pad[i].inf = 1; }
  }
  /* run_postprocess, filter.hpp:64-106.  Blocks are sorted lazily here (piecewise_sort
   * has no cross-block dependency, filter.hpp:45-53), which keeps memory O(k). */
  uint64_t emitted = 0;
#define EMIT(S) do { if (emitted < keep) y[emitted] = (S).v; ++emitted; } while (0)
  sort_block(pad, K, tmp, pb);
  block_construct(&B, pad, pb);                      /* :81 */
  EMIT(block_peek(&B));                              /* :82 */
  for (uint64_t j = 1; j < b && emitted < keep; ++j) {
    orc_block t = A; A = B; B = t;                   /* :84 swap */
    sort_block(pad + j * k, K, tmp, pb);
    block_construct(&B, pad + j * k, pb);            /* :85 */
    block_unwind(&B);                                /* :86 */
    for (uint32_t i = 0; i < K; ++i) {               /* :87-101 */
      block_del(&A, i);
      block_undel(&B, i);
      if (A.s + B.s < h) {                           /* :90 */
        if (!s_less(block_peek(&B), block_peek(&A))) block_advance(&A); /* ties -> A, :92-93 */
        else block_advance(&B);
      }
      if (trace && emitted < keep) {
        trace[emitted].mA = A.m; trace[emitted].mB = B.m;
        trace[emitted].sA = (uint32_t)A.s; trace[emitted].sB = (uint32_t)B.s;
      }
      orc_sample qa = block_peek(&A), qb = block_peek(&B);
      EMIT(s_less(qb, qa) ? qb : qa);                /* :98-100 */
      if (emitted >= keep) break;                    /* never walk sentinel windows */
    }
  }
#undef EMIT
out:
  free(pad); free(pa); free(pb); free(tmp);
  block_free(&A); block_free(&B);
  return st;
}

int orc_median_filter_i64(const int64_t *x, uint64_t n, uint64_t k, int64_t *y) {
  return median_filter_core(x, n, k, y, NULL);
}
int orc_median_filter_trace_i64(const int64_t *x, uint64_t n, uint64_t k, int64_t *y,
                                uint32_t *trace4) {
  return median_filter_core(x, n, k, y, (orc_state *)trace4);
}
int orc_median_filter_i32(const int32_t *x, uint64_t n, uint64_t k, int32_t *y) {
  uint64_t keep; int st = orc_window_spec(n, k, NULL, NULL, &keep);
  if (st) return st;
  int64_t *w = (int64_t *)malloc(sizeof(int64_t) * n), *o = (int64_t *)malloc(sizeof(int64_t) * (keep + 1));
  if (!w || !o) { free(w); free(o); return ORC_NO_MEMORY; }
  for (uint64_t i = 0; i < n; ++i) w[i] = x[i];
  st = median_filter_core(w, n, k, o, NULL);
  for (uint64_t i = 0; i < keep; ++i) y[i] = (int32_t)o[i];
  free(w); free(o);
  return st;
}
int orc_median_filter_f32(const uint32_t *x, uint64_t n, uint64_t k, uint32_t *y) {
  uint64_t keep; int st = orc_window_spec(n, k, NULL, NULL, &keep);
  if (st) return st;
  int32_t *kx = (int32_t *)malloc(sizeof(int32_t) * n), *ky = (int32_t *)malloc(sizeof(int32_t) * (keep + 1));
  if (!kx || !ky) { free(kx); free(ky); return ORC_NO_MEMORY; }
  orc_keymap_f32(x, kx, n);
  st = orc_median_filter_i32(kx, n, k, ky);
  orc_keymap_f32((const uint32_t *)ky, (int32_t *)y, keep);  /* involution maps back */
  free(kx); free(ky);
  return st;
}
int orc_median_filter_f64(const uint64_t *x, uint64_t n, uint64_t k, uint64_t *y) {
  uint64_t keep; int st = orc_window_spec(n, k, NULL, NULL, &keep);
  if (st) return st;
  int64_t *kx = (int64_t *)malloc(sizeof(int64_t) * n), *ky = (int64_t *)malloc(sizeof(int64_t) * (keep + 1));
  if (!kx || !ky) { free(kx); free(ky); return ORC_NO_MEMORY; }
  orc_keymap_f64(x, kx, n);
  st = median_filter_core(kx, n, k, ky, NULL);
  orc_keymap_f64((const uint64_t *)ky, (int64_t *)y, keep);
  free(kx); free(ky);
  return st;
}

/* ---- piecewise_sort exported for phase parity: perms[j*k + t] (filter.hpp:41-54) ---- */
int orc_piecewise_sort_i64(const int64_t *x, uint64_t n, uint64_t k, uint32_t *perms) {
  uint64_t h, b; int st = orc_window_spec(n, k, &h, &b, NULL);
  if (st) return st;
  orc_pair *tmp = (orc_pair *)malloc(sizeof(orc_pair) * k);
  orc_sample *blk = (orc_sample *)malloc(sizeof(orc_sample) * k);
  if (!tmp || !blk) { free(tmp); free(blk); return ORC_NO_MEMORY; }
  for (uint64_t j = 0; j < b; ++j) {
    for (uint64_t i = 0; i < k; ++i) {
      uint64_t g = j * k + i;
      blk[i].v = g < n ? x[g] : INT64_MAX; blk[i].inf = g >= n;
    }
    sort_block(blk, (uint32_t)k, tmp, perms + j * k);
  }
  free(tmp); free(blk);
  return ORC_OK;
}

/* ---- naive_median_filter, baselines.hpp:287-300: copy + sort every window ---- */
static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}
int orc_naive_i64(const int64_t *x, uint64_t n, uint64_t k, int64_t *y) {
  uint64_t h, keep; int st = orc_window_spec(n, k, &h, NULL, &keep);
  if (st) return st;
  int64_t *w = (int64_t *)malloc(sizeof(int64_t) * k);
  if (!w) return ORC_NO_MEMORY;
  for (uint64_t i = 0; i < keep; ++i) {
    memcpy(w, x + i, sizeof(int64_t) * k);
    qsort(w, k, sizeof(int64_t), cmp_i64);
    y[i] = w[h];
  }
  free(w);
  return ORC_OK;
}

/* ---- fold_checksum, io.hpp:17-28: FNV-1a over sign-extended 64-bit values ---- */
uint64_t orc_fold_checksum_i64(const int64_t *v, uint64_t n) {
  uint64_t hsh = 1469598103934665603ull;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t bits = (uint64_t)v[i];
    for (int byte = 0; byte < 8; ++byte) { hsh ^= (bits >> (8 * byte)) & 0xff; hsh *= 1099511628211ull; }
  }
  return hsh;
}
uint64_t orc_fold_checksum_i32(const int32_t *v, uint64_t n) {
  uint64_t hsh = 1469598103934665603ull;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t bits = (uint64_t)(int64_t)v[i];
    for (int byte = 0; byte < 8; ++byte) { hsh ^= (bits >> (8 * byte)) & 0xff; hsh *= 1099511628211ull; }
  }
  return hsh;
}

/* ---- multi-threaded halo-sharded run (the CPU baseline on all host cores).
 * Shard g computes outputs [o_g, o_{g+1}) from x[o_g, o_{g+1}+k-1): SURVEY.md §0.7 / §8(e). ---- */
typedef struct { const int64_t *x; uint64_t n, k; int64_t *y; int st; } orc_job;
static void *orc_job_run(void *p) {
  orc_job *j = (orc_job *)p;
  j->st = median_filter_core(j->x, j->n, j->k, j->y, NULL);
  return NULL;
}
int orc_median_filter_threads_i64(const int64_t *x, uint64_t n, uint64_t k, int64_t *y, int threads) {
  uint64_t keep; int st = orc_window_spec(n, k, NULL, NULL, &keep);
  if (st) return st;
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > keep) threads = keep ? (int)keep : 1;
  if (keep == 0) return ORC_OK;
  pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * threads);
  orc_job *jobs = (orc_job *)malloc(sizeof(orc_job) * threads);
  for (int g = 0; g < threads; ++g) {
    uint64_t o0 = keep * g / threads, o1 = keep * (g + 1) / threads;
    jobs[g].x = x + o0; jobs[g].n = o1 - o0 + k - 1; jobs[g].k = k; jobs[g].y = y + o0; jobs[g].st = 0;
    pthread_create(&tid[g], NULL, orc_job_run, &jobs[g]);
  }
  for (int g = 0; g < threads; ++g) { pthread_join(tid[g], NULL); if (jobs[g].st) st = jobs[g].st; }
  free(tid); free(jobs);
  return st;
}

/* ---- SplitMix64, generators.hpp:16-29, and the BASELINE input recipes ---- */
static inline uint64_t sm64_next(uint64_t *s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
void orc_splitmix64(uint64_t seed, uint64_t *out, uint64_t n) {
  uint64_t s = seed;
  for (uint64_t i = 0; i < n; ++i) out[i] = sm64_next(&s);
}
/* uniform f64 in [0,1): (next>>11) * 2^-53 */
void orc_gen_uniform_f64(uint64_t seed, double *out, uint64_t n) {
  uint64_t s = seed;
  for (uint64_t i = 0; i < n; ++i) out[i] = (double)(sm64_next(&s) >> 11) * 0x1.0p-53;
}
/* uniform f32 in [0,1): (float)((next>>40) * 2^-24) -- exact */
void orc_gen_uniform_f32(uint64_t seed, float *out, uint64_t n) {
  uint64_t s = seed;
  for (uint64_t i = 0; i < n; ++i) out[i] = (float)((double)(sm64_next(&s) >> 40) * 0x1.0p-24);
}
/* c3: next() % 16 as int32, one stream row-major */
void orc_gen_mod_i32(uint64_t seed, uint64_t mod, int32_t *out, uint64_t n) {
  uint64_t s = seed;
  for (uint64_t i = 0; i < n; ++i) out[i] = (int32_t)(sm64_next(&s) % mod);
}
/* c4: x_i = i/n + 0.01 * sqrt(-2 ln(1-u1)) * cos(2 pi u2), evaluated left to right exactly as
 * written ((0.01*sqrt)*cos); pinned by the golden in_cksum.  Build with -ffp-contract=off. */
void orc_gen_trend_f64(uint64_t seed, double *out, uint64_t n) {
  uint64_t s = seed;
  const double two_pi = 2.0 * 3.14159265358979323846;
  for (uint64_t i = 0; i < n; ++i) {
    double u1 = (double)(sm64_next(&s) >> 11) * 0x1.0p-53;
    double u2 = (double)(sm64_next(&s) >> 11) * 0x1.0p-53;
    out[i] = (double)i / (double)n + 0.01 * sqrt(-2.0 * log(1.0 - u1)) * cos(two_pi * u2);
  }
}

/* ---- the SPEC generator kinds, generators.hpp:91-142 (asc..r-block), 64-bit values ---- */
int orc_generate_i64(int kind, uint64_t n, uint64_t seed, int width, int64_t *out) {
  uint64_t s = seed;
  const uint64_t noise = 10000, base_bound = 1000000, blen = 1000;
  if (n == 0) return ORC_BAD_ARG;
  uint64_t base = 0;
  for (uint64_t i = 0; i < n; ++i) {
    switch (kind) {
      case 0: out[i] = (int64_t)i; break;                                   /* asc */
      case 1: out[i] = (int64_t)(n - i); break;                             /* desc */
      case 2: out[i] = (int64_t)(i + sm64_next(&s) % noise); break;         /* r-asc */
      case 3: out[i] = (int64_t)(n - i + sm64_next(&s) % noise); break;     /* r-desc */
      case 4: {                                                             /* r-large */
        uint64_t r = sm64_next(&s);
        out[i] = width == 32 ? (int64_t)(int32_t)(uint32_t)r : (int64_t)r;
        break;
      }
      case 5: out[i] = (int64_t)(sm64_next(&s) % noise); break;             /* r-small */
      case 6:                                                               /* r-block */
        if (i % blen == 0) base = sm64_next(&s) % base_bound;
        out[i] = (int64_t)(base + sm64_next(&s) % noise);
        break;
      default: return ORC_BAD_ARG;
    }
  }
  return ORC_OK;
}
