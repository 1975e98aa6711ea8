/*
 * fm_oracle.c — CPU restatement of the reference's hot path, used ONLY as a
 * test checker and as the CPU baseline of bench.py.  TEST INFRASTRUCTURE:
 * nothing in the product package (paper_1811_06127_b200/) links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs do.
 *
 * It reads the index exactly as the reference stores it: .fmi bucket records
 * of 4 x u64 base + 32 packed bytes per 128 characters (index.py:24-36,
 * serialize.py:87-92), and follows the reference algorithms line by line:
 *
 *   all4_bytelut      kernels.py:80-93, 238-247  (the AUTO/default kernel)
 *   occ_all           occ.py:44-56
 *   occ_pair_all      occ.py:59-96
 *   exact_search      search.py:74-94 (init_interval 50-57, extend 60-71)
 *   inexact_search    search.py:97-159 (LIFO DFS, dict dedup, sorted output)
 *   psi_inverse_fused search.py:172-186
 *   locate_row        search.py:189-208
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/, tests/test_oracle.py).  Batch wrappers split the work over
 * POSIX threads in contiguous shards.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const uint8_t* rec; /* nb x 64 bytes */
  uint64_t nb, n, sentinel_row;
  uint64_t c[5];
  const uint64_t* samples; /* n/32 + 1, may be NULL */
} fmo_index;

/* _BYTE_COUNTS_PACKED (kernels.py:80-93): the four symbol counts of one byte
 * packed 8 bits per symbol. */
static uint32_t g_lut[256];
static pthread_once_t g_lut_once = PTHREAD_ONCE_INIT;
static void build_lut(void) {
  for (int b = 0; b < 256; ++b) {
    uint32_t packed = 0;
    for (int sh = 0; sh < 8; sh += 2) packed += 1u << (((b >> sh) & 3) << 3);
    g_lut[b] = packed;
  }
}

static inline uint64_t base_of(const fmo_index* ix, uint64_t j, int s) {
  uint64_t v;
  memcpy(&v, ix->rec + j * 64 + 8 * s, 8);
  return v;
}

/* _all4_bytelut (kernels.py:238-247): counts among the first prefix_len fields. */
static void all4_bytelut(const uint8_t* chars, int prefix_len, uint64_t out[4]) {
  int full = prefix_len >> 2, rem = prefix_len & 3;
  uint32_t packed = 0;
  for (int i = 0; i < full; ++i) packed += g_lut[chars[i]];
  for (int s = 0; s < 4; ++s) out[s] = (packed >> (s << 3)) & 0xFF;
  if (rem) {
    uint8_t b = chars[full];
    for (int f = 0; f < rem; ++f) out[(b >> (f << 1)) & 3]++;
  }
}

/* occ_all (occ.py:44-56); k in [-1, n]. Returns 0, or -1 on a bad position. */
int fmo_occ_all(const fmo_index* ix, int64_t k, uint64_t out[4]) {
  pthread_once(&g_lut_once, build_lut);
  if (k == -1) {
    out[0] = out[1] = out[2] = out[3] = 0;
    return 0;
  }
  if (k < 0 || (uint64_t)k > ix->n) return -1;
  uint64_t j = (uint64_t)k >> 7, r = (uint64_t)k & 127;
  uint64_t inside[4];
  all4_bytelut(ix->rec + j * 64 + 32, (int)r + 1, inside);
  for (int s = 0; s < 4; ++s) out[s] = base_of(ix, j, s) + inside[s];
  if (ix->sentinel_row <= (uint64_t)k) out[0] -= 1;
  return 0;
}

/* occ_pair_all (occ.py:59-96); out = [low A,C,G,T, high A,C,G,T]. */
int fmo_occ_pair_all(const fmo_index* ix, int64_t low, int64_t high, uint64_t out[8]) {
  pthread_once(&g_lut_once, build_lut);
  if (low > high) return -1;
  if (low == high) {
    if (fmo_occ_all(ix, high, out + 4)) return -1;
    memcpy(out, out + 4, 32);
    return 0;
  }
  if (low < 0) {
    if (low != -1) return -1;
    out[0] = out[1] = out[2] = out[3] = 0;
    return fmo_occ_all(ix, high, out + 4);
  }
  if ((uint64_t)high > ix->n) return -1;
  uint64_t jl = (uint64_t)low >> 7, rl = (uint64_t)low & 127;
  uint64_t jh = (uint64_t)high >> 7, rh = (uint64_t)high & 127;
  if (jl != jh) {
    fmo_occ_all(ix, low, out);
    fmo_occ_all(ix, high, out + 4);
    return 0;
  }
  const uint8_t* chars = ix->rec + jl * 64 + 32;
  uint64_t in_l[4], in_h[4];
  all4_bytelut(chars, (int)rl + 1, in_l);
  all4_bytelut(chars, (int)rh + 1, in_h);
  for (int s = 0; s < 4; ++s) {
    out[s] = base_of(ix, jl, s) + in_l[s];
    out[4 + s] = base_of(ix, jl, s) + in_h[s];
  }
  if (ix->sentinel_row <= (uint64_t)low) out[0] -= 1;
  if (ix->sentinel_row <= (uint64_t)high) out[4] -= 1;
  return 0;
}

/* exact_search (search.py:74-94) on codes[0..m), m >= 1. */
void fmo_exact(const fmo_index* ix, const uint8_t* codes, uint64_t m, int64_t* k_out, int64_t* l_out) {
  int b = codes[m - 1];
  int64_t k = (int64_t)ix->c[b] + 1, l = (int64_t)ix->c[b + 1]; /* init_interval */
  uint64_t pair[8];
  for (uint64_t t = m - 1; t-- > 0;) {
    if (k > l) break;
    int s = codes[t];
    fmo_occ_pair_all(ix, k - 1, l, pair); /* extend_backward */
    int64_t cs = (int64_t)ix->c[s];
    k = cs + (int64_t)pair[s] + 1;
    l = cs + (int64_t)pair[4 + s];
  }
  *k_out = k;
  *l_out = l;
}

/* ---- inexact_search (search.py:97-159) ---------------------------------- */

typedef struct {
  int64_t i, budget, k, l;
} node_t;
typedef struct {
  int64_t k, l, used;
} term_t;

typedef struct {
  term_t* v;
  uint64_t n, cap;
} termvec;

static int termvec_push(termvec* tv, int64_t k, int64_t l, int64_t used) {
  if (tv->n == tv->cap) {
    uint64_t nc = tv->cap ? tv->cap * 2 : 64;
    term_t* nv = (term_t*)realloc(tv->v, nc * sizeof(term_t));
    if (!nv) return -1;
    tv->v = nv;
    tv->cap = nc;
  }
  tv->v[tv->n].k = k;
  tv->v[tv->n].l = l;
  tv->v[tv->n].used = used;
  tv->n++;
  return 0;
}

static int cmp_term(const void* a, const void* b) {
  const term_t* x = (const term_t*)a;
  const term_t* y = (const term_t*)b;
  if (x->k != y->k) return x->k < y->k ? -1 : 1;
  if (x->l != y->l) return x->l < y->l ? -1 : 1;
  if (x->used != y->used) return x->used < y->used ? -1 : 1;
  return 0;
}

/* Appends the deduplicated, sorted results of one pattern to `out`; returns
 * the number appended, or -1 on allocation failure.  `steps` (optional)
 * accumulates the Occ steps executed (one per non-terminal pop). */
static int64_t inexact_one(const fmo_index* ix, const uint8_t* codes, uint64_t m, int64_t z, termvec* out,
                           uint64_t* steps) {
  node_t* stack = NULL;
  uint64_t sp = 0, cap = 0;
  termvec raw = {NULL, 0, 0};
#define PUSH(I, B, K, L)                                                  \
  do {                                                                    \
    if (sp == cap) {                                                      \
      uint64_t nc = cap ? cap * 2 : 256;                                  \
      node_t* ns = (node_t*)realloc(stack, nc * sizeof(node_t));          \
      if (!ns) goto oom;                                                  \
      stack = ns;                                                         \
      cap = nc;                                                           \
    }                                                                     \
    stack[sp].i = (I);                                                    \
    stack[sp].budget = (B);                                               \
    stack[sp].k = (K);                                                    \
    stack[sp].l = (L);                                                    \
    sp++;                                                                 \
  } while (0)

  PUSH((int64_t)m - 1, z, 0, (int64_t)ix->n); /* root, search.py:125 */
  uint64_t pair[8];
  while (sp) {
    node_t nd = stack[--sp];
    if (nd.i < 0) {
      if (termvec_push(&raw, nd.k, nd.l, z - nd.budget)) goto oom;
      continue;
    }
    if (nd.budget > 0) PUSH(nd.i - 1, nd.budget - 1, nd.k, nd.l); /* skip */
    fmo_occ_pair_all(ix, nd.k - 1, nd.l, pair);
    if (steps) (*steps)++;
    int want = codes[nd.i];
    for (int s = 0; s < 4; ++s) {
      int64_t base = (int64_t)ix->c[s];
      int64_t k2 = base + (int64_t)pair[s] + 1;
      int64_t l2 = base + (int64_t)pair[4 + s];
      if (k2 > l2) continue;
      if (nd.budget > 0) PUSH(nd.i, nd.budget - 1, k2, l2); /* insert */
      if (s == want)
        PUSH(nd.i - 1, nd.budget, k2, l2); /* match */
      else if (nd.budget > 0)
        PUSH(nd.i - 1, nd.budget - 1, k2, l2); /* mismatch */
    }
  }
#undef PUSH
  free(stack);
  /* best[(k, l)] = min used; sorted by (k, l, diffs) */
  if (raw.n) qsort(raw.v, raw.n, sizeof(term_t), cmp_term);
  int64_t added = 0;
  for (uint64_t i = 0; i < raw.n; ++i) {
    if (i > 0 && raw.v[i].k == raw.v[i - 1].k && raw.v[i].l == raw.v[i - 1].l) continue;
    if (termvec_push(out, raw.v[i].k, raw.v[i].l, raw.v[i].used)) {
      free(raw.v);
      return -1;
    }
    added++;
  }
  free(raw.v);
  return added;
oom:
  free(stack);
  free(raw.v);
  return -1;
}

/* psi_inverse_fused (search.py:172-186): returns -1 at the sentinel row,
 * -2 on a bad row; else the predecessor row, with *sym set. */
int64_t fmo_psi(const fmo_index* ix, int64_t i, int* sym) {
  pthread_once(&g_lut_once, build_lut);
  if (i < 0 || (uint64_t)i > ix->n) return -2;
  if ((uint64_t)i == ix->sentinel_row) return -1;
  uint64_t j = (uint64_t)i >> 7, r = (uint64_t)i & 127;
  const uint8_t* chars = ix->rec + j * 64 + 32;
  int s = (chars[r >> 2] >> ((r & 3) << 1)) & 3;
  uint64_t inside[4];
  all4_bytelut(chars, (int)r + 1, inside); /* count_fn(kernel)(chars, r+1, s) */
  int64_t count = (int64_t)(base_of(ix, j, s) + inside[s]);
  if (s == 0 && ix->sentinel_row <= (uint64_t)i) count -= 1;
  *sym = s;
  return (int64_t)ix->c[s] + count;
}

/* locate_row (search.py:189-208); -1 on a corrupt walk. */
int64_t fmo_locate_row(const fmo_index* ix, int64_t i) {
  int64_t steps = 0;
  for (;;) {
    if ((uint64_t)i == ix->sentinel_row) return steps;
    if ((i & 31) == 0) return (int64_t)ix->samples[i >> 5] + steps;
    int sym;
    i = fmo_psi(ix, i, &sym);
    if (i < 0) return -1;
    steps++;
    if ((uint64_t)steps > ix->n + 1) return -1;
  }
}

/* ---- threaded batch wrappers --------------------------------------------- */

typedef struct {
  const fmo_index* ix;
  uint64_t lo, hi;
  int kind;
  const int64_t* a;
  const int64_t* b;
  uint32_t* out32;
  const uint8_t* codes;
  const uint64_t* offsets;
  int64_t* kl;
  int64_t z;
  termvec res;
  uint32_t* counts;
  uint64_t steps;
  int failed;
} job_t;

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  uint64_t pair[8];
  for (uint64_t q = j->lo; q < j->hi; ++q) {
    switch (j->kind) {
      case 0: /* occ pairs */
        if (fmo_occ_pair_all(j->ix, j->a[q], j->b[q], pair)) {
          j->failed = 1;
          memset(pair, 0, sizeof(pair));
        }
        for (int s = 0; s < 8; ++s) j->out32[q * 8 + s] = (uint32_t)pair[s];
        break;
      case 1: /* exact */
        fmo_exact(j->ix, j->codes + j->offsets[q], j->offsets[q + 1] - j->offsets[q], &j->kl[2 * q],
                  &j->kl[2 * q + 1]);
        break;
      case 2: { /* inexact */
        int64_t r = inexact_one(j->ix, j->codes + j->offsets[q], j->offsets[q + 1] - j->offsets[q], j->z,
                                &j->res, &j->steps);
        if (r < 0) {
          j->failed = 1;
          return NULL;
        }
        j->counts[q] = (uint32_t)r;
        break;
      }
      case 3: /* locate */
        j->kl[q] = fmo_locate_row(j->ix, j->a[q]);
        break;
    }
  }
  return NULL;
}

static int run_jobs(job_t* proto, uint64_t count, int nthreads, job_t** jobs_out) {
  if (nthreads < 1) nthreads = 1;
  if ((uint64_t)nthreads > count) nthreads = count ? (int)count : 1;
  job_t* jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  if (!jobs || !th) {
    free(jobs);
    free(th);
    return -1;
  }
  uint64_t chunk = (count + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = *proto;
    jobs[t].lo = chunk * t < count ? chunk * t : count;
    jobs[t].hi = chunk * (t + 1) < count ? chunk * (t + 1) : count;
    pthread_create(&th[t], NULL, run_job, &jobs[t]);
  }
  int failed = 0;
  for (int t = 0; t < nthreads; ++t) {
    pthread_join(th[t], NULL);
    failed |= jobs[t].failed;
  }
  free(th);
  if (jobs_out)
    *jobs_out = jobs;
  else
    free(jobs);
  return failed ? -1 : nthreads;
}

int fmo_occ_pair_batch(const fmo_index* ix, const int64_t* low, const int64_t* high, uint64_t count, uint32_t* out,
                       int nthreads) {
  pthread_once(&g_lut_once, build_lut);
  job_t p;
  memset(&p, 0, sizeof(p));
  p.ix = ix;
  p.kind = 0;
  p.a = low;
  p.b = high;
  p.out32 = out;
  return run_jobs(&p, count, nthreads, NULL) < 0 ? -1 : 0;
}

int fmo_exact_batch(const fmo_index* ix, const uint8_t* codes, const uint64_t* offsets, uint64_t count,
                    int64_t* kl_out, int nthreads) {
  pthread_once(&g_lut_once, build_lut);
  job_t p;
  memset(&p, 0, sizeof(p));
  p.ix = ix;
  p.kind = 1;
  p.codes = codes;
  p.offsets = offsets;
  p.kl = kl_out;
  return run_jobs(&p, count, nthreads, NULL) < 0 ? -1 : 0;
}

int fmo_locate_batch(const fmo_index* ix, const int64_t* rows, uint64_t count, int64_t* pos_out, int nthreads) {
  pthread_once(&g_lut_once, build_lut);
  job_t p;
  memset(&p, 0, sizeof(p));
  p.ix = ix;
  p.kind = 3;
  p.a = rows;
  p.kl = pos_out;
  return run_jobs(&p, count, nthreads, NULL) < 0 ? -1 : 0;
}

/* Inexact batch: results land in a library-owned CSR (fmo_inexact_fetch). */
typedef struct {
  uint64_t count, total, steps;
  uint64_t* row_off;
  int64_t* k;
  int64_t* l;
  uint8_t* diffs;
} fmo_matches;

fmo_matches* fmo_inexact_batch(const fmo_index* ix, const uint8_t* codes, const uint64_t* offsets, uint64_t count,
                               int64_t z, int nthreads) {
  pthread_once(&g_lut_once, build_lut);
  fmo_matches* m = (fmo_matches*)calloc(1, sizeof(fmo_matches));
  uint32_t* counts = (uint32_t*)calloc(count ? count : 1, sizeof(uint32_t));
  if (!m || !counts) {
    free(m);
    free(counts);
    return NULL;
  }
  job_t p;
  memset(&p, 0, sizeof(p));
  p.ix = ix;
  p.kind = 2;
  p.codes = codes;
  p.offsets = offsets;
  p.z = z;
  p.counts = counts;
  job_t* jobs = NULL;
  int nt = run_jobs(&p, count, nthreads, &jobs);
  if (nt < 0) {
    free(counts);
    free(m);
    free(jobs);
    return NULL;
  }
  m->count = count;
  m->row_off = (uint64_t*)calloc(count + 1, sizeof(uint64_t));
  for (uint64_t q = 0; q < count; ++q) m->row_off[q + 1] = m->row_off[q] + counts[q];
  m->total = m->row_off[count];
  m->k = (int64_t*)malloc((m->total ? m->total : 1) * sizeof(int64_t));
  m->l = (int64_t*)malloc((m->total ? m->total : 1) * sizeof(int64_t));
  m->diffs = (uint8_t*)malloc(m->total ? m->total : 1);
  uint64_t o = 0;
  for (int t = 0; t < nt; ++t) { /* shards are contiguous and in order */
    for (uint64_t i = 0; i < jobs[t].res.n; ++i, ++o) {
      m->k[o] = jobs[t].res.v[i].k;
      m->l[o] = jobs[t].res.v[i].l;
      m->diffs[o] = (uint8_t)jobs[t].res.v[i].used;
    }
    m->steps += jobs[t].steps;
    free(jobs[t].res.v);
  }
  free(jobs);
  free(counts);
  return m;
}

uint64_t fmo_matches_total(const fmo_matches* m) { return m->total; }
uint64_t fmo_matches_steps(const fmo_matches* m) { return m->steps; }
void fmo_matches_fetch(const fmo_matches* m, uint64_t* row_off, int64_t* k, int64_t* l, uint8_t* diffs) {
  memcpy(row_off, m->row_off, (m->count + 1) * sizeof(uint64_t));
  if (m->total) {
    memcpy(k, m->k, m->total * sizeof(int64_t));
    memcpy(l, m->l, m->total * sizeof(int64_t));
    memcpy(diffs, m->diffs, m->total);
  }
}
void fmo_matches_free(fmo_matches* m) {
  if (!m) return;
  free(m->row_off);
  free(m->k);
  free(m->l);
  free(m->diffs);
  free(m);
}
