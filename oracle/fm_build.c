/*
 * fm_build.c — CPU restatement of the reference's index construction, used
 * ONLY by the test/benchmark infrastructure (bench.py --impl reference and
 * its cpu_baseline leg, tests/).  TEST INFRASTRUCTURE: the product package
 * never links or loads this file; it exists so that the reference arm builds
 * its index without touching libfmgpu.so (the product's host or GPU builder).
 *
 * Restates:
 *   build_suffix_array  suffix.py:21-45   prefix doubling over rank pairs
 *                                         (rank(c) = code + 1, terminator 0)
 *   bwt_from_sa         suffix.py:48-71   row i = char before suffix sa[i],
 *                                         '$' at the row of suffix 0
 *   build_index         index.py:67-101   c table of the BWT symbol totals
 *                                         ('$' excluded), 128-char buckets of
 *                                         4 x u64 exclusive base ('$' counted
 *                                         as A, code 0) + 32 packed bytes,
 *                                         sa_samples = sa[0::32]
 *
 * The suffix array of a string is unique, so the doubling may start from
 * 8-character keys and refine only the groups that are still tied (the
 * classic Manber-Myers / Larsson-Sadakane refinement of the same algorithm):
 * after round h every group holds the suffixes that agree on their first h
 * characters, ranked by group start, exactly as the reference's rank array.
 * Tied groups are refined in parallel by POSIX threads (chunks of groups
 * claimed from an atomic counter).
 *
 * Memory: 12 bytes per character (sa, rank, key) plus the initial counting
 * sort's 64 MiB histogram.  n + 1 < 2^32.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t start, len;
} group_t;

typedef struct {
  group_t* g;
  uint64_t n, cap;
} groupvec;

static int gv_push(groupvec* v, uint64_t start, uint64_t len) {
  if (v->n == v->cap) {
    uint64_t cap = v->cap ? v->cap * 2 : 1024;
    group_t* g = (group_t*)realloc(v->g, cap * sizeof(group_t));
    if (!g) return -1;
    v->g = g;
    v->cap = cap;
  }
  v->g[v->n].start = start;
  v->g[v->n].len = len;
  v->n++;
  return 0;
}

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

/* Rank of text position i in the doubling alphabet (suffix.py:29-31):
 * code + 1 for characters, 0 for the terminator and beyond. */
static inline uint32_t sym_rank(const uint8_t* codes, uint64_t n, uint64_t i) {
  return i < n ? (uint32_t)codes[i] + 1u : 0u;
}

/* Suffix array of codes[0..n) + terminator: sa[0..n]. Returns 0, or -1 on
 * allocation failure / n too large. */
typedef struct {
  const uint8_t* codes;
  uint64_t n, h;
  uint32_t *sa, *rank, *key;
  const group_t* groups;
  uint64_t n_groups;
  uint64_t next; /* atomic: next group chunk */
  int err;
} refine_job;

static void* refine_worker(void* arg) {
  refine_job* jb = (refine_job*)arg;
  uint64_t* tmp = NULL;
  uint64_t tcap = 0;
  for (;;) {
    const uint64_t g0 = __atomic_fetch_add(&jb->next, 64, __ATOMIC_RELAXED);
    if (g0 >= jb->n_groups) break;
    const uint64_t g1 = g0 + 64 < jb->n_groups ? g0 + 64 : jb->n_groups;
    for (uint64_t gi = g0; gi < g1; ++gi) {
      const group_t g = jb->groups[gi];
      if (g.len > tcap) {
        free(tmp);
        tcap = g.len * 2;
        tmp = (uint64_t*)malloc(tcap * sizeof(uint64_t));
        if (!tmp) {
          __atomic_store_n(&jb->err, 1, __ATOMIC_RELAXED);
          return NULL;
        }
      }
      for (uint64_t q = 0; q < g.len; ++q) {
        const uint32_t x = jb->sa[g.start + q];
        /* a tied suffix is longer than h (its first h ranks hold no
         * terminator, which is unique), so x + h <= n */
        tmp[q] = ((uint64_t)jb->rank[x + jb->h] << 32) | x;
      }
      qsort(tmp, g.len, sizeof(uint64_t), cmp_u64);
      for (uint64_t q = 0; q < g.len; ++q) {
        jb->sa[g.start + q] = (uint32_t)tmp[q];
        jb->key[g.start + q] = (uint32_t)(tmp[q] >> 32);
      }
    }
  }
  free(tmp);
  return NULL;
}

int fmo_build_sa(const uint8_t* codes, uint64_t n, uint32_t* sa, int nthreads) {
  const uint64_t N = n + 1;
  if (N >= 0xFFFFFFFFull) return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  /* round 0: counting sort by the first 8 ranks (3 bits each) */
  const int H0 = 8;
  const uint64_t K = 1ull << (3 * H0);
  uint32_t* rank = (uint32_t*)malloc(N * sizeof(uint32_t));
  uint32_t* key = (uint32_t*)malloc(N * sizeof(uint32_t));
  uint64_t* cnt = (uint64_t*)calloc(K + 1, sizeof(uint64_t));
  if (!rank || !key || !cnt) {
    free(rank);
    free(key);
    free(cnt);
    return -1;
  }
  for (uint64_t i = 0; i < N; ++i) {
    uint32_t k = 0;
    for (int d = 0; d < H0; ++d) k = (k << 3) | sym_rank(codes, n, (uint64_t)i + d);
    key[i] = k;
  }
  for (uint64_t i = 0; i < N; ++i) cnt[key[i] + 1]++;
  for (uint64_t k = 0; k < K; ++k) cnt[k + 1] += cnt[k];
  /* rank = group start (number of suffixes with a smaller key) */
  for (uint64_t i = 0; i < N; ++i) rank[i] = (uint32_t)cnt[key[i]];
  for (uint64_t i = 0; i < N; ++i) sa[cnt[key[i]]++] = (uint32_t)i; /* stable scatter */
  free(cnt);

  groupvec cur = {0, 0, 0};
  for (uint64_t j = 0; j < N;) {
    uint64_t e = j + 1;
    while (e < N && rank[sa[e]] == rank[sa[j]]) ++e;
    if (e - j > 1 && gv_push(&cur, j, e - j)) goto fail;
    j = e;
  }

  for (uint64_t h = H0; cur.n > 0; h <<= 1) {
    /* pass 1: sort each tied group by the rank h characters on (old ranks
     * only are read: key[] holds rank[sa[j] + h] for the group members) */
    refine_job jb = {codes, n, h, sa, rank, key, cur.g, cur.n, 0, 0};
    pthread_t th[256];
    int started = 0;
    for (int t = 1; t < nthreads && (uint64_t)t * 64 < cur.n; ++t)
      if (pthread_create(&th[started], NULL, refine_worker, &jb) == 0) ++started;
    refine_worker(&jb);
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
    const int err = jb.err;
    if (err) goto fail;
    /* pass 2: new ranks (group start of each sub-run) and the groups still tied */
    groupvec nxt = {0, 0, 0};
    for (uint64_t gi = 0; gi < cur.n; ++gi) {
      const group_t g = cur.g[gi];
      for (uint64_t a = 0; a < g.len;) {
        uint64_t b = a + 1;
        while (b < g.len && key[g.start + b] == key[g.start + a]) ++b;
        for (uint64_t q = a; q < b; ++q) rank[sa[g.start + q]] = (uint32_t)(g.start + a);
        if (b - a > 1 && gv_push(&nxt, g.start + a, b - a)) {
          free(nxt.g);
          goto fail;
        }
        a = b;
      }
    }
    free(cur.g);
    cur = nxt;
  }
  free(cur.g);
  free(rank);
  free(key);
  return 0;
fail:
  free(cur.g);
  free(rank);
  free(key);
  return -1;
}

/* bwt_from_sa + build_index (suffix.py:48-71, index.py:67-101).
 * rec: nb x 64 bytes, nb = n / 128 + 1; samples: n / 32 + 1 entries.
 * Outputs c[5] and *sentinel_row. */
int fmo_build_records(const uint8_t* codes, uint64_t n, const uint32_t* sa, uint8_t* rec, uint64_t* samples,
                      uint64_t c[5], uint64_t* sentinel_row) {
  const uint64_t N = n + 1, nb = n / 128 + 1;
  uint64_t base[4] = {0, 0, 0, 0}, totals[4] = {0, 0, 0, 0};
  uint64_t srow = (uint64_t)-1;
  memset(rec, 0, nb * 64);
  for (uint64_t j = 0; j < nb; ++j) {
    uint8_t* r = rec + j * 64;
    memcpy(r, base, 32); /* 4 x u64 little-endian, exclusive */
    const uint64_t lo = j * 128, hi = lo + 128 < N ? lo + 128 : N;
    for (uint64_t i = lo; i < hi; ++i) {
      const uint32_t p = sa[i];
      uint32_t code;
      if (p == 0) {
        code = 0; /* terminator packed as A (index.py:83-84) */
        srow = i;
      } else {
        code = codes[p - 1];
        totals[code]++;
      }
      base[code]++;
      r[32 + ((i - lo) >> 2)] |= (uint8_t)(code << (((i - lo) & 3) << 1));
    }
  }
  if (srow == (uint64_t)-1) return -1;
  c[0] = 0;
  for (int s = 0; s < 4; ++s) c[s + 1] = c[s] + totals[s];
  *sentinel_row = srow;
  for (uint64_t i = 0, q = 0; i < N; i += 32, ++q) samples[q] = sa[i];
  return 0;
}
