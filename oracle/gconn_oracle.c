/*
 * gconn_oracle.c — CPU restatement of the reference connectivity path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker (and the CPU baseline
 * arm of bench.py); the product (paper_2008_11839_b200 / libgconn.so) never
 * links, loads or calls it.  It restates, in plain C, the algorithms of the
 * reference package connlab (/root/reference/pkg/src/connlab), each function
 * citing the reference lines it follows.  Parity of this restatement is
 * pinned against fixtures produced by the reference itself
 * (tests/golden/make_golden.py -> tests/golden/*.json, *.npz) by the CPU test
 * suite (tests/test_oracle.py).
 *
 * Build: oracle/build.sh  ->  oracle/build/libgconn_oracle.so
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------ PCG64
 * numpy's default_rng bit generator (the reference's RNG for gen_rmat,
 * graphs.py:231, and random_edge_pairs, tests/helpers.py:33-37). */
static const u128 PCG_MUL = (((u128)0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull;

typedef struct { u128 s, inc; } pcg_t;

static inline uint64_t pcg_next(pcg_t* p) {
  p->s = p->s * PCG_MUL + p->inc;
  uint64_t hi = (uint64_t)(p->s >> 64), lo = (uint64_t)p->s;
  unsigned rot = (unsigned)(p->s >> 122);
  uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
static inline double pcg_double(pcg_t* p) { return (double)(pcg_next(p) >> 11) * (1.0 / 9007199254740992.0); }

static void pcg_advance(pcg_t* p, uint64_t delta) {
  u128 am = 1, ap = 0, cm = PCG_MUL, cp = p->inc;
  while (delta) {
    if (delta & 1) { am *= cm; ap = ap * cm + cp; }
    cp = (cm + 1) * cp;
    cm *= cm;
    delta >>= 1;
  }
  p->s = am * p->s + ap;
}

/* gen_rmat (graphs.py:210-245).  Level L draws an (m,4) noise block then m
 * quadrant draws; we walk both sub-streams per level.  Volatile temporaries
 * keep every product and sum individually rounded (no FMA contraction). */
int or_gen_rmat(int scale, int64_t m, const double* base, uint64_t s_hi, uint64_t s_lo,
                uint64_t i_hi, uint64_t i_lo, int64_t* src, int64_t* dst) {
  pcg_t g0;
  g0.s = ((u128)s_hi << 64) | s_lo;
  g0.inc = ((u128)i_hi << 64) | i_lo;
  memset(src, 0, sizeof(int64_t) * (size_t)m);
  memset(dst, 0, sizeof(int64_t) * (size_t)m);
  for (int lev = 0; lev < scale; ++lev) {
    const int64_t bit = (int64_t)1 << (scale - 1 - lev);
#pragma omp parallel
    {
      int64_t nt = 1, tid = 0;
#ifdef _OPENMP
      nt = omp_get_num_threads();
      tid = omp_get_thread_num();
#endif
      int64_t lo = m * tid / nt, hi = m * (tid + 1) / nt;
      pcg_t pn = g0, pr = g0;
      pcg_advance(&pn, (uint64_t)(5 * m * lev + 4 * lo));
      pcg_advance(&pr, (uint64_t)(5 * m * lev + 4 * m + lo));
      for (int64_t i = lo; i < hi; ++i) {
        volatile double p[4];
        for (int j = 0; j < 4; ++j) {
          volatile double r = pcg_double(&pn);
          volatile double t = 0.2 * r;
          volatile double nz = 0.9 + t;
          p[j] = base[j] * nz;
        }
        volatile double s01 = p[0] + p[1];
        volatile double s012 = s01 + p[2];
        volatile double sum = s012 + p[3];
        double r = pcg_double(&pr);
        volatile double cut = 0.0;
        int quad = 0;
        for (int j = 0; j < 4; ++j) {
          volatile double pj = p[j] / sum;
          cut = j == 0 ? pj : cut + pj;
          quad += r >= cut;
        }
        if (quad > 3) quad = 3;
        src[i] += bit * (quad >= 2);
        dst[i] += bit * (quad & 1);
      }
    }
  }
  return 0;
}

/* ------------------------------------------------------------- build_csr
 * graphs.py:90-121: symmetrize, drop self-loops, dedupe, sort. */
static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

/* LSD radix sort on 16-bit digits (keys < 2^bits). */
static void radix_sort_u64(uint64_t* a, uint64_t* tmp, int64_t n, int bits) {
  const int D = 16;
  for (int shift = 0; shift < bits; shift += D) {
    int64_t* cnt = calloc((size_t)1 << D, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) cnt[(a[i] >> shift) & 0xFFFF]++;
    int64_t acc = 0;
    for (int64_t d = 0; d < ((int64_t)1 << D); ++d) { int64_t c = cnt[d]; cnt[d] = acc; acc += c; }
    for (int64_t i = 0; i < n; ++i) tmp[cnt[(a[i] >> shift) & 0xFFFF]++] = a[i];
    memcpy(a, tmp, sizeof(uint64_t) * (size_t)n);
    free(cnt);
  }
}

int64_t or_build_csr(int64_t n, const int64_t* src, const int64_t* dst, int64_t k, int64_t* off,
                     int32_t* tgt /* capacity 2k */) {
  int bits = 1;
  while (((int64_t)1 << bits) < n) ++bits;
  uint64_t* keys = malloc(sizeof(uint64_t) * (size_t)(2 * k + 1));
  int64_t c = 0;
  for (int64_t i = 0; i < k; ++i) {
    int64_t u = src[i], v = dst[i];
    if (u < 0 || v < 0 || u >= n || v >= n) { free(keys); return -1 - i; }
    if (u == v) continue;
    keys[c++] = ((uint64_t)u << bits) | (uint64_t)v;
    keys[c++] = ((uint64_t)v << bits) | (uint64_t)u;
  }
  if (c > 4096) {
    uint64_t* tmp = malloc(sizeof(uint64_t) * (size_t)c);
    radix_sort_u64(keys, tmp, c, 2 * bits);
    free(tmp);
  } else {
    qsort(keys, (size_t)c, sizeof(uint64_t), cmp_u64);
  }
  int64_t m = 0;
  for (int64_t i = 0; i < c; ++i)
    if (i == 0 || keys[i] != keys[i - 1]) keys[m++] = keys[i];
  const uint64_t mask = ((uint64_t)1 << bits) - 1;
  int64_t row = 0;
  off[0] = 0;
  for (int64_t j = 0; j < m; ++j) {
    int64_t u = (int64_t)(keys[j] >> bits);
    while (row < u) off[++row] = j;
    tgt[j] = (int32_t)(keys[j] & mask);
  }
  while (row < n) off[++row] = m;
  free(keys);
  return m;
}

/* ------------------------------------------------------------ components
 * validate.py:101-122 oracle_components_unionfind: sequential union-find,
 * smaller root wins, full compression; labels are component minima (the
 * canonical form of oracle_components, validate.py:74-98). */
static int32_t uf_find(int32_t* p, int32_t x) {
  int32_t r = x;
  while (p[r] != r) r = p[r];
  while (p[x] != r) { int32_t nx = p[x]; p[x] = r; x = nx; }
  return r;
}

int64_t or_components(int64_t n, const int64_t* off, const int32_t* tgt, int32_t* labels) {
  for (int64_t v = 0; v < n; ++v) labels[v] = (int32_t)v;
  for (int64_t u = 0; u < n; ++u)
    for (int64_t j = off[u]; j < off[u + 1]; ++j) {
      int32_t t = tgt[j];
      if (t >= u) break; /* rows are sorted: each undirected edge once */
      int32_t ru = uf_find(labels, (int32_t)u), rv = uf_find(labels, t);
      if (ru != rv) { if (ru < rv) { int32_t x = ru; ru = rv; rv = x; } labels[ru] = rv; }
    }
  int64_t comps = 0;
  for (int64_t v = 0; v < n; ++v) { labels[v] = uf_find(labels, (int32_t)v); comps += labels[v] == v; }
  return comps;
}

/* ------------------------------------------------------------ check_forest
 * validate.py:178-244, vectorisable form of the four clauses:
 *   out[0] edges_exist, out[1] acyclic, out[2] count, out[3] components_match
 * (1 = ok).  fu/fv hold slot-indexed edges, -1 = empty.  witness[0..1]
 * receives the first offending edge / vertex. */
void or_check_forest(int64_t n, const int64_t* off, const int32_t* tgt, const int32_t* fu,
                     const int32_t* fv, const int32_t* oracle, int32_t* out, int64_t* witness) {
  out[0] = out[1] = out[2] = out[3] = 1;
  witness[0] = witness[1] = -1;
  int64_t pop = 0;
  for (int64_t r = 0; r < n; ++r) {
    if (fu[r] < 0) continue;
    ++pop;
    int32_t u = fu[r], v = fv[r];
    int64_t lo = off[u], hi = off[u + 1];
    while (lo < hi) { int64_t mid = (lo + hi) / 2; if (tgt[mid] < v) lo = mid + 1; else hi = mid; }
    if ((lo >= off[u + 1] || tgt[lo] != v) && out[0]) { out[0] = 0; witness[0] = r; }
  }
  int32_t* p = malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  for (int64_t v = 0; v < n; ++v) p[v] = (int32_t)v;
  for (int64_t r = 0; r < n; ++r) {
    if (fu[r] < 0) continue;
    int32_t a = uf_find(p, fu[r]), b = uf_find(p, fv[r]);
    if (a == b) { if (out[1]) { out[1] = 0; witness[0] = r; } continue; }
    if (a < b) p[b] = a; else p[a] = b;
  }
  int64_t comps = 0;
  for (int64_t v = 0; v < n; ++v) comps += oracle[v] == v;
  if (pop != n - comps) out[2] = 0;
  for (int64_t v = 0; v < n; ++v) {
    int32_t f = uf_find(p, (int32_t)v);
    /* forest roots are component minima after min-linking: compare directly */
    if (f != oracle[v]) { out[3] = 0; witness[1] = v; break; }
  }
  free(p);
}

/* --------------------------------------------------------- SequentialUF
 * validate.py:125-155 replayed over an op stream with batch barriers
 * (driver.py:695-708): within a batch all inserts apply first, then the
 * queries read.  bits[i] = 1 for connected queries. */
void or_incremental_replay(int64_t cap, const int32_t* us, const int32_t* vs, const uint8_t* isq,
                           int64_t len, int64_t batch, uint8_t* bits, int32_t* labels) {
  int32_t* p = malloc(sizeof(int32_t) * (size_t)(cap ? cap : 1));
  for (int64_t v = 0; v < cap; ++v) p[v] = (int32_t)v;
  for (int64_t b0 = 0; b0 < len; b0 += batch) {
    int64_t b1 = b0 + batch < len ? b0 + batch : len;
    for (int64_t i = b0; i < b1; ++i) {
      if (isq[i]) continue;
      int32_t a = uf_find(p, us[i]), b = uf_find(p, vs[i]);
      if (a != b) { if (a < b) p[b] = a; else p[a] = b; }
    }
    for (int64_t i = b0; i < b1; ++i)
      bits[i] = isq[i] ? (uf_find(p, us[i]) == uf_find(p, vs[i])) : 0;
  }
  for (int64_t v = 0; v < cap; ++v) labels[v] = uf_find(p, (int32_t)v);
  free(p);
}

/* ===================================================================== *
 * Static pipeline port (the CPU baseline arm of bench.py).               *
 * driver.py:454-500 `_pipeline` for union-find finishes with the none /  *
 * k-out (FIRST_K) samplers, over the dset.py union / find / splice menu, *
 * multi-threaded with OpenMP; CAS = __atomic compare-exchange (the       *
 * reference's striped-lock CAS, parallel.py:17-36).                      *
 * ===================================================================== */
enum { OR_ASYNC = 0, OR_REM_CAS = 4 };
enum { OR_NAIVE = 0, OR_SPLIT = 1, OR_HALVE = 2, OR_COMPRESS = 3 };
enum { OR_SPLIT_ONE = 1, OR_HALVE_ONE = 2, OR_SPLICE = 3 };

static inline int32_t ld(int32_t* p) { return __atomic_load_n(p, __ATOMIC_RELAXED); }
static inline int casw(int32_t* p, int32_t e, int32_t d) {
  return __atomic_compare_exchange_n(p, &e, d, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED);
}

/* dset.py:109-147 */
static int32_t or_find(int find, int32_t u, int32_t* P) {
  if (find == OR_NAIVE) {
    int32_t pu;
    while ((pu = ld(P + u)) != u) u = pu;
    return u;
  }
  if (find == OR_COMPRESS) {
    int32_t r = u, pr, j;
    while ((pr = ld(P + r)) != r) r = pr;
    while ((j = ld(P + u)) > r) { casw(P + u, j, r); u = j; }
    return r;
  }
  int32_t v = ld(P + u), w = ld(P + v);
  while (v != w) {
    casw(P + u, v, w);
    u = find == OR_SPLIT ? v : ld(P + u);
    v = ld(P + u);
    w = ld(P + v);
  }
  return v;
}

/* dset.py:222-234 */
static void or_union_async(int find, int32_t u, int32_t v, int32_t* P) {
  int32_t pu = or_find(find, u, P), pv = or_find(find, v, P);
  while (pu != pv) {
    if (pu < pv) { int32_t t = pu; pu = pv; pv = t; }
    if (ld(P + pu) == pu && casw(P + pu, pu, pv)) return;
    pu = or_find(find, u, P);
    pv = or_find(find, v, P);
  }
}

/* dset.py:303-316 with the splices of dset.py:180-207 */
static void or_union_rem(int find, int splice, int32_t u, int32_t v, int32_t* P) {
  int32_t ru = u, rv = v;
  for (;;) {
    int32_t pru = ld(P + ru), prv = ld(P + rv);
    if (pru == prv) return;
    if (pru < prv) { int32_t t = ru; ru = rv; rv = t; t = pru; pru = prv; prv = t; }
    if (ru == pru && casw(P + ru, ru, prv)) {
      if (find != OR_NAIVE) { or_find(find, u, P); or_find(find, v, P); }
      return;
    }
    if (splice == OR_SPLICE) {
      casw(P + ru, pru, prv);
      ru = pru;
    } else {
      int32_t pu = ld(P + ru), w = ld(P + pu);
      if (pu != w) casw(P + ru, pu, w);
      ru = splice == OR_SPLIT_ONE ? pu : w;
    }
  }
}

static inline void or_unite(int uni, int find, int splice, int32_t u, int32_t v, int32_t* P) {
  if (uni == OR_REM_CAS) or_union_rem(find, splice, u, v, P);
  else or_union_async(find, u, v, P);
}

static double wall(void) {
#ifdef _OPENMP
  return omp_get_wtime();
#else
  return 0.0;
#endif
}

/* stats[0] insp_sample, [1] insp_finish, [2] l_max, [3] components,
 * [4] active vertices; times[0..2] sample / finish / finalize seconds. */
int or_static_uf(int64_t n, const int64_t* off, const int32_t* tgt, int sample, int k, int uni,
                 int find, int splice, int threads, int32_t* P, int64_t* stats, double* times) {
  if (threads > 0) {
#ifdef _OPENMP
    omp_set_num_threads(threads);
#endif
  }
  int64_t insp_s = 0, insp_f = 0;
  double t0 = wall();
  /* DisjointSets.__init__ (dset.py:359) */
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) P[v] = (int32_t)v;
  int32_t lmax = (int32_t)n;
  if (sample == 1) {
    /* kout_sample FIRST_K (sampling.py:61-86) */
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : insp_s)
    for (int64_t v = 0; v < n; ++v) {
      int64_t b = off[v], d = off[v + 1] - b, take = d < k ? d : k;
      insp_s += take;
      for (int64_t j = 0; j < take; ++j) or_unite(uni, find, splice, (int32_t)v, tgt[b + j], P);
    }
    /* compress_all (sampling.py:38-47) */
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; ++v) {
      int32_t r = P[v];
      while (P[r] != r) r = P[r];
      P[v] = r;
    }
    /* most_frequent_label (sampling.py:29-35): exact histogram, ties low */
    int32_t* cnt = calloc((size_t)(n ? n : 1), sizeof(int32_t));
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; ++v) __atomic_fetch_add(cnt + P[v], 1, __ATOMIC_RELAXED);
    int64_t best = -1;
    lmax = 0;
    for (int64_t v = 0; v < n; ++v)
      if (cnt[v] > best) { best = cnt[v]; lmax = (int32_t)v; }
    free(cnt);
  }
  double t1 = wall();
  /* _union_finish over the active vertices (driver.py:333-348, :473) */
  int64_t active = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : insp_f, active)
  for (int64_t u = 0; u < n; ++u) {
    if (P[u] == lmax) continue;
    ++active;
    insp_f += off[u + 1] - off[u];
    for (int64_t j = off[u]; j < off[u + 1]; ++j) or_unite(uni, find, splice, (int32_t)u, tgt[j], P);
  }
  double t2 = wall();
  /* label_finalization (driver.py:420-429): roots are component minima */
  int64_t comps = 0;
#pragma omp parallel for schedule(static) reduction(+ : comps)
  for (int64_t v = 0; v < n; ++v) {
    int32_t r = ld(P + v);
    while (ld(P + r) != r) r = ld(P + r);
    P[v] = r;
    comps += r == v;
  }
  double t3 = wall();
  stats[0] = insp_s; stats[1] = insp_f; stats[2] = lmax; stats[3] = comps; stats[4] = active;
  times[0] = t1 - t0; times[1] = t2 - t1; times[2] = t3 - t2;
  return 0;
}

int or_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
