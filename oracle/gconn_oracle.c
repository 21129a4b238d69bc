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
 * Pipeline port (the CPU baseline arm of bench.py / bench_configs.py).   *
 * driver.py:454-536 `_pipeline` / `spanning_forest` and driver.py:567-   *
 * 725 `incremental` restated over the dset.py union / find / splice      *
 * menu, the samplers of sampling.py (none / k-out FIRST_K / BFS) and the *
 * Jacobi round finishes of minbased.py (SV, the Liu-Tarjan family),      *
 * multi-threaded with OpenMP; CAS = __atomic compare-exchange (the       *
 * reference's striped-lock CAS, parallel.py:17-36), np.minimum.at = an   *
 * atomic-min loop.  Every phase reads the snapshot the reference reads   *
 * (e.g. the active set is taken before the finish starts linking,        *
 * driver.py:473), so counters and labels are deterministic.              *
 * ===================================================================== */
enum { OR_ASYNC = 0, OR_REM_CAS = 4, OR_SV = 6, OR_LT = 7 };
enum { OR_NAIVE = 0, OR_SPLIT = 1, OR_HALVE = 2, OR_COMPRESS = 3 };
enum { OR_SPLIT_ONE = 1, OR_HALVE_ONE = 2, OR_SPLICE = 3 };
enum { OR_S_NONE = 0, OR_S_KOUT = 1, OR_S_BFS = 3 };

static inline int32_t ld(int32_t* p) { return __atomic_load_n(p, __ATOMIC_RELAXED); }
static inline void st(int32_t* p, int32_t v) { __atomic_store_n(p, v, __ATOMIC_RELAXED); }
static inline int casw(int32_t* p, int32_t e, int32_t d) {
  return __atomic_compare_exchange_n(p, &e, d, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED);
}
/* np.minimum.at (minbased.py) as an atomic min */
static inline void amin(int32_t* p, int32_t v) {
  int32_t cur = ld(p);
  while (v < cur && !__atomic_compare_exchange_n(p, &cur, v, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
  }
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

/* forest slot r <- (u, v) when root r is hooked (dset.py:391-393) */
static inline void rec(int32_t* fu, int32_t* fv, int32_t r, int32_t u, int32_t v) {
  if (fu) { fu[r] = u; fv[r] = v; }
}

/* dset.py:222-234 */
static void or_union_async(int find, int32_t u, int32_t v, int32_t* P, int32_t* fu, int32_t* fv) {
  int32_t pu = or_find(find, u, P), pv = or_find(find, v, P);
  while (pu != pv) {
    if (pu < pv) { int32_t t = pu; pu = pv; pv = t; }
    if (ld(P + pu) == pu && casw(P + pu, pu, pv)) { rec(fu, fv, pu, u, v); return; }
    pu = or_find(find, u, P);
    pv = or_find(find, v, P);
  }
}

/* dset.py:303-316 with the splices of dset.py:180-207 */
static void or_union_rem(int find, int splice, int32_t u, int32_t v, int32_t* P, int32_t* fu,
                         int32_t* fv) {
  int32_t ru = u, rv = v;
  for (;;) {
    int32_t pru = ld(P + ru), prv = ld(P + rv);
    if (pru == prv) return;
    if (pru < prv) { int32_t t = ru; ru = rv; rv = t; t = pru; pru = prv; prv = t; }
    if (ru == pru && casw(P + ru, ru, prv)) {
      rec(fu, fv, ru, u, v);
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

static inline void or_unite(int uni, int find, int splice, int32_t u, int32_t v, int32_t* P,
                            int32_t* fu, int32_t* fv) {
  if (uni == OR_REM_CAS) or_union_rem(find, splice, u, v, P, fu, fv);
  else or_union_async(find, u, v, P, fu, fv);
}

static double wall(void) {
#ifdef _OPENMP
  return omp_get_wtime();
#else
  return 0.0;
#endif
}

/* full pointer jump to the fixpoint (sampling.py:38-47 compress_all,
 * minbased.py:87-92 _full_shortcut): order-free, every value is an ancestor */
static void full_shortcut(int32_t* L, int64_t n) {
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) {
    int32_t r = ld(L + v);
    while (ld(L + r) != r) r = ld(L + r);
    st(L + v, r);
  }
}

/* most_frequent_label (sampling.py:29-35): exact histogram, ties low */
static int32_t mode_label(const int32_t* L, int64_t n, int64_t* count) {
  int32_t* cnt = calloc((size_t)(n ? n : 1), sizeof(int32_t));
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) __atomic_fetch_add(cnt + L[v], 1, __ATOMIC_RELAXED);
  int64_t best = -1;
  int32_t lmax = 0;
  for (int64_t v = 0; v < n; ++v)
    if (cnt[v] > best) { best = cnt[v]; lmax = (int32_t)v; }
  free(cnt);
  *count = n ? best : 0;
  return lmax;
}

/* ------------------------------------------------------------ BFS sample
 * sampling.py:120-172: level-synchronous BFS from `s`; a vertex reached at a
 * level takes as parent its smallest frontier neighbour (the reference's
 * frontier is ascending and the first discoverer wins); the reached set takes
 * the minimum id.  Forest: the discovery tree re-rooted at that minimum.
 * Returns the inspections (sum of frontier degrees per level). */
static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return x < y ? -1 : x > y;
}

static int64_t or_bfs(int64_t n, const int64_t* off, const int32_t* tgt, int64_t s, int32_t* labels,
                      int32_t* fu, int32_t* fv, int64_t* levels_out) {
  int32_t* parent = malloc(sizeof(int32_t) * (size_t)n);
  uint8_t* seen = calloc((size_t)n, 1);
  int32_t* front = malloc(sizeof(int32_t) * (size_t)n);
  int32_t* next = malloc(sizeof(int32_t) * (size_t)n);
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) parent[v] = INT32_MAX;
  int64_t nf = 1, insp = 0, levels = 0, mn = s;
  front[0] = (int32_t)s;
  seen[s] = 1;
  parent[s] = -1;
  while (nf) {
    int64_t tot = 0, nn = 0;
    /* claim: parent[t] = min frontier neighbour among this level's finders */
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : tot)
    for (int64_t i = 0; i < nf; ++i) {
      const int32_t u = front[i];
      tot += off[u + 1] - off[u];
      for (int64_t j = off[u]; j < off[u + 1]; ++j) {
        const int32_t t = tgt[j];
        if (__atomic_load_n(seen + t, __ATOMIC_RELAXED)) continue;
        int32_t cur = ld(parent + t);
        if (cur == INT32_MAX && casw(parent + t, INT32_MAX, u)) {
          int64_t slot = __atomic_fetch_add(&nn, 1, __ATOMIC_RELAXED);
          next[slot] = t;
        } else {
          amin(parent + t, u);
        }
      }
    }
    insp += tot;
    if (tot == 0) break;
    /* the next frontier in ascending id order, marked seen */
    qsort(next, (size_t)nn, sizeof(int32_t), cmp_i32);
#pragma omp parallel for schedule(static) reduction(min : mn)
    for (int64_t i = 0; i < nn; ++i) {
      seen[next[i]] = 1;
      if (next[i] < mn) mn = next[i];
    }
    int32_t* t = front; front = next; next = t;
    nf = nn;
    ++levels;
  }
  /* labels: the reached set takes its minimum (sampling.py:158-160) */
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v)
    if (seen[v]) labels[v] = (int32_t)mn;
  if (fu) {
    /* re-root at the minimum (sampling.py:161-171) */
    int32_t cur = (int32_t)mn, prev = -1;
    while (cur != -1) {
      int32_t nx = parent[cur];
      parent[cur] = prev;
      prev = cur;
      cur = nx;
    }
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n; ++r)
      if (seen[r] && r != mn) { fu[r] = parent[r]; fv[r] = (int32_t)r; }
  }
  free(parent); free(seen); free(front); free(next);
  if (levels_out) *levels_out = levels;
  return insp;
}

/* ------------------------------------------------------ round finishes
 * minbased.py:124-155 shiloach_vishkin and :163-243 liu_tarjan (Jacobi
 * rounds over the gathered COO of the active vertices).  Returns rounds;
 * *insp += the working-edge count charged per round. */
typedef struct { int32_t* u; int32_t* v; int64_t len; } coo_t;

static coo_t gather_coo(const int64_t* off, const int32_t* tgt, const int32_t* act, int64_t na) {
  /* driver.py:325-330 _gather_edges: all directed edges of the active rows */
  int64_t* pos = malloc(sizeof(int64_t) * (size_t)(na + 1));
  pos[0] = 0;
  for (int64_t i = 0; i < na; ++i) pos[i + 1] = pos[i] + (off[act[i] + 1] - off[act[i]]);
  coo_t c;
  c.len = pos[na];
  c.u = malloc(sizeof(int32_t) * (size_t)(c.len ? c.len : 1));
  c.v = malloc(sizeof(int32_t) * (size_t)(c.len ? c.len : 1));
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < na; ++i) {
    const int32_t u = act[i];
    int64_t p = pos[i];
    for (int64_t j = off[u]; j < off[u + 1]; ++j, ++p) { c.u[p] = u; c.v[p] = tgt[j]; }
  }
  free(pos);
  return c;
}

static int64_t or_sv(int64_t n, coo_t c, int32_t* L, int64_t* insp) {
  int32_t* prev = malloc(sizeof(int32_t) * (size_t)n);
  memcpy(prev, L, sizeof(int32_t) * (size_t)n);
  int64_t rounds = 0;
  for (;;) {
    ++rounds;
    *insp += c.len;
    int changed = 0;
#pragma omp parallel for schedule(static) reduction(| : changed)
    for (int64_t e = 0; e < c.len; ++e) {
      const int32_t pu = prev[c.u[e]], pv = prev[c.v[e]];
      /* labels[eu] / labels[ev] are read before any write of the round: the
       * snapshot prev equals labels at the round start */
      const int32_t lo = pu < pv ? pu : pv, hi = pu < pv ? pv : pu;
      if (lo != hi && prev[hi] == hi) { amin(L + hi, lo); changed = 1; }
    }
    full_shortcut(L, n);
    memcpy(prev, L, sizeof(int32_t) * (size_t)n);
    if (!changed) break;
  }
  free(prev);
  return rounds;
}

static int64_t or_lt(int64_t n, coo_t c, int32_t* L, int connect, int update, int shortcut, int alter,
                     int64_t* insp) {
  /* working edges start mapped through the labels (minbased.py:176-177) */
  int64_t w = c.len;
  int32_t* wu = malloc(sizeof(int32_t) * (size_t)(w ? w : 1));
  int32_t* wv = malloc(sizeof(int32_t) * (size_t)(w ? w : 1));
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < w; ++e) { wu[e] = L[c.u[e]]; wv[e] = L[c.v[e]]; }
  int32_t* xu = alter ? malloc(sizeof(int32_t) * (size_t)(w ? w : 1)) : NULL;
  int32_t* xv = alter ? malloc(sizeof(int32_t) * (size_t)(w ? w : 1)) : NULL;
  int32_t* start = malloc(sizeof(int32_t) * (size_t)n);
  int32_t* msg = malloc(sizeof(int32_t) * (size_t)n);
  int nt = 1;
#ifdef _OPENMP
  nt = omp_get_max_threads();
#endif
  int64_t* cnt = malloc(sizeof(int64_t) * (size_t)(nt + 1));
  int64_t rounds = 0;
  for (;;) {
    ++rounds;
    *insp += w;
    memcpy(start, L, sizeof(int32_t) * (size_t)n);
    memcpy(msg, L, sizeof(int32_t) * (size_t)n);
    /* connect (minbased.py:188-208) */
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < w; ++e) {
      const int32_t a = wu[e], b = wv[e];
      if (connect == 0) { amin(msg + a, b); amin(msg + b, a); }
      else {
        const int32_t pa = start[a], pb = start[b];
        amin(msg + pa, pb); amin(msg + pb, pa);
        if (connect == 2) { amin(msg + a, pb); amin(msg + b, pa); }
      }
    }
    /* update (minbased.py:213-219) */
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; ++v)
      if (update == 0 || start[v] == v) L[v] = msg[v];
    /* shortcut (minbased.py:227-230) */
    if (shortcut) full_shortcut(L, n);
    else {
      memcpy(msg, L, sizeof(int32_t) * (size_t)n);
#pragma omp parallel for schedule(static)
      for (int64_t v = 0; v < n; ++v) L[v] = msg[msg[v]];
    }
    /* alter (minbased.py:233-239): rewrite, drop closed edges, keeping
     * the order (a per-thread count, a prefix, then each thread copies its
     * kept entries into the spare buffers) */
    if (alter) {
#pragma omp parallel
      {
        int t = 0, T = 1;
#ifdef _OPENMP
        t = omp_get_thread_num();
        T = omp_get_num_threads();
#endif
        const int64_t lo = w * t / T, hi = w * (t + 1) / T;
        int64_t k = 0;
        for (int64_t e = lo; e < hi; ++e) {
          wu[e] = L[wu[e]];
          wv[e] = L[wv[e]];
          k += wu[e] != wv[e];
        }
        cnt[t + 1] = k;
#pragma omp barrier
#pragma omp single
        {
          cnt[0] = 0;
          for (int i = 1; i <= T; ++i) cnt[i] += cnt[i - 1];
        }
        int64_t p = cnt[t];
        for (int64_t e = lo; e < hi; ++e)
          if (wu[e] != wv[e]) { xu[p] = wu[e]; xv[p] = wv[e]; ++p; }
#pragma omp single
        w = cnt[T];
      }
      int32_t* tu = wu; wu = xu; xu = tu;
      int32_t* tv = wv; wv = xv; xv = tv;
    }
    int same = 1;
#pragma omp parallel for schedule(static) reduction(& : same)
    for (int64_t v = 0; v < n; ++v) same &= L[v] == start[v];
    if (same) break;
  }
  free(wu); free(wv); free(xu); free(xv); free(start); free(msg); free(cnt);
  return rounds;
}

/* ----------------------------------------------------------- pipeline
 * stats: [0] insp_sample [1] insp_finish [2] l_max [3] components
 *        [4] active vertices [5] l_max count [6] rounds [7] BFS levels
 * times: sample / finish / finalize seconds.  fu/fv (nullable): forest
 * slots (-1 = empty), union-find and BFS recording (driver.py:523-536). */
typedef struct {
  int32_t sample, kout_k, finish, find, splice, lt_connect, lt_update, lt_shortcut, lt_alter;
  int32_t pad;
  int64_t bfs_source;
} or_spec;

int or_pipeline(int64_t n, const int64_t* off, const int32_t* tgt, const or_spec* sp, int threads,
                int32_t* P, int32_t* fu, int32_t* fv, int64_t* stats, double* times) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  const int uf = sp->finish == OR_ASYNC || sp->finish == OR_REM_CAS;
  int64_t insp_s = 0, insp_f = 0, rounds = 0, levels = 0, lmax_count = n ? 1 : 0; /* identity labels */
  if (fu) {
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; ++v) { fu[v] = -1; fv[v] = -1; }
  }
  double t0 = wall();
  /* DisjointSets.__init__ (dset.py:359) / identity labels */
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) P[v] = (int32_t)v;
  int32_t lmax = (int32_t)n;
  if (sp->sample == OR_S_KOUT) {
    /* kout_sample FIRST_K (sampling.py:61-86) on the finish's own rule, or
     * the async + halve fallback for round finishes (driver.py:96) */
    const int su = uf ? sp->finish : OR_ASYNC, sf = uf ? sp->find : OR_HALVE, ss = uf ? sp->splice : 0;
    const int64_t k = sp->kout_k;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : insp_s)
    for (int64_t v = 0; v < n; ++v) {
      int64_t b = off[v], d = off[v + 1] - b, take = d < k ? d : k;
      insp_s += take;
      for (int64_t j = 0; j < take; ++j) or_unite(su, sf, ss, (int32_t)v, tgt[b + j], P, fu, fv);
    }
    full_shortcut(P, n);
    lmax = mode_label(P, n, &lmax_count);
  } else if (sp->sample == OR_S_BFS) {
    if (n && off[n]) insp_s = or_bfs(n, off, tgt, sp->bfs_source, P, fu, fv, &levels);
    lmax = mode_label(P, n, &lmax_count);
  }
  double t1 = wall();
  /* the active set, snapshotted before the finish links anything
   * (driver.py:473 np.flatnonzero(post_sample != l_max)) */
  int32_t* act = malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int64_t na = 0;
  for (int64_t u = 0; u < n; ++u)
    if (P[u] != lmax) act[na++] = (int32_t)u;
  if (uf) {
    /* _union_finish (driver.py:333-348) */
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : insp_f)
    for (int64_t i = 0; i < na; ++i) {
      const int32_t u = act[i];
      insp_f += off[u + 1] - off[u];
      for (int64_t j = off[u]; j < off[u + 1]; ++j)
        or_unite(sp->finish, sp->find, sp->splice, u, tgt[j], P, fu, fv);
    }
  } else if (na) {
    /* _rounds_finish (driver.py:351-375, skipped when nothing is active,
     * driver.py:475): gather once (charged once), then the rounds charge
     * their working set per round */
    coo_t c = gather_coo(off, tgt, act, na);
    insp_f += c.len;
    if (sp->finish == OR_SV) rounds = or_sv(n, c, P, &insp_f);
    else rounds = or_lt(n, c, P, sp->lt_connect, sp->lt_update, sp->lt_shortcut, sp->lt_alter, &insp_f);
    free(c.u); free(c.v);
  }
  free(act);
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
  stats[0] = insp_s; stats[1] = insp_f; stats[2] = lmax; stats[3] = comps; stats[4] = na;
  stats[5] = lmax_count; stats[6] = rounds; stats[7] = levels;
  times[0] = t1 - t0; times[1] = t2 - t1; times[2] = t3 - t2;
  return 0;
}

/* the union-find static pipeline (bench.py reference arm) */
int or_static_uf(int64_t n, const int64_t* off, const int32_t* tgt, int sample, int k, int uni,
                 int find, int splice, int threads, int32_t* P, int64_t* stats, double* times) {
  or_spec sp;
  memset(&sp, 0, sizeof(sp));
  sp.sample = sample;
  sp.kout_k = k;
  sp.finish = uni;
  sp.find = find;
  sp.splice = splice;
  return or_pipeline(n, off, tgt, &sp, threads, P, NULL, NULL, stats, times);
}

/* ------------------------------------------------------ incremental
 * One insert-only batch (driver.py:620-649): ensure_init by CAS(sentinel ->
 * v) for both endpoints, then the union rule, all pairs in parallel.  P has
 * cap slots with the sentinel `cap` for uninitialised ones. */
int or_incr_insert(int64_t cap, int32_t* P, const int32_t* us, const int32_t* vs, int64_t len, int uni,
                   int find, int splice, int threads, double* seconds) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  const int32_t sentinel = (int32_t)cap;
  double t0 = wall();
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < len; ++i) {
    const int32_t u = us[i], v = vs[i];
    casw(P + u, sentinel, u);
    casw(P + v, sentinel, v);
    or_unite(uni, find, splice, u, v, P, NULL, NULL);
  }
  *seconds = wall() - t0;
  return 0;
}

int or_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
