// uf_kernels.cu — union-find batch kernels and the compile-time dispatch
// over the 32-configuration matrix of dset.py:60-76.
//
// union_rows: the shared shape of k-out sampling (sampling.py:61-86),
// HB phase 2 (sampling.py:110-116) and the union-find finish
// (driver.py:333-348).  Work decomposition: a warp owns 32 consecutive
// rows; rows of at most kSmall entries are walked by their own lane (the
// paper's edge-serialization "ER": all edges of a vertex are unioned by one
// thread), larger rows are walked by the whole warp, one
// row at a time (warp-cooperative hub handling).
#include <climits>
#include <cstdlib>

#include "internal.h"
#include "uf.cuh"

namespace gc {

constexpr int kSmall = 32;
constexpr int kRowBlock = 512;  // measured: 512 -> 0.3505 ms, 256 -> 0.3522, 1024 -> 0.3549 (k-out s24)

template <class R>
__global__ void __launch_bounds__(kRowBlock)
k_union_rows(UFState s, const int64_t* __restrict__ off, const int32_t* __restrict__ tgt,
             const int32_t* __restrict__ list, const unsigned long long* count_dev,
             int64_t count_host, int32_t take_max, int32_t lower_only,
             unsigned long long* insp, int64_t row_base, unsigned long long* stamps, unsigned stamp_mask) {
  entry_stamp(stamps, stamp_mask);
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (int64_t(blockIdx.x) * kRowBlock + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * kRowBlock) >> 5;
  int64_t count = count_host;
  if (count_dev) {
    int64_t c = int64_t(*count_dev);
    count = c < count ? c : count;
  }
  unsigned long long my_insp = 0;
  const uint64_t pol = evict_first_policy();
  for (int64_t base = warp0 * 32; base < count; base += nwarps * 32) {
    const int64_t i = base + lane;
    int32_t u = -1;
    int64_t b = 0;
    int32_t take = 0;
    if (i < count) {
      u = list ? ldg32(list + i) : int32_t(row_base + i);
      // offsets stream through (no L1 allocation, L2 evict-first); targets
      // keep the default L1 path, which measured faster for the
      // neighbouring-row reuse within a warp
      b = ld_stream64(off + u, pol);
      const int64_t e = ld_stream64(off + u + 1, pol);
      const int64_t d = e - b;
      take = int32_t(d < take_max ? d : take_max);
      my_insp += take;
    }
    const bool big = take > kSmall;
    if (!big) {
      // the first two targets are fetched together (one DRAM round trip for
      // k-out's default k = 2); later ones on demand
      const int32_t f0 = take > 0 ? ldg32(tgt + b) : 0;
      const int32_t f1 = take > 1 ? ldg32(tgt + b + 1) : 0;
      for (int32_t j = 0; j < take; ++j) {
        const int32_t t = j == 0 ? f0 : j == 1 ? f1 : ldg32(tgt + b + j);
        if (lower_only && t >= u) break;
        R::unite(s, u, t);
      }
    }
    unsigned mask = __ballot_sync(0xffffffffu, big);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const int32_t uu = __shfl_sync(0xffffffffu, u, src);
      const int64_t bb = __shfl_sync(0xffffffffu, b, src);
      const int32_t tk = __shfl_sync(0xffffffffu, take, src);
      for (int32_t j = lane; j < tk; j += 32) {
        const int32_t t = ldg32(tgt + bb + j);
        if (lower_only && t >= uu) break;
        R::unite(s, uu, t);
      }
    }
  }
  if (insp) block_add<kRowBlock>(insp, my_insp);
}

// Edge-parallel form of the all-active lower-only finish for graphs with
// fewer rows than resident threads (RMAT s16: 65k rows on 303k thread slots,
// each lane walking a whole row): one thread per CSR entry, its row by a
// binary search over the (cached) offsets; entry (u, t) is unioned when t < u
// — the same edge set as the row form.
template <class R>
__global__ void __launch_bounds__(256)
k_union_csr_edges(UFState s, const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, int32_t n,
                  int64_t m, unsigned long long* stamps, unsigned stamp_mask) {
  entry_stamp(stamps, stamp_mask);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m; j += stride) {
    const int32_t t = ldg32(tgt + j);
    int32_t lo = 0, hi = n - 1;  // last row with off[row] <= j
    while (lo < hi) {
      const int32_t mid = (lo + hi + 1) >> 1;
      if (__ldg(off + mid) <= j) lo = mid;
      else hi = mid - 1;
    }
    if (t < lo) R::unite(s, lo, t);
  }
}

template <class R, bool GIANT>
__global__ void __launch_bounds__(256)
k_union_coo(UFState s, const int32_t* __restrict__ us, const int32_t* __restrict__ vs, int64_t k,
            const uint8_t* __restrict__ skip, int32_t sentinel, unsigned int* bad,
            const unsigned long long* kdev, GiantPass alt) {
  // giant filter (GIANT, incremental handles of the non-async rules): as in
  // the lock-step async kernel, *kdev is the compaction's survivor count
  // (endpoints carry bit 31 = "giant bit set") or ~0 (the caller's batch);
  // these rules do not expose the union's root, so an endpoint is marked
  // only when the other one already carried its bit (the marks spread from
  // the anchor along the inserted edges)
  bool flags = false;
  if (GIANT && kdev) {
    const unsigned long long c = *kdev;
    if (c == ~0ull) {
      us = alt.us;
      vs = alt.vs;
      skip = alt.skip;
      k = alt.k;
    } else {
      k = min(k, int64_t(c));
      flags = true;
    }
  }
  const int32_t anc = GIANT && s.gbits ? ld_acq(s.ganchor) : -1;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < k; i += stride) {
    if (skip && skip[i]) continue;
    int32_t u = ldg32(us + i), v = ldg32(vs + i);
    unsigned need = 0;  // bit 0 / 1: u / v lacks its giant bit
    if (GIANT && flags) {
      need = (u < 0 ? 0u : 1u) | (v < 0 ? 0u : 2u);
      u &= 0x7fffffff;
      v &= 0x7fffffff;
    }
    if (bad && (uint32_t(u) >= uint32_t(s.n) || uint32_t(v) >= uint32_t(s.n))) {
      atomicOr(bad, 1u);  // malformed pair: never touches the parent array
      continue;
    }
    if (GIANT && anc >= 0 && !flags) {
      const uint64_t bpol = bits_policy(s.gkeep);
      const bool bu = gbit(ld_bits(s.gbits + (u >> 5), bpol), u), bv = gbit(ld_bits(s.gbits + (v >> 5), bpol), v);
      if (bu && bv) continue;  // both connected to the anchor already
      need = (bu ? 0u : 1u) | (bv ? 0u : 2u);
    }
    if (sentinel >= 0) {
      // ensure_init (driver.py:620-625) fused into the insert: every parent
      // a union reads is either one of its own endpoints (initialised right
      // here) or an ancestor, which was a root — hence initialised — when it
      // was linked.  The launcher turns L1-cached reads off for this mode.
      // Both endpoint reads are issued together and handed to the union as
      // its first parent reads (a CAS result is a held value too).
      int32_t pu = ld_acq(s.P + u);
      int32_t pv = ld_acq(s.P + v);
      if (pu == sentinel) {
        const int32_t o = atomicCAS(s.P + u, sentinel, u);
        pu = o == sentinel ? u : o;
      }
      if (pv == sentinel) {
        const int32_t o = atomicCAS(s.P + v, sentinel, v);
        pv = o == sentinel ? v : o;
      }
      R::unite_known(s, u, v, pu, pv);
      if (GIANT && anc >= 0) {
        const uint64_t bpol = bits_policy(s.gkeep);
        if (need == 1u) red_or_bits(s.gbits + (u >> 5), 1u << (u & 31), bpol);
        else if (need == 2u) red_or_bits(s.gbits + (v >> 5), 1u << (v & 31), bpol);
      }
      continue;
    }
    R::unite(s, u, v);
  }
}

// Async union (dset.py:222-234) over a COO batch with K unions per thread
// walked in lock step.  One union is a chain of dependent parent reads (the
// endpoint slots are random DRAM reads once the parent array outgrows L2;
// config 4's is 268 MB), so a thread that owns one union keeps one read in
// flight and the batch is latency-bound (ncu, k_union_coo at RMAT s26: DRAM
// 8.6%, IPC 0.58).  Here each step issues the next read of all 2K find chains
// of the thread together, then consumes them.
//
// A find chain is the hop sequence x -> P[x] -> ...; the compression writes
// of split / halve (dset.py:126-147) fall out of the hop sequence: split
// swings P[prev] from x to P[x] at every hop, halving at every other hop.
// Their CAS results are never consumed (a failed compression CAS is dropped,
// as in the reference) and the walk continues from the value it read — an
// ancestor either way, so the root found is the same.  A link is
// CAS(P[hi], hi, lo) on the two roots; a failed link resumes the hi chain
// from the value the CAS saw (hi's new parent) and the lo chain from lo.
// GIANT = false compiles the giant-filter machinery out (batches without a
// filter: static union_edge_list, sharded merges, GC_INCR_GIANT=0)
template <class R, int K, bool WEAK, bool GIANT>
// min resident blocks (registers vs occupancy), measured on config 4's
// stream: unfiltered 5 (34 registers; 8 -> 32 registers was 2% faster there
// but spills the filter form); giant-filter form 6 (40 registers, 4 bytes of
// spill) 13.2 ms vs 13.4 at 5 and 14.0 at 8 (profiles/r3f)
#ifndef GC_MLP_MINB
#define GC_MLP_MINB 5
#endif
#ifndef GC_MLP_MINB_G
#define GC_MLP_MINB_G 6
#endif
__global__ void __launch_bounds__(256, K <= 2 ? (GIANT ? GC_MLP_MINB_G : GC_MLP_MINB) : 1)
k_union_coo_async_mlp(UFState s, const int32_t* __restrict__ us, const int32_t* __restrict__ vs, int64_t k,
                      const uint8_t* __restrict__ skip, int32_t sentinel, unsigned int* bad,
                      const unsigned long long* kdev, GiantPass alt, bool lazy_self) {
  static_assert(R::kUnion == GC_FINISH_ASYNC, "lock-step form of the async rule");
  // giant filter: *kdev = survivors of the compaction (their endpoints
  // carry bit 31 = "giant bit already set"), or ~0 when the compaction
  // passed the batch through (the caller's arrays, no flags)
  bool flags = false;
  if (GIANT && kdev) {
    const unsigned long long c = *kdev;
    if (c == ~0ull) {
      us = alt.us;
      vs = alt.vs;
      skip = alt.skip;
      k = alt.k;
    } else {
      k = min(k, int64_t(c));
      flags = true;
    }
  }
  constexpr int F = R::kFind;
  int32_t* P = s.P;
  // L1-cacheable reads (static batches) only for the first hops: after that
  // every read goes to L2, so a stale line cannot stall a retry loop
  int it = 0;
  auto ld = [&](const int32_t* p) { return (WEAK && it < 8) ? ld_weak(p) : ld_acq(p); };
  const int32_t anc = GIANT && s.gbits ? ld_acq(s.ganchor) : -1;
  const uint64_t bpol = bits_policy(s.gkeep);
  const int64_t span = int64_t(blockDim.x) * K;
  for (int64_t base = int64_t(blockIdx.x) * span; base < k; base += int64_t(gridDim.x) * span) {
    int32_t eu[K], ev[K];     // endpoints (forest records)
    int32_t x[K][2];          // chain position
    int32_t px[K][2];         // P[x] once read (valid when have bit set)
    int32_t pv[K][2];         // previous node (split / halve writes), -1 = none
    unsigned have = 0;        // bit 2j+c: px[j][c] holds P[x[j][c]]
    unsigned live = 0;        // bit 2j+c: chain still walking
    unsigned slot = 0;        // bit j: union j unfinished
    unsigned gneed = 0;       // giant filter: bit 2j+c = endpoint c of union j lacks its bit
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int64_t i = base + int64_t(j) * blockDim.x + threadIdx.x;
      eu[j] = ev[j] = 0;
      if (i < k && !(skip && skip[i])) {
        eu[j] = ldg32(us + i);
        ev[j] = ldg32(vs + i);
        if (flags) {
          // compacted batch: bit 31 = the endpoint's giant bit is already set
          gneed |= (eu[j] < 0 ? 0u : 1u) << (2 * j) | (ev[j] < 0 ? 0u : 2u) << (2 * j);
          eu[j] &= 0x7fffffff;
          ev[j] &= 0x7fffffff;
        }
        if (bad && (uint32_t(eu[j]) >= uint32_t(s.n) || uint32_t(ev[j]) >= uint32_t(s.n))) {
          atomicOr(bad, 1u);  // malformed pair: never touches the parent array
        } else {
          slot |= 1u << j;
        }
      }
      x[j][0] = eu[j];
      x[j][1] = ev[j];
      pv[j][0] = pv[j][1] = -1;
      px[j][0] = px[j][1] = 0;
    }
    // giant filter (the batch was compacted by k_giant_compact): a union
    // that ends at the anchor root marks both endpoints as connected to it
    auto mark = [&](int j, int32_t root) {
      // connected to the anchor once the union is done: its root is the
      // anchor, or one endpoint already carried its bit
      if (root != anc && (gneed >> (2 * j) & 3u) == 3u) return;
      if (gneed >> (2 * j) & 1u) red_or_bits(s.gbits + (eu[j] >> 5), 1u << (eu[j] & 31), bpol);
      if (gneed >> (2 * j) & 2u) red_or_bits(s.gbits + (ev[j] >> 5), 1u << (ev[j] & 31), bpol);
    };
    // passed-through batch: the endpoints' bits are not probed (reading them
    // beside the first parent reads measured 0.3 ms slower over config 4's
    // stream than marking blind); a union that ends at the anchor root sets
    // both (red.or is idempotent)
    if (anc >= 0 && !flags) {
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (slot >> j & 1u) gneed |= 3u << (2 * j);
    }
    // endpoint reads, all issued together; lazy init (driver.py:620-625)
    // of the slots still holding the sentinel
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (slot >> j & 1u) {
        px[j][0] = ld(P + x[j][0]);
        px[j][1] = ld(P + x[j][1]);
      }
    // lazy init (driver.py:620-625) without a returning CAS per endpoint: an
    // uninitialised slot (the sentinel) reads as its own root; the link CAS
    // expects the value actually stored (sentinel or the id), and whoever
    // links under an uninitialised root initialises it with a
    // fire-and-forget CAS — every touched vertex ends initialised, as the
    // reference's ensure_init leaves it, without two dependent atomics per
    // insert (early batches: every endpoint is fresh)
    unsigned sent = 0;  // bit 2j+c: x[j][c]'s slot read as the sentinel
    if (sentinel >= 0 && !lazy_self) {
      // A/B form: claim every fresh endpoint with a returning CAS first
#pragma unroll
      for (int j = 0; j < K; ++j)
#pragma unroll
        for (int c = 0; c < 2; ++c)
          if ((slot >> j & 1u) && px[j][c] == sentinel) {
            const int32_t o = atomicCAS(P + x[j][c], sentinel, x[j][c]);
            px[j][c] = o == sentinel ? x[j][c] : o;
          }
    } else if (sentinel >= 0) {
#pragma unroll
      for (int j = 0; j < K; ++j)
#pragma unroll
        for (int c = 0; c < 2; ++c)
          if ((slot >> j & 1u) && px[j][c] == sentinel) {
            px[j][c] = x[j][c];
            sent |= 1u << (2 * j + c);
          }
    }
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (slot >> j & 1u) {
        have |= 3u << (2 * j);
        live |= 3u << (2 * j);
      }
    for (it = 0; slot; ++it) {
      // 1. issue every missing parent read of a walking chain
#pragma unroll
      for (int j = 0; j < K; ++j)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const unsigned b = 1u << (2 * j + c);
          if ((live & b) && !(have & b)) {
            px[j][c] = ld(P + x[j][c]);
            if (sentinel >= 0 && px[j][c] == sentinel) {
              px[j][c] = x[j][c];
              sent |= b;
            } else {
              sent &= ~b;
            }
          }
        }
      have |= live;
      // 2. advance the chains one hop (compression writes fire and forget)
#pragma unroll
      for (int j = 0; j < K; ++j)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const unsigned b = 1u << (2 * j + c);
          if (!(live & b)) continue;
          const int32_t nx = px[j][c];
          if (nx == x[j][c]) {
            live &= ~b;  // x is a root
            continue;
          }
          if constexpr (F == GC_FIND_SPLIT || F == GC_FIND_HALVE) {
            if (pv[j][c] >= 0) atomicCAS(P + pv[j][c], x[j][c], nx);
            pv[j][c] = (F == GC_FIND_HALVE && pv[j][c] >= 0) ? -1 : x[j][c];
          }
          x[j][c] = nx;
          have &= ~b;
          sent &= ~b;
        }
      // 3. link the unions whose two roots are known (all CASes issued first)
      int32_t old[K];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        old[j] = -1;
        if ((slot >> j & 1u) && !(live >> (2 * j) & 3u)) {
          const int32_t ru = x[j][0], rv = x[j][1];
          if (ru == rv) {
            slot &= ~(1u << j);
            // an insert (u, u) of a fresh vertex initialises it
            if (sent >> (2 * j) & 3u) atomicCAS(P + ru, sentinel, ru);
            if (anc >= 0) mark(j, ru);
          } else {
            const int32_t hi = ru > rv ? ru : rv, lo = ru > rv ? rv : ru;
            const bool hs = (sent >> (2 * j + (ru > rv ? 0 : 1))) & 1u;
            old[j] = atomicCAS(P + hi, hs ? sentinel : hi, lo);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (old[j] < 0) continue;
        const int32_t ru = x[j][0], rv = x[j][1];
        const int32_t hi = ru > rv ? ru : rv, lo = ru > rv ? rv : ru;
        const unsigned bh = 1u << (2 * j + (ru > rv ? 0 : 1)), bl = 1u << (2 * j + (ru > rv ? 1 : 0));
        const bool hs = sent & bh;
        if (old[j] == (hs ? sentinel : hi)) {
          if (s.lflag) s.lflag[base + int64_t(j) * blockDim.x + threadIdx.x] = 1;
          else record<R::kForest>(s, hi, eu[j], ev[j]);
          // lo may still be uninitialised: it is a root with children now
          if (sent & bl) atomicCAS(P + lo, sentinel, lo);
          slot &= ~(1u << j);
          if (anc >= 0) mark(j, lo);
        } else if (sentinel >= 0 && (old[j] == hi || old[j] == sentinel)) {
          // hi is still a root: only its slot was initialised meanwhile;
          // link again next step with the value now stored
          sent = old[j] == sentinel ? (sent | bh) : (sent & ~bh);
        } else {
          // hi was linked meanwhile: resume both finds from the roots
          // (register selects, no dynamic index into the chain arrays)
          const bool h0 = ru > rv;
          x[j][0] = h0 ? hi : lo;
          x[j][1] = h0 ? lo : hi;
          px[j][0] = old[j];
          px[j][1] = old[j];
          pv[j][0] = pv[j][1] = -1;
          have = (have & ~(3u << (2 * j))) | (1u << (2 * j + (h0 ? 0 : 1)));
          live |= 3u << (2 * j);
          sent &= ~(3u << (2 * j));  // old is a real parent; lo is read again
        }
      }
    }
  }
}

// read-only root chase; an uninitialised slot is its own root (driver.py:556-564)
__device__ __forceinline__ int32_t chase(const int32_t* P, int32_t x, int32_t sentinel) {
  int32_t px = ld_acq(P + x);
  if (px == sentinel) return x;
  while (px != x) {
    x = px;
    px = ld_acq(P + x);
  }
  return x;
}

template <class R>
__global__ void __launch_bounds__(256)
k_incr_racy(UFState s, const int32_t* __restrict__ us, const int32_t* __restrict__ vs, int64_t k,
            const uint8_t* __restrict__ is_query, int32_t sentinel, uint32_t* bits, unsigned int* bad) {
  // a warp owns 32 consecutive ops = one packed result word
  const int lane = threadIdx.x & 31;
  const int64_t words = (k + 31) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < words; w += nwarps) {
    const int64_t i = (w << 5) + lane;
    bool hit = false;
    if (i < k) {
      const int32_t u = us[i], v = vs[i];
      if (bad && (uint32_t(u) >= uint32_t(s.n) || uint32_t(v) >= uint32_t(s.n))) {
        atomicOr(bad, 1u);
      } else if (is_query[i]) {
        hit = chase(s.P, u, sentinel) == chase(s.P, v, sentinel);
      } else {
        atomicCAS(s.P + u, sentinel, u);  // ensure_init (driver.py:620-625)
        atomicCAS(s.P + v, sentinel, v);
        R::unite(s, u, v);
      }
    }
    const uint32_t word = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) bits[w] = word;
  }
}

bool valid_uf(const UFConfig& c) {
  switch (c.unite) {
    case GC_FINISH_ASYNC:
    case GC_FINISH_HOOKS:
    case GC_FINISH_EARLY:
      return c.find >= GC_FIND_NAIVE && c.find <= GC_FIND_COMPRESS && c.splice == GC_SPLICE_NONE;
    case GC_FINISH_REM_LOCK:
    case GC_FINISH_REM_CAS:
      return c.find >= GC_FIND_NAIVE && c.find <= GC_FIND_HALVE &&
             c.splice >= GC_SPLICE_SPLIT_ONE && c.splice <= GC_SPLICE_ATOMIC;
    case GC_FINISH_JTB:
      return (c.find == GC_FIND_NAIVE || c.find == GC_FIND_TWO_TRY) && c.splice == GC_SPLICE_NONE;
    default:
      return false;
  }
}

int num_sms() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    GC_CUDA(cudaGetDevice(&dev));
    GC_CUDA(cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev));
  }
  return cached;
}

// unions per thread of the lock-step async kernel (GC_COO_MLP; 0 selects
// the one-union-per-thread k_union_coo).  Config 4 (54 x 10M inserts into
// RMAT s26), measured: K = 0 / 2 / 4 / 8 -> 17.5 / 16.3 / 18.2 / 24.6 ms —
// the batch is bound by random 32-byte-sector DRAM reads of the 268 MB
// parent array (ncu: 1.5 GB read per 10M batch), not by per-thread latency,
// so more unions per thread only cost occupancy
int coo_mlp() {
  static const int k = [] {
    const char* e = getenv("GC_COO_MLP");
    return e ? atoi(e) : 2;
  }();
  return k;
}

bool giant_keep() {
  static const bool on = [] {
    const char* e = getenv("GC_GIANT_KEEP");
    return !(e && e[0] == '0');
  }();
  return on;
}

namespace {

// Functor-style launchers so one dispatch switch serves both kernels.
struct RowsLaunch {
  const RowUnionArgs& a;
  cudaStream_t st;
  template <class R>
  void go() const {
    UFState s{a.P, a.H, a.L, a.R, a.fu, a.fv, a.n, a.lu, a.lv, a.lcount};
    s.fpair = a.fpair;
    if (a.all_edges >= 0 && !a.list && a.lower_only && a.count_host == a.n &&
        a.count_host < int64_t(num_sms()) * 2048) {
      if (a.all_edges == 0) return;
      int64_t blocks = (a.all_edges + 255) / 256;
      const int64_t cap = int64_t(num_sms()) * 8 * 16;
      if (blocks > cap) blocks = cap;
      const unsigned sm = a.stamps ? take_stamps() : 0u;
      (k_union_csr_edges<R><<<int(blocks), 256, 0, st>>>(s, a.off, a.tgt, a.n, a.all_edges, a.stamps, sm),
       ::gc::count_launch());
      GC_CHECK_LAUNCH();
      return;
    }
    int64_t warps = (a.count_host + 31) / 32;
    int64_t blocks = (warps * 32 + kRowBlock - 1) / kRowBlock;
    // one resident wave, grid-stride over 32-row groups
    const int64_t cap = int64_t(num_sms()) * (2048 / kRowBlock);
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    const unsigned sm = a.stamps ? take_stamps() : 0u;
    (k_union_rows<R><<<int(blocks), kRowBlock, 0, st>>>(s, a.off, a.tgt, a.list, a.count_dev,
                                                        a.count_host, a.take_max, a.lower_only,
                                                        a.insp, a.row_base, a.stamps, sm), ::gc::count_launch());
    GC_CHECK_LAUNCH();
  }
};

// GC_INCR_LAZY=0: incremental inserts claim every fresh endpoint with a
// returning CAS before the union (instead of reading the sentinel as "its
// own root" and initialising linked-under roots fire-and-forget)
bool lazy_self() {
  static const bool on = [] {
    const char* e = getenv("GC_INCR_LAZY");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class R, int K>
void launch_mlp(const UFState& s, const CooUnionArgs& a, cudaStream_t st) {
  int64_t blocks = (a.k + 256 * K - 1) / (256 * K);
  // a compacted batch (giant filter, survivors counted on the device) is
  // walked grid-stride by one resident wave; a full batch takes the wide
  // grid (one wave over a full 10M batch measured 40% slower).  kdev_wave
  // is the host's view of the device's mode (a batch or two stale at worst:
  // either grid is correct for either mode)
  static const int per_sm = [] {
    int b = 0;
    GC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_union_coo_async_mlp<R, K, false, true>, 256, 0));
    return b > 0 ? b : 1;
  }();
  const int64_t cap = int64_t(num_sms()) * (a.kdev && a.kdev_wave ? per_sm : 8 * 16);
  if (blocks > cap) blocks = cap;
  if (s.weak)
    (k_union_coo_async_mlp<R, K, true, false><<<int(blocks), 256, 0, st>>>(s, a.us, a.vs, a.k, a.skip,
                                                                            a.init_sentinel, a.bad, nullptr,
                                                                            a.alt, lazy_self()),
     ::gc::count_launch());
  else if (s.gbits)
    (k_union_coo_async_mlp<R, K, false, true><<<int(blocks), 256, 0, st>>>(s, a.us, a.vs, a.k, a.skip,
                                                                            a.init_sentinel, a.bad, a.kdev, a.alt,
                                                                            lazy_self()),
     ::gc::count_launch());
  else
    (k_union_coo_async_mlp<R, K, false, false><<<int(blocks), 256, 0, st>>>(s, a.us, a.vs, a.k, a.skip,
                                                                             a.init_sentinel, a.bad, nullptr,
                                                                             a.alt, lazy_self()),
     ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

struct CooLaunch {
  const CooUnionArgs& a;
  cudaStream_t st;
  template <class R>
  void go() const {
    if (a.k <= 0) return;
    UFState s{a.P, a.H, a.L, a.R, a.fu, a.fv, a.n, a.lu, a.lv, a.lcount};
    s.weak = a.init_sentinel < 0;
    // the giant filter (incremental handles of the non-JTB rules: roots
    // are component minima)
    if (a.gbits && R::kUnion != GC_FINISH_JTB) {
      s.gbits = a.gbits;
      s.ganchor = a.ganchor;
      s.gkeep = giant_keep();
    }
    s.lflag = a.lflag;
    if constexpr (R::kUnion == GC_FINISH_ASYNC && R::kFind != GC_FIND_COMPRESS) {
      switch (coo_mlp()) {
        case 2: return launch_mlp<R, 2>(s, a, st);
        case 4: return launch_mlp<R, 4>(s, a, st);
        case 8: return launch_mlp<R, 8>(s, a, st);
        default: break;
      }
    }
    int64_t blocks = (a.k + 255) / 256;
    const int64_t cap = int64_t(num_sms()) * 8 * 16;
    if (blocks > cap) blocks = cap;
    if (s.gbits)
      (k_union_coo<R, true><<<int(blocks), 256, 0, st>>>(s, a.us, a.vs, a.k, a.skip, a.init_sentinel, a.bad,
                                                         a.kdev, a.alt), ::gc::count_launch());
    else
      (k_union_coo<R, false><<<int(blocks), 256, 0, st>>>(s, a.us, a.vs, a.k, a.skip, a.init_sentinel, a.bad,
                                                          nullptr, a.alt), ::gc::count_launch());
    GC_CHECK_LAUNCH();
  }
};

struct RacyLaunch {
  const CooUnionArgs& a;
  const uint8_t* is_query;
  int32_t sentinel;
  uint32_t* bits;
  cudaStream_t st;
  template <class R>
  void go() const {
    if (a.k <= 0) return;
    UFState s{a.P, a.H, a.L, a.R, a.fu, a.fv, a.n};
    s.weak = false;  // slots are initialised inside this launch
    int64_t blocks = (a.k + 255) / 256;
    const int64_t cap = int64_t(num_sms()) * 8 * 16;
    if (blocks > cap) blocks = cap;
    (k_incr_racy<R><<<int(blocks), 256, 0, st>>>(s, a.us, a.vs, a.k, is_query, sentinel, bits, a.bad),
     ::gc::count_launch());
    GC_CHECK_LAUNCH();
  }
};

template <int U, int F, int S, class L>
void go_forest(bool forest, const L& l) {
  if (forest) {
    if constexpr (S != GC_SPLICE_ATOMIC) l.template go<Rule<U, F, S, true>>();
    else throw Error(GC_ERR_CONFIG, "atomic splice is not root-based: no forest recording");
  } else {
    l.template go<Rule<U, F, S, false>>();
  }
}

template <int U, class L>
void go_find_nosplice(const UFConfig& c, bool forest, const L& l) {
  switch (c.find) {
    case GC_FIND_NAIVE: return go_forest<U, GC_FIND_NAIVE, GC_SPLICE_NONE>(forest, l);
    case GC_FIND_SPLIT: return go_forest<U, GC_FIND_SPLIT, GC_SPLICE_NONE>(forest, l);
    case GC_FIND_HALVE: return go_forest<U, GC_FIND_HALVE, GC_SPLICE_NONE>(forest, l);
    case GC_FIND_COMPRESS: return go_forest<U, GC_FIND_COMPRESS, GC_SPLICE_NONE>(forest, l);
  }
  throw Error(GC_ERR_CONFIG, "invalid find rule");
}

template <int U, int F, class L>
void go_splice(const UFConfig& c, bool forest, const L& l) {
  switch (c.splice) {
    case GC_SPLICE_SPLIT_ONE: return go_forest<U, F, GC_SPLICE_SPLIT_ONE>(forest, l);
    case GC_SPLICE_HALVE_ONE: return go_forest<U, F, GC_SPLICE_HALVE_ONE>(forest, l);
    case GC_SPLICE_ATOMIC: return go_forest<U, F, GC_SPLICE_ATOMIC>(forest, l);
  }
  throw Error(GC_ERR_CONFIG, "invalid splice rule");
}

template <int U, class L>
void go_rem(const UFConfig& c, bool forest, const L& l) {
  switch (c.find) {
    case GC_FIND_NAIVE: return go_splice<U, GC_FIND_NAIVE>(c, forest, l);
    case GC_FIND_SPLIT: return go_splice<U, GC_FIND_SPLIT>(c, forest, l);
    case GC_FIND_HALVE: return go_splice<U, GC_FIND_HALVE>(c, forest, l);
  }
  throw Error(GC_ERR_CONFIG, "invalid find rule for rem");
}

template <class L>
void dispatch(const UFConfig& c, bool forest, const L& l) {
  if (!valid_uf(c)) throw Error(GC_ERR_CONFIG, "unsupported union-find combination");
  switch (c.unite) {
    case GC_FINISH_ASYNC: return go_find_nosplice<GC_FINISH_ASYNC>(c, forest, l);
    case GC_FINISH_HOOKS: return go_find_nosplice<GC_FINISH_HOOKS>(c, forest, l);
    case GC_FINISH_EARLY: return go_find_nosplice<GC_FINISH_EARLY>(c, forest, l);
    case GC_FINISH_REM_LOCK: return go_rem<GC_FINISH_REM_LOCK>(c, forest, l);
    case GC_FINISH_REM_CAS: return go_rem<GC_FINISH_REM_CAS>(c, forest, l);
    case GC_FINISH_JTB:
      if (c.find == GC_FIND_NAIVE) return go_forest<GC_FINISH_JTB, GC_FIND_NAIVE, GC_SPLICE_NONE>(forest, l);
      return go_forest<GC_FINISH_JTB, GC_FIND_TWO_TRY, GC_SPLICE_NONE>(forest, l);
  }
}

}  // namespace

void launch_union_rows(const UFConfig& cfg, bool forest, const RowUnionArgs& a, cudaStream_t st) {
  if (a.count_host <= 0) return;
  dispatch(cfg, forest || a.lu != nullptr, RowsLaunch{a, st});
}

void launch_union_coo(const UFConfig& cfg, bool forest, const CooUnionArgs& a, cudaStream_t st) {
  dispatch(cfg, forest || a.lu != nullptr, CooLaunch{a, st});
}

void launch_incr_racy(const UFConfig& cfg, const CooUnionArgs& a, const uint8_t* is_query,
                      int32_t sentinel, uint32_t* bits, cudaStream_t st) {
  dispatch(cfg, false, RacyLaunch{a, is_query, sentinel, bits, st});
}

}  // namespace gc
