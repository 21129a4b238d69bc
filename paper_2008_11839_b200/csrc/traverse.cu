// traverse.cu — the traversal samplers: BFS (sampling.py:120-172) and the
// new LDD sampler.
//
// Both are frontier expansions whose per-vertex claim is one 64-bit word
//     key[x] = (round << 32) | payload          (~0 = unclaimed)
// resolved with a single atomicMin: the earliest round wins, and among the
// claims of that round the smallest payload wins (BFS: the parent id, LDD:
// the cluster id).  The claimant that sees the old value ~0 enqueues x.  One
// atomic per examined edge replaces the load / CAS / min triple, and the
// result is deterministic, which makes the BFS forest bit-identical to the
// reference's "first discoverer in the sorted frontier" rule.
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "pipeline.cuh"
#include "samplers.h"

namespace gc {

namespace cg = cooperative_groups;

namespace {

constexpr int kTB = 256;                  // traversal block
#ifndef GC_TRAV_MINB
#define GC_TRAV_MINB 1  // min resident blocks of the frontier-expansion kernels
#endif
constexpr int kQCap = kTB * 16;           // 16 KB staging per block
__device__ __forceinline__ void red_or_u32(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// LDD claims: cluster[x] (u32, kFreeCluster = unclaimed) takes the minimum
// claimant of the first round x is reached in; croud[x] (u16) = that round
// + 1, written by the winner, tells later rounds to keep off.  True for the
// unique first claimant.  A claim of an earlier round is visible to every
// later round (one launch per round), and two claimants of the same round
// both pass the round filter, so the atomicMin picks the round's minimum —
// the semantics of one packed 64-bit (round, cluster) key, in 6 bytes per
// vertex instead of 8 and with a 2-byte filter read.
constexpr uint32_t kFreeCluster = ~0u;
__device__ __forceinline__ bool claim(uint32_t* cluster, uint16_t* croud, int32_t x, int32_t round, uint32_t c) {
  const uint16_t cr = croud[x];
  if (cr != 0 && int32_t(cr) - 1 < round) return false;          // reached in an earlier round
  if (uint32_t(ld_weak(reinterpret_cast<const int32_t*>(cluster + x))) <= c) return false;  // a smaller claimant won
  if (atomicMin(cluster + x, c) != kFreeCluster) return false;
  croud[x] = uint16_t(round + 1);
  return true;
}

__device__ __forceinline__ int32_t warp_min(int32_t v) {
  for (int o = 16; o > 0; o >>= 1) {
    const int32_t t = __shfl_xor_sync(0xffffffffu, v, o);
    v = t < v ? t : v;
  }
  return v;
}

// ------------------------------------------------------------------- BFS ---
// Direction-optimising level-synchronous BFS: top-down over a frontier
// queue while the frontier is small, bottom-up over a frontier bitmap (n/8
// bytes, L2-resident) once its edges dominate (Beamer's rule).  Bottom-up
// takes the first frontier vertex of x's ascending row — the same minimum
// the top-down atomicMin selects — so the forest does not depend on the
// direction schedule.  Frontier stats [count, degree sum] feed the switch
// and the inspection count (sum of frontier degrees, sampling.py:141-144).
//
// State: par[v] (u32, kUnreached until claimed, kSourcePar for the source)
// and the visited bitmap vis (n/8 bytes, L2-resident).  A top-down level
// reads vis frozen at the level start — vertices reached in earlier levels
// are skipped with a bit test instead of a random claim-word read — and
// resolves this level's claims with one 32-bit atomicMin of the frontier id
// per edge; the first claimant (old == kUnreached) enqueues.  The level's
// claims are merged into vis afterwards (k_or_words).
constexpr uint32_t kUnreached = 0xffffffffu;
constexpr uint32_t kSourcePar = 0xfffffffeu;

__device__ __forceinline__ bool test_bit(const uint32_t* bits, int32_t x) {
  return (__ldg(bits + (x >> 5)) >> (x & 31)) & 1u;
}


// One top-down level over the frontier queue q (count in qstat[0]); claims
// go to qn through the caller's block queue.  `frozen`: the visited bitmap
// is read through the non-coherent path (a separate launch froze it); the
// persistent form reads it coherently (other CTAs marked it in this launch).
template <bool COHERENT>
__device__ __forceinline__ void bfs_td_level(BlockQueue<kQCap>& bq, const int64_t* __restrict__ off,
                                             const int32_t* __restrict__ tgt, const int32_t* q, int64_t count,
                                             uint32_t* par, const uint32_t* vis, int32_t* qn,
                                             unsigned long long* nstat, uint32_t* nbits, int32_t* minv,
                                             unsigned long long* insp);

__global__ void __launch_bounds__(kTB, GC_TRAV_MINB)
k_bfs_td(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, const int32_t* __restrict__ q,
         const unsigned long long* qstat, uint32_t* par, const uint32_t* vis, int32_t* qn,
         unsigned long long* nstat, uint32_t* nbits, int32_t* minv, unsigned long long* insp,
         unsigned long long* zero_next) {
  __shared__ BlockQueue<kQCap> bq;
  bq.init();
  // batched levels: clear the stat slot the level after next will fill
  if (zero_next && blockIdx.x == 0 && threadIdx.x == 0) zero_next[0] = zero_next[1] = 0;
  bfs_td_level<false>(bq, off, tgt, q, int64_t(qstat[0]), par, vis, qn, nstat, nbits, minv, insp);
}

__device__ __forceinline__ uint32_t ld_vis(const uint32_t* p, bool coherent) {
  if (!coherent) return __ldg(p);
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <bool COHERENT>
__device__ __forceinline__ void bfs_td_level(BlockQueue<kQCap>& bq, const int64_t* __restrict__ off,
                                             const int32_t* __restrict__ tgt, const int32_t* q, int64_t count,
                                             uint32_t* par, const uint32_t* vis, int32_t* qn,
                                             unsigned long long* nstat, uint32_t* nbits, int32_t* minv,
                                             unsigned long long* insp) {
  const int lane = threadIdx.x & 31;
  auto claim_p = [&](int32_t x, int32_t f) {
    const uint32_t vw = ld_vis(vis + (x >> 5), COHERENT);
    const uint32_t seen = uint32_t(ld_weak(reinterpret_cast<const int32_t*>(par + x)));
    if ((vw >> (x & 31)) & 1u) return false;
    if (seen <= uint32_t(f)) return false;
    return atomicMin(par + x, uint32_t(f)) == kUnreached;
  };
  unsigned long long degs = 0;
  int32_t my_min = INT_MAX;
  auto take = [&](bool fresh, int32_t x) {
    if (fresh) {
      if (nbits) atomicOr(nbits + (x >> 5), 1u << (x & 31));
      my_min = x < my_min ? x : my_min;
    }
    bq.push(fresh, x, qn, nstat);
  };
  // a warp takes vpw frontier vertices per step: 32 while the frontier
  // fills every warp, fewer on narrow levels so that every warp of the grid
  // holds part of the level (a high-diameter level is a few thousand rows:
  // 32 rows per warp left most warps idle and the rest walking ~6 claim
  // steps each)
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  int64_t vpw64 = (count + nwarps - 1) / nwarps;
  const int vpw = int(vpw64 < 1 ? 1 : (vpw64 > 32 ? 32 : vpw64));
  for (int64_t base = gw * vpw; base < count; base += nwarps * vpw) {
    const int64_t i = base + lane;
    int32_t f = -1;
    int64_t b = 0, d = 0;
    if (lane < vpw && i < count) {
      f = COHERENT ? ld_acq(q + i) : q[i];
      b = off[f];
      d = off[f + 1] - b;
      degs += static_cast<unsigned long long>(d);  // frontier degree (counted at expansion)
    }
    const bool big = d > 32;
    // rows of at most 32 entries: the warp concatenates them and every lane
    // claims one entry per step (its row found by a binary search over the
    // warp's degree prefix), so a level costs one claim latency per 32 row
    // entries of the warp instead of one per entry of the longest row
    int32_t incl = big ? 0 : int32_t(d);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const int32_t dsm = big ? 0 : int32_t(d);
    for (int32_t e0 = 0; e0 < total; e0 += 32) {
      const int32_t e = e0 + lane;
      int lo = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int32_t v = __shfl_sync(0xffffffffu, incl, lo + step - 1);
        if (v <= e) lo += step;
      }
      const int src = lo > 31 ? 31 : lo;
      const int32_t se = __shfl_sync(0xffffffffu, incl, src);
      const int32_t sd = __shfl_sync(0xffffffffu, dsm, src);
      const int64_t sb = __shfl_sync(0xffffffffu, b, src);
      const int32_t sf = __shfl_sync(0xffffffffu, f, src);
      int32_t x = 0;
      bool fresh = false;
      if (e < total) {
        x = tgt[sb + (e - (se - sd))];
        fresh = claim_p(x, sf);
      }
      take(fresh, x);
    }
    unsigned mask = __ballot_sync(0xffffffffu, big);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const int32_t ff = __shfl_sync(0xffffffffu, f, src);
      const int64_t bb = __shfl_sync(0xffffffffu, b, src);
      const int64_t dd = __shfl_sync(0xffffffffu, d, src);
      for (int64_t j0 = 0; j0 < dd; j0 += 32) {
        const int64_t j = j0 + lane;
        int32_t x = 0;
        bool fresh = false;
        if (j < dd) {
          x = tgt[bb + j];
          fresh = claim_p(x, ff);
        }
        take(fresh, x);
      }
    }
    // (warps run different trip counts: no block-wide flush inside the loop;
    // a full staging area spills straight to the queue)
  }
  bq.flush(qn, nstat);
  if (insp) block_add<kTB>(insp, degs);
  my_min = warp_min(my_min);
  if (lane == 0 && my_min != INT_MAX) atomic_min_if_lower(minv, my_min);
}

// Narrow top-down levels in ONE persistent cooperative launch (SURVEY hard
// part 6: a 256^3 grid has 765 levels, and a launch pair per level cost
// ~21 us).  Per level: the claims of bfs_td_level, a grid barrier, the new
// queue's vertices marked visited (the bitmap stays frozen while a level
// claims, so same-level claimants all reach the atomicMin and the smallest
// frontier id wins, as in the reference), a grid barrier.  The launch stops
// after max_levels levels, on an empty frontier, or once the frontier
// reaches nf_stop (the host then re-evaluates the direction switch).
// Frontier stats [count, degree sum] use the ring of three slots of the
// launch-per-level form; out[0] = levels run.
__global__ void __launch_bounds__(kTB, GC_TRAV_MINB)
k_bfs_persist(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, int32_t* q0, int32_t* q1,
              unsigned long long* stat, int64_t level0, int32_t max_levels, unsigned long long nf_stop,
              uint32_t* par, uint32_t* vis, int32_t* minv, unsigned long long* reached,
              unsigned long long* out) {
  cg::grid_group grid = cg::this_grid();
  __shared__ BlockQueue<kQCap> bq;
  bq.init();
  const int64_t gtid = int64_t(blockIdx.x) * kTB + threadIdx.x;
  const int64_t gthreads = int64_t(gridDim.x) * kTB;
  int32_t k = 0;
  while (k < max_levels) {
    const int64_t L = level0 + k;
    int32_t* q = (L & 1) ? q1 : q0;
    int32_t* qn = (L & 1) ? q0 : q1;
    unsigned long long* cur = stat + 2 * (L % 3);
    unsigned long long* nxt = stat + 2 * ((L + 1) % 3);
    if (gtid == 0) {
      unsigned long long* z = stat + 2 * ((L + 2) % 3);
      z[0] = z[1] = 0;
    }
    const int64_t count = int64_t(*reinterpret_cast<volatile unsigned long long*>(cur));
    bfs_td_level<true>(bq, off, tgt, q, count, par, vis, qn, nxt, nullptr, minv, nullptr);
    grid.sync();
    const unsigned long long nn = *reinterpret_cast<volatile unsigned long long*>(nxt);
    for (int64_t i = gtid; i < int64_t(nn); i += gthreads) {
      const int32_t x = ld_acq(qn + i);
      atomicOr(vis + (x >> 5), 1u << (x & 31));
    }
    if (gtid == 0 && nn) atomicAdd(reached, nn);
    ++k;
    grid.sync();
    if (nn == 0 || nn >= nf_stop) break;
  }
  if (gtid == 0) out[0] = static_cast<unsigned long long>(k);
}

// Wide top-down levels (the frontier is no longer narrow) run in two
// passes, neither of which touches the parent array at random:
//   mark: every frontier row sets the next-frontier bit of each unvisited
//     neighbour (red.or into the n/8-byte bitmap, which stays in L2; no lane
//     waits on an atomic's result; rows are walked four entries at a time);
//   pull: every newly reached vertex, in id order, takes the first frontier
//     vertex of its ascending row as parent — the smallest frontier
//     neighbour, which is what the returning atomicMin of the narrow form
//     leaves — and writes it with a coalesced store.
// A returning atomicMin per claim into the 4n-byte parent array (n = 2^27:
// 537 MB, far beyond L2) made such a level a stream of random DRAM
// read-modify-writes.
__global__ void __launch_bounds__(kTB)
k_bfs_td_mark(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, const int32_t* __restrict__ q,
              const unsigned long long* qstat, const uint32_t* __restrict__ vis, uint32_t* nbits) {
  const int lane = threadIdx.x & 31;
  const int64_t count = int64_t(qstat[0]);
  for (int64_t i = int64_t(blockIdx.x) * kTB + threadIdx.x; i - lane < count; i += int64_t(gridDim.x) * kTB) {
    int64_t b = 0, d = 0;
    if (i < count) {
      const int32_t f = q[i];
      b = off[f];
      d = off[f + 1] - b;
    }
    const bool big = d > 32;
    if (!big) {
      for (int64_t j = 0; j < d; j += 4) {
        int32_t x[4];
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = j + k < d ? tgt[b + j + k] : -1;
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = x[k] >= 0 ? __ldg(vis + (x[k] >> 5)) : ~0u;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (x[k] >= 0 && !((w[k] >> (x[k] & 31)) & 1u))
            asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(nbits + (x[k] >> 5)),
                         "r"(1u << (x[k] & 31))
                         : "memory");
      }
    }
    unsigned mask = __ballot_sync(0xffffffffu, big);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const int64_t bb = __shfl_sync(0xffffffffu, b, src);
      const int64_t dd = __shfl_sync(0xffffffffu, d, src);
      for (int64_t j = lane; j < dd; j += 32) {
        const int32_t x = tgt[bb + j];
        if (!test_bit(vis, x))
          asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(nbits + (x >> 5)), "r"(1u << (x & 31))
                       : "memory");
      }
    }
  }
}

// pull pass over the new frontier's queue (ascending ids: k_bits_to_queue)
__global__ void __launch_bounds__(kTB)
k_bfs_pull(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, const int32_t* __restrict__ q,
           const unsigned long long* qstat, const uint32_t* __restrict__ cbits, uint32_t* par) {
  const int64_t count = int64_t(qstat[0]);
  for (int64_t i = int64_t(blockIdx.x) * kTB + threadIdx.x; i < count; i += int64_t(gridDim.x) * kTB) {
    const int32_t v = q[i];
    const int64_t b = off[v], e = off[v + 1];
    for (int64_t j = b; j < e; ++j) {
      const int32_t t = tgt[j];
      if (test_bit(cbits, t)) {
        par[v] = uint32_t(t);
        break;
      }
    }
  }
}

// bottom-up: a warp owns 32 consecutive vertices and writes its next-bitmap
// word whole; the visited bitmap word (one broadcast load per warp) skips
// reached vertices, and each unreached vertex stops at its first frontier
// neighbour in row order — the smallest one, as the top-down atomicMin picks.
__global__ void __launch_bounds__(kTB)
k_bfs_bu(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, int32_t n, uint32_t* par,
         const uint32_t* __restrict__ cbits, uint32_t* nbits, uint32_t* vis, unsigned long long* nstat,
         int32_t* minv) {
  const int lane = threadIdx.x & 31;
  unsigned long long cnt = 0, degs = 0;
  int32_t my_min = INT_MAX;
  const int64_t stride = int64_t(gridDim.x) * kTB;
  for (int64_t base = int64_t(blockIdx.x) * kTB; base < n; base += stride) {
    const int64_t v = base + threadIdx.x;
    const int64_t wi = (base + (threadIdx.x & ~31)) >> 5;
    const uint32_t vw = wi * 32 < n ? vis[wi] : ~0u;
    bool found = false;
    if (v < n && !((vw >> lane) & 1u)) {
      const int64_t b = off[v], e = off[v + 1];
      for (int64_t j = b; j < e; ++j) {
        const int32_t t = tgt[j];
        if (test_bit(cbits, t)) {
          found = true;
          par[v] = uint32_t(t);
          break;
        }
      }
      if (found) degs += static_cast<unsigned long long>(e - b);
    }
    const unsigned word = __ballot_sync(0xffffffffu, found);
    if (lane == 0 && word) {
      nbits[wi] = word;
      vis[wi] = vw | word;
    }
    if (found) {
      ++cnt;
      my_min = int32_t(v) < my_min ? int32_t(v) : my_min;
    }
  }
  block_add<kTB>(nstat, cnt);
  block_add<kTB>(nstat + 1, degs);
  my_min = warp_min(my_min);
  if (lane == 0 && my_min != INT_MAX) atomic_min_if_lower(minv, my_min);
}

// narrow levels: the visited bitmap takes the claimed queue's vertices
// (work ~ frontier, not n); `total` accumulates the reached count
__global__ void k_mark_queue(const int32_t* q, const unsigned long long* qstat, uint32_t* vis,
                             unsigned long long* total) {
  const int64_t count = int64_t(qstat[0]);
  if (blockIdx.x == 0 && threadIdx.x == 0 && count) atomicAdd(total, static_cast<unsigned long long>(count));
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    const int32_t x = q[i];
    atomicOr(vis + (x >> 5), 1u << (x & 31));
  }
}

// frontier queue -> bitmap (leaving batched mode for a bottom-up level)
__global__ void k_queue_to_bits(const int32_t* q, const unsigned long long* qstat, uint32_t* bits) {
  const int64_t count = int64_t(qstat[0]);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    const int32_t x = q[i];
    atomicOr(bits + (x >> 5), 1u << (x & 31));
  }
}

__global__ void k_or_words(uint32_t* dst, const uint32_t* src, int64_t words) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < words; w += stride) {
    const uint32_t x = src[w];
    if (x) dst[w] |= x;
  }
}

// bitmap -> queue (switching back to top-down): one thread per 32-bit word
__global__ void __launch_bounds__(kEwBlock)
k_bits_to_queue(uint32_t* bits, int32_t n, int32_t* q, unsigned long long* qc, int32_t* minv, int clear,
                const unsigned int* gate = nullptr, unsigned int* gate_next = nullptr) {
  using Scan = cub::BlockScan<int, kEwBlock>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long base;
  // LDD rounds: gate = "the round claimed something" (an empty bitmap has
  // nothing to scan); gate_next is the other parity's flag, which no kernel
  // reads now, cleared for the next round to set
  if (gate_next && blockIdx.x == 0 && threadIdx.x == 0) *gate_next = 0u;
  if (gate && *gate == 0u) return;
  const int64_t words = (int64_t(n) + 31) / 32;
  for (int64_t w0 = int64_t(blockIdx.x) * kEwBlock; w0 < words; w0 += int64_t(gridDim.x) * kEwBlock) {
    const int64_t wi = w0 + threadIdx.x;
    uint32_t word = wi < words ? bits[wi] : 0u;
    if (clear && word) bits[wi] = 0u;  // consumed: ready for the next round
    int rank, total;
    Scan(tmp).ExclusiveSum(__popc(word), rank, total);
    if (threadIdx.x == 0) base = total ? atomicAdd(qc, static_cast<unsigned long long>(total)) : 0ull;
    __syncthreads();
    unsigned long long p = base + rank;
    if (minv) {  // the smallest vertex reached (first set bit of the block's words)
      int32_t lo = word ? int32_t(wi * 32 + __ffs(word) - 1) : INT_MAX;
      lo = warp_min(lo);
      if ((threadIdx.x & 31) == 0 && lo != INT_MAX) atomic_min_if_lower(minv, lo);
    }
    while (word) {
      const int bit = __ffs(word) - 1;
      word &= word - 1;
      q[p++] = int32_t(wi * 32 + bit);
    }
    __syncthreads();
  }
}

__global__ void k_bfs_seed(const int64_t* off, uint32_t* par, int32_t* q, unsigned long long* qstat,
                           uint32_t* bits, uint32_t* vis, int32_t s, int32_t* minv) {
  par[s] = kSourcePar;
  q[0] = s;
  qstat[0] = 1;
  qstat[1] = static_cast<unsigned long long>(off[s + 1] - off[s]);
  bits[s >> 5] |= 1u << (s & 31);
  vis[s >> 5] |= 1u << (s & 31);
  *minv = s;
}

// k_bfs_seed with the source picked on the device (sampling.py:130-132):
// the first probe (sorted, distinct) of maximum degree, as np.argmax; the
// key (degree, -position) is reduced over the block
constexpr int kProbeTB = 256;
__global__ void __launch_bounds__(kProbeTB)
k_bfs_seed_probe(const int64_t* off, const int32_t* probes, int32_t np, uint32_t* par, int32_t* q,
                 unsigned long long* qstat, uint32_t* bits, uint32_t* vis, int32_t* minv) {
  __shared__ unsigned long long best;
  if (threadIdx.x == 0) best = 0ull;
  __syncthreads();
  unsigned long long mine = 0ull;
  for (int32_t i = threadIdx.x; i < np; i += kProbeTB) {
    const int32_t p = probes[i];
    const int64_t dd = off[p + 1] - off[p];
    const unsigned long long d = dd < 0xffffffffll ? static_cast<unsigned long long>(dd) : 0xffffffffull;
    // degree < 2^32 here (ids are int32); position breaks ties toward the first
    const unsigned long long key = (d << 32) | (0xffffffffull - uint32_t(i));
    mine = key > mine ? key : mine;
  }
  atomicMax(&best, mine);
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int32_t s = probes[0xffffffffull - (best & 0xffffffffull)];
  par[s] = kSourcePar;
  q[0] = s;
  qstat[0] = 1;
  qstat[1] = static_cast<unsigned long long>(off[s + 1] - off[s]);
  bits[s >> 5] |= 1u << (s & 31);
  vis[s >> 5] |= 1u << (s & 31);
  *minv = s;
}

// label the component with its minimum (sampling.py:158-160), emit forest
// slots (slot v = (parent, v)), and count the sample inspections: the
// reference adds every frontier's degree sum (:141-144), i.e. the degree of
// every reached vertex once.  Every slot is written (unreached: P[v] = v,
// empty forest slot), so the pipeline skips the label init and the forest
// fill when this pass runs.  Four vertices per thread, 16-byte loads and
// stores throughout.
__global__ void k_bfs_label(const uint32_t* __restrict__ par, const int32_t* minv, const int64_t* __restrict__ off,
                            int32_t n, int32_t* P, int32_t* fu, int32_t* fv, unsigned long long* insp, int vec) {
  const int32_t mn = *minv;
  unsigned long long degs = 0;
  const int64_t nq = (int64_t(n) + 3) / 4;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nq; i += stride) {
    const int64_t v0 = 4 * i;
    if (vec && v0 + 3 < n) {
      const uint4 pp = *reinterpret_cast<const uint4*>(par + v0);
      const uint32_t p[4] = {pp.x, pp.y, pp.z, pp.w};
      const int32_t v = int32_t(v0);
      int32_t lab[4], u[4], w[4];
      bool any = false;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool r = p[j] != kUnreached;
        any |= r;
        lab[j] = r ? mn : v + j;
        const bool slot = r && v + j != mn && p[j] != kSourcePar;
        u[j] = slot ? int32_t(p[j]) : -1;
        w[j] = slot ? v + j : -1;
      }
      reinterpret_cast<int4*>(P)[i] = make_int4(lab[0], lab[1], lab[2], lab[3]);
      if (fu) {
        reinterpret_cast<int4*>(fu)[i] = make_int4(u[0], u[1], u[2], u[3]);
        reinterpret_cast<int4*>(fv)[i] = make_int4(w[0], w[1], w[2], w[3]);
      }
      if (any) {
        const longlong2 o01 = *reinterpret_cast<const longlong2*>(off + v0);
        const longlong2 o23 = *reinterpret_cast<const longlong2*>(off + v0 + 2);
        const int64_t o4 = off[v0 + 4];
        const int64_t o[5] = {o01.x, o01.y, o23.x, o23.y, o4};
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (p[j] != kUnreached) degs += static_cast<unsigned long long>(o[j + 1] - o[j]);
      }
    } else {
      for (int64_t v = v0; v < n; ++v) {
        const uint32_t p = par[v];
        const bool r = p != kUnreached;
        P[v] = r ? mn : int32_t(v);
        if (r) degs += static_cast<unsigned long long>(off[v + 1] - off[v]);
        if (fu) {
          const bool slot = r && v != mn && p != kSourcePar;
          fu[v] = slot ? int32_t(p) : -1;
          fv[v] = slot ? int32_t(v) : -1;
        }
      }
    }
  }
  block_add<kEwBlock>(insp, degs);
}

// re-root the discovery tree at the component minimum (sampling.py:161-168):
// reverse the slots along the path mn -> ... -> source (one thread; the
// path has at most depth-many vertices)
__global__ void k_bfs_reroot(const uint32_t* par, const int32_t* minv, int32_t* fu, int32_t* fv) {
  int32_t cur = *minv;
  fu[cur] = -1;
  fv[cur] = -1;
  while (true) {
    const uint32_t p = par[cur];
    if (p == kSourcePar) break;  // reached the source
    fu[p] = cur;                 // slot p now holds (cur, p)
    fv[p] = int32_t(p);
    cur = int32_t(p);
  }
}

// ------------------------------------------------------------------- LDD ---
// Low-diameter decomposition (new; absent from the reference, driver.py:
// 65-69; ConnectIt, which GConn extends).  Miller-Peng-Xu:
//   delta_v ~ Exp(beta) from a counter hash of (seed, v); v may start its own
//   cluster at round floor(delta_max - delta_v); clusters grow one hop per
//   round; a vertex first reached in round r joins the smallest cluster id
//   among that round's claimants (its own id if it starts then).
// Vertices are bucketed by start round once, so each round touches only its
// own centres.  Labels are cluster minima: P[v] <= v and every class is
// connected, so the partition refines the true one (validate.py:290-297).

__device__ __forceinline__ float ldd_delta(uint64_t seed, int64_t v, float beta) {
  // a 24-bit uniform in (0, 1] from a 32-bit finaliser (murmur3 fmix32; the
  // 64-bit mix is emulated 64-bit multiplies) and the hardware log: delta <=
  // 24 ln 2 / beta (the double-precision form cost 0.19 ms of two passes at
  // 2^24)
  uint32_t h = uint32_t(v) * 0x9e3779b1u ^ uint32_t(seed) ^ uint32_t(seed >> 32) * 0x85ebca77u;
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  const float u = float((h >> 8) + 1u) * (1.0f / 16777216.0f);
  return -__logf(u) / beta;
}

__global__ void k_ldd_delta_max(int32_t n, uint64_t seed, float beta, int32_t* dmax_bits) {
  float mx = 0.f;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    mx = fmaxf(mx, ldd_delta(seed, v, beta));
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  // one atomic per block (one per warp serialised ~75K atomics on the one
  // word: 53 us at 2^24)
  __shared__ float wmax[32];
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = 0.f;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) b = fmaxf(b, wmax[w]);
    atomicMax(dmax_bits, __float_as_int(b));  // positive floats order as ints
  }
}

constexpr int kBuckets = kLddMaxRounds + 1;

// start round per vertex + block-aggregated bucket histogram
__global__ void __launch_bounds__(kEwBlock)
k_ldd_start(int32_t n, uint64_t seed, float beta, const int32_t* dmax_bits, uint16_t* start,
            uint32_t* cluster, uint16_t* croud, unsigned int* bcount, uint32_t* csize = nullptr,
            int32_t* pmin = nullptr) {
  __shared__ unsigned int hist[kBuckets];
  for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const float dmax = __int_as_float(*dmax_bits);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    float r = floorf(dmax - ldd_delta(seed, v, beta));
    r = r < 0.f ? 0.f : (r > float(kLddMaxRounds) ? float(kLddMaxRounds) : r);
    start[v] = uint16_t(r);
    cluster[v] = kFreeCluster;
    if (croud) croud[v] = 0;
    if (csize) csize[v] = 0;
    if (pmin) pmin[v] = INT_MAX;
    atomicAdd(hist + int(r), 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBuckets; i += blockDim.x)
    if (hist[i]) atomicAdd(bcount + i, hist[i]);
}

// exclusive scan of the bucket counts (one block); boff[kBuckets] = n
__global__ void __launch_bounds__(1024) k_ldd_bucket_scan(unsigned int* boff, unsigned int* cursor) {
  using Scan = cub::BlockScan<unsigned int, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  constexpr int kPer = (kBuckets + 1023) / 1024;
  unsigned int v[kPer];
  for (int j = 0; j < kPer; ++j) {
    const int i = threadIdx.x * kPer + j;
    v[j] = i < kBuckets ? boff[i] : 0u;
  }
  unsigned int total;
  Scan(tmp).ExclusiveSum(v, v, total);
  for (int j = 0; j < kPer; ++j) {
    const int i = threadIdx.x * kPer + j;
    if (i < kBuckets) boff[i] = cursor[i] = v[j];
  }
  if (threadIdx.x == 0) boff[kBuckets] = total;
}

// scatter vertices into their start-round buckets (order within a bucket is
// irrelevant: claims are resolved by atomicMin)
__global__ void __launch_bounds__(kEwBlock)
k_ldd_scatter(int32_t n, const uint16_t* start, unsigned int* cursor, int32_t* order) {
  __shared__ unsigned int hist[kBuckets];
  __shared__ unsigned int base[kBuckets];
  const int64_t span = int64_t(kEwBlock) * 16;  // vertices per block step
  for (int64_t b0 = int64_t(blockIdx.x) * span; b0 < n; b0 += int64_t(gridDim.x) * span) {
    for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    unsigned int local[16];
    for (int k = 0; k < 16; ++k) {
      const int64_t v = b0 + int64_t(k) * kEwBlock + threadIdx.x;
      local[k] = v < n ? atomicAdd(hist + start[v], 1u) : 0u;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kBuckets; i += blockDim.x)
      base[i] = hist[i] ? atomicAdd(cursor + i, hist[i]) : 0u;
    __syncthreads();
    for (int k = 0; k < 16; ++k) {
      const int64_t v = b0 + int64_t(k) * kEwBlock + threadIdx.x;
      if (v < n) order[base[start[v]] + local[k]] = int32_t(v);
    }
    __syncthreads();
  }
}

// One LDD round in one launch: grow the previous frontier, then start the
// centres of bucket r; both append to the same block queue.  Frontier
// counters form a ring of three so the kernel can zero the counter the
// next round will fill without touching the one it reads.
__global__ void __launch_bounds__(kTB)
k_ldd_round(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, uint32_t* cluster, uint16_t* croud,
            const int32_t* order, const unsigned int* boff, int32_t r, int32_t last_start, const int32_t* qin,
            const unsigned long long* cin, int32_t* qout, unsigned long long* cout, unsigned long long* cnext,
            unsigned long long* insp, uint32_t* nbits, unsigned int* any_claim) {
  __shared__ BlockQueue<kQCap> bq;
  bq.init();
  if (blockIdx.x == 0 && threadIdx.x == 0) *cnext = 0;
  unsigned long long my_insp = 0;
  bool claimed = false;
  if (r > 0) {
    const int64_t count = int64_t(*cin);
    for (int64_t base = int64_t(blockIdx.x) * kTB; base < count; base += int64_t(gridDim.x) * kTB) {
      const int64_t i = base + threadIdx.x;
      uint32_t c = 0;
      int64_t b = 0, d = 0;
      if (i < count) {
        const int32_t f = qin[i];
        c = cluster[f];  // final since round r-1
        b = off[f];
        d = off[f + 1] - b;
        my_insp += d;
      }
      int64_t dmax = d;
      for (int o = 16; o > 0; o >>= 1) {
        const int64_t t = __shfl_xor_sync(0xffffffffu, dmax, o);
        dmax = t > dmax ? t : dmax;
      }
      for (int64_t j = 0; j < dmax; ++j) {
        bool fresh = false;
        int32_t x = 0;
        if (j < d) {
          x = tgt[b + j];
          fresh = claim(cluster, croud, x, r, c);
        }
        if (nbits) {
          if (fresh) red_or_u32(nbits + (x >> 5), 1u << (x & 31));
          claimed |= fresh;
        } else {
          bq.push(fresh, x, qout, cout);
        }
      }
      if (!nbits) bq.maybe_flush(qout, cout, kQCap / 2);
    }
  }
  if (r <= last_start) {
    const int64_t lo = boff[r], hi = boff[r + 1];
    for (int64_t b0 = lo + int64_t(blockIdx.x) * kTB; b0 < hi; b0 += int64_t(gridDim.x) * kTB) {
      const int64_t i = b0 + threadIdx.x;
      int32_t v = 0;
      bool fresh = false;
      if (i < hi) {
        v = order[i];
        fresh = claim(cluster, croud, v, r, uint32_t(v));
      }
      if (nbits) {
        if (fresh) red_or_u32(nbits + (v >> 5), 1u << (v & 31));
        claimed |= fresh;
      } else {
        bq.push(fresh, v, qout, cout);
        bq.maybe_flush(qout, cout, kQCap / 2);
      }
    }
  }
  bq.flush(qout, cout);
  block_add<kTB>(insp, my_insp);
  if (any_claim && __syncthreads_or(int(claimed)) && threadIdx.x == 0) *any_claim = 1u;
}

// minimum member per cluster: lanes holding the same cluster (neighbouring
// ids usually share one) elect their lowest lane, which holds the smallest
// id, for a single atomicMin
__global__ void k_ldd_mins(const uint32_t* cluster, int32_t* mins, int32_t n) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
    const int64_t v = base + threadIdx.x;
    const uint32_t c = v < n ? cluster[v] : kFreeCluster;
    const unsigned peers = __match_any_sync(0xffffffffu, c);
    if (v < n && lane == __ffs(int(peers)) - 1) atomicMin(mins + c, int32_t(v));
  }
}

__global__ void k_ldd_label(const uint32_t* cluster, const int32_t* mins, int32_t* P, int32_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    P[v] = mins[cluster[v]];
}

// All LDD rounds in one persistent cooperative launch (one CTA group per
// SM, grid-wide barrier between rounds).  Round r expands the frontier of
// round r-1 and starts bucket r's centres.  Claim state is the 6-byte form
// of the launch-per-round kernel: cluster[x] (u32, atomicMin) and croud[x]
// (u16, claim round + 1, written by the first claimant).  The croud filter
// rejects vertices claimed in an earlier round with a 2-byte read of a
// 2n-byte array that stays in L2 (ncu of an 8-byte packed (round, cluster)
// key: 10.3 GB of DRAM reads for one LDD on the permuted 256^3 grid, L2 hit
// 25%); only vertices unclaimed or claimed in this round reach the
// cluster atomicMin, so the result is the deterministic MPX clustering.
// The frontier is expanded edge-parallel inside each warp (32 frontier
// vertices, their rows concatenated, one edge per lane per step: a lane's
// source is found by a binary search over the warp's degree prefix); fresh
// claims go to a block queue flushed once per round.  Per-round frontier
// counters form a ring of three; the first start round and the end of the
// rounds are read on the device, so the sampler needs no host round trip.
// After the rounds the same launch takes the minimum member of each cluster
// and writes the labels.
__device__ __forceinline__ uint32_t ld_rlx_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint16_t ld_rlx_u16(const uint16_t* p) {
  uint16_t v;
  asm volatile("ld.relaxed.gpu.global.u16 %0, [%1];" : "=h"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool claim_rel(uint32_t* cluster, uint16_t* croud, int32_t x, int32_t round, uint32_t c) {
  const uint16_t cr = ld_rlx_u16(croud + x);
  if (cr != 0 && int32_t(cr) - 1 != round) return false;  // reached in an earlier round
  if (atomicMin(cluster + x, c) != kFreeCluster) return false;
  croud[x] = uint16_t(round + 1);
  return true;
}

// Packed claim state (n <= 2^24 and every round < 255): one u32 per vertex,
// key = round << 24 | cluster.  atomicMin on the key keeps the earliest
// round and, within it, the smallest cluster — the MPX rule itself — so the
// separate claim-round array (and its write) goes away: 4 bytes of claim
// state per vertex instead of 6 (67 MB at 2^24, which the L2 can hold).  The
// filter read rejects keys of earlier rounds before the atomic.
constexpr uint32_t kPackMask = 0xffffffu;

// Block-aggregated append of (u, v) pairs (the cut edges LDD emits): warps
// stage into shared memory, the block reserves its range with one counter
// atomic per flush; a full stage overflows per warp to the global list.
template <int CAP>
struct PairQueue {
  int2 items[CAP];
  int count;
  unsigned long long base;
  __device__ __forceinline__ void init() {
    if (threadIdx.x == 0) count = 0;
    __syncthreads();
  }
  __device__ __forceinline__ void push(bool p, int32_t a, int32_t b, int32_t* gu, int32_t* gv,
                                       unsigned long long* gc) {
    const unsigned bal = __ballot_sync(0xffffffffu, p);
    if (!bal) return;
    const int lane = threadIdx.x & 31;
    int pos = 0;
    if (lane == 0) pos = atomicAdd(&count, __popc(bal));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    const int mine = pos + __popc(bal & ((1u << lane) - 1u));
    if (p && mine < CAP) items[mine] = make_int2(a, b);
    const unsigned over = __ballot_sync(0xffffffffu, p && mine >= CAP);
    if (!over) return;
    unsigned long long g = 0;
    if (lane == __ffs(int(over)) - 1) g = atomicAdd(gc, static_cast<unsigned long long>(__popc(over)));
    g = __shfl_sync(0xffffffffu, g, __ffs(int(over)) - 1) + __popc(over & ((1u << lane) - 1u));
    if (p && mine >= CAP) {
      gu[g] = a;
      gv[g] = b;
    }
  }
  __device__ __forceinline__ void flush(int32_t* gu, int32_t* gv, unsigned long long* gc) {
    __syncthreads();
    const int c = count < CAP ? count : CAP;
    if (threadIdx.x == 0) base = c ? atomicAdd(gc, static_cast<unsigned long long>(c)) : 0ull;
    __syncthreads();
    for (int i = threadIdx.x; i < c; i += blockDim.x) {
      gu[base + i] = items[i].x;
      gv[base + i] = items[i].y;
    }
    __syncthreads();
    if (threadIdx.x == 0) count = 0;
    __syncthreads();
  }
};
__device__ __forceinline__ bool claim_packed(uint32_t* key, int32_t x, int32_t round, uint32_t c) {
  const uint32_t k = ld_rlx_u32(key + x);
  if ((k >> 24) < uint32_t(round)) return false;  // reached in an earlier round (free = round 255)
  return atomicMin(key + x, (uint32_t(round) << 24) | c) == kFreeCluster;
}

template <bool PACKED>
__global__ void __launch_bounds__(kTB, 6)
k_ldd_persist(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, int32_t n, uint32_t* cluster,
              uint16_t* croud, const int32_t* __restrict__ order, const unsigned int* __restrict__ boff,
              const int32_t* dmax_bits, int32_t max_rounds, int32_t* q0, int32_t* q1, unsigned long long* ring,
              unsigned long long* insp, int32_t* mins, int32_t* P, unsigned long long* rounds_out,
              unsigned int* trace, uint32_t* csize, unsigned long long* ctr, int32_t* cut_u, int32_t* cut_v,
              unsigned long long* cut_count) {
  cg::grid_group grid = cg::this_grid();
  // 12 KB of frontier staging + 8 KB of cut-pair staging: the same shared
  // memory as the 16 KB frontier stage plus a 4 KB pair stage (a larger
  // total costs the cooperative grid resident blocks: 2048 pairs measured
  // the sampler 2.6 -> 4.6 ms)
  __shared__ BlockQueue<kTB * 12> bq;
  __shared__ PairQueue<1024> pq;
  bq.init();
  pq.init();
  // cut-edge emission (packed form, labels-only rounds finishes): expanding
  // a vertex of cluster c claimed in round r - 1, a neighbour x whose claim
  // is final (claimed in an earlier round) and in another cluster is a cut
  // edge; of two vertices claimed in the same round only the smaller id
  // emits — every edge between two clusters exactly once, so the finish
  // needs no gather over the active rows
  const bool emit = PACKED && cut_u != nullptr;
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (int64_t(blockIdx.x) * kTB + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * kTB) >> 5;
  const int64_t gtid = int64_t(blockIdx.x) * kTB + threadIdx.x;
  const int64_t gthreads = int64_t(gridDim.x) * kTB;
  int32_t last_start = int32_t(floorf(__int_as_float(*dmax_bits)));
  last_start = last_start < 0 ? 0 : (last_start > max_rounds ? max_rounds : last_start);
  unsigned long long my_insp = 0;
  const uint64_t pol = evict_first_policy();
  // One round (frontier expansion + the round's centres) over the warps /
  // threads [w0, w0 + nw) / [t0, t0 + nt); ends with the block queues
  // flushed.  The caller synchronises the participants.
  auto round = [&](int32_t r, int64_t w0, int64_t nw, int64_t t0, int64_t nt) -> unsigned long long* {
    int32_t* qin = (r & 1) ? q0 : q1;  // round r reads the queue round r-1 wrote
    int32_t* qout = (r & 1) ? q1 : q0;
    unsigned long long* cout = ring + (r + 1) % 3;
    if (t0 == 0) ring[(r + 2) % 3] = 0;  // read by nobody this round; written next round
    const int64_t count = r > 0 ? int64_t(*reinterpret_cast<volatile unsigned long long*>(ring + r % 3)) : 0;
    // vpw frontier vertices per warp step: fewer than 32 on narrow rounds so
    // every warp of the grid takes part (see bfs_td_level)
    const int64_t vpw64 = (count + nw - 1) / nw;
    const int vpw = int(vpw64 < 1 ? 1 : (vpw64 > 32 ? 32 : vpw64));
    for (int64_t wb = w0 * vpw; wb < count; wb += nw * vpw) {
      const int64_t i = wb + lane;
      uint32_t c = 0;
      int64_t b = 0;
      int32_t d = 0;
      int32_t f = INT_MAX;
      if (lane < vpw && i < count) {
        f = ld_acq(qin + i);
        c = ld_rlx_u32(cluster + f);  // final since round r-1
        if constexpr (PACKED) c &= kPackMask;
        // graph data is read once: L2 evict-first keeps the claim state resident
        b = ld_stream64(off + f, pol);
        d = int32_t(ld_stream64(off + f + 1, pol) - b);
        my_insp += d;
      }
      if constexpr (PACKED) {
        // every claimed vertex is expanded exactly once, in the round after
        // its (final) claim: count it for its cluster here — the exact
        // cluster sizes, so the pipeline needs no label histogram for the
        // mode (lanes holding the same cluster add once)
        const bool has = lane < vpw && i < count;
        const unsigned peers = __match_any_sync(0xffffffffu, has ? c : kFreeCluster);
        // and its minimum member, straight into P[c] (P[v] = INT_MAX until
        // the labelling; a non-empty cluster's centre c is its own member,
        // so P[c] ends as its own label and can serve as the cluster slot)
        const unsigned fmin = __reduce_min_sync(peers, unsigned(f));
        if (has && lane == __ffs(int(peers)) - 1) {
          atomicAdd(csize + c, unsigned(__popc(peers)));
          atomicMin(P + c, int32_t(fmin));
        }
      }
      int32_t incl = d;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
      // two edges per lane per step (e and e + 32): two independent claim
      // chains in flight per lane
      for (int32_t e0 = 0; e0 < total; e0 += 64) {
        int32_t x[2], sf[2];
        uint32_t sc[2];
        bool ok[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int32_t e = e0 + 32 * h + lane;
          // source lane: the first lane whose inclusive prefix exceeds e
          int lo = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const int32_t v = __shfl_sync(0xffffffffu, incl, lo + step - 1);
            if (v <= e) lo += step;
          }
          const int src = lo > 31 ? 31 : lo;
          const int32_t se = __shfl_sync(0xffffffffu, incl, src);
          const int32_t sd = __shfl_sync(0xffffffffu, d, src);
          const int64_t sb = __shfl_sync(0xffffffffu, b, src);
          sc[h] = __shfl_sync(0xffffffffu, c, src);
          sf[h] = __shfl_sync(0xffffffffu, f, src);
          ok[h] = e < total;
          x[h] = ok[h] ? ld_stream(tgt + sb + (e - (se - sd)), pol) : 0;
        }
        bool fresh[2], cut[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          cut[h] = false;
          if constexpr (PACKED) {
            fresh[h] = false;
            if (ok[h]) {
              const uint32_t kx = ld_rlx_u32(cluster + x[h]);
              const uint32_t kr = kx >> 24;
              if (kr < uint32_t(r)) {  // claimed in an earlier round: final
                cut[h] = emit && (kx & kPackMask) != sc[h] && (kr != uint32_t(r - 1) || sf[h] < x[h]);
              } else {
                fresh[h] = atomicMin(cluster + x[h], (uint32_t(r) << 24) | sc[h]) == kFreeCluster;
              }
            }
          } else {
            fresh[h] = ok[h] && claim_rel(cluster, croud, x[h], r, sc[h]);
          }
        }
        bq.push(fresh[0], x[0], qout, cout);
        bq.push(fresh[1], x[1], qout, cout);
        if (emit) {
          pq.push(cut[0], sf[0], x[0], cut_u, cut_v, cut_count);
          pq.push(cut[1], sf[1], x[1], cut_u, cut_v, cut_count);
        }
      }
    }
    if (r <= last_start) {  // centres of bucket r
      const int64_t lo = boff[r], hi = boff[r + 1];
      for (int64_t b0 = lo + (t0 - int64_t(threadIdx.x)); b0 < hi; b0 += nt) {
        const int64_t i = b0 + threadIdx.x;
        int32_t v = 0;
        bool fresh = false;
        if (i < hi) {
          v = order[i];
          if constexpr (PACKED) fresh = claim_packed(cluster, v, r, uint32_t(v));
          else fresh = claim_rel(cluster, croud, v, r, uint32_t(v));
        }
        bq.push(fresh, v, qout, cout);
      }
    }
    bq.flush(qout, cout);
    if (emit) pq.flush(cut_u, cut_v, cut_count);
    return cout;
  };
  int32_t r = 0;
  // every claim is a fresh vertex: once all n are claimed the remaining
  // start buckets hold only claimed vertices and their rounds would claim
  // nothing (the trace of the permuted 256^3 grid shows ~18 such trailing
  // rounds, each a grid barrier)
  unsigned long long claimed = 0;
  for (;; ++r) {
    unsigned long long* cout = round(r, gwarp, nwarps, gtid, gthreads);
    grid.sync();
    const unsigned long long next = *reinterpret_cast<volatile unsigned long long*>(cout);
    claimed += next;
    if (trace && gtid == 0 && r < max_rounds) trace[r] = unsigned(next);
    if ((next == 0 && r >= last_start) || (next == 0 && claimed >= static_cast<unsigned long long>(n))) break;
  }
  block_add<kTB>(insp, my_insp);
  if (gtid == 0 && rounds_out) *rounds_out = (unsigned long long)(r + 1);
  if constexpr (PACKED) {
    // the cluster minima are in P[centre] already (taken while expanding):
    // every other vertex reads its centre's slot, which never changes
    for (int64_t v = gtid; v < n; v += gthreads) {
      const int32_t c = int32_t(ld_rlx_u32(cluster + v) & kPackMask);
      if (c != v) P[v] = ld_acq(P + c);
    }
    mins = P;  // the mode pass below reads the minima from the centres' slots
  } else {
  // labels: minimum member id per cluster (warp-elected atomicMin over the
  // lanes holding the same cluster), then P[v] = mins[cluster(v)]
  for (int64_t v = gtid; v < n; v += gthreads) mins[v] = INT_MAX;
  grid.sync();
  for (int64_t base = gtid - lane; base < n; base += gthreads) {
    const int64_t v = base + lane;
    uint32_t c = v < n ? ld_rlx_u32(cluster + v) : kFreeCluster;
    if constexpr (PACKED) c = v < n ? c & kPackMask : c;
    const unsigned peers = __match_any_sync(0xffffffffu, c);
    if (v < n && lane == __ffs(int(peers)) - 1) atomicMin(mins + c, int32_t(v));
  }
  grid.sync();
  for (int64_t v = gtid; v < n; v += gthreads) {
    uint32_t c = ld_rlx_u32(cluster + v);
    if constexpr (PACKED) c &= kPackMask;
    P[v] = ld_acq(mins + c);
  }
  }
  if constexpr (PACKED) {
    // the mode: the largest cluster, ties to the smaller label (its minimum
    // member), as np.bincount(...).argmax() (sampling.py:29-35)
    unsigned long long best = 0;
    for (int64_t c = gtid; c < n; c += gthreads) {
      const uint32_t sz = csize[c];
      if (sz) {
        const unsigned long long key =
            (static_cast<unsigned long long>(sz) << 32) | (0xffffffffull - uint32_t(ld_acq(mins + c)));
        best = key > best ? key : best;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
      best = t > best ? t : best;
    }
    if (lane == 0 && best) atomicMax(ctr + C_SCRATCH0, best);
    grid.sync();
    if (gtid == 0) {
      const unsigned long long k = ctr[C_SCRATCH0];
      ctr[C_CAND] = 0xffffffffull - (k & 0xffffffffull);
      ctr[C_SCRATCH0] = 0;
      ctr[C_MODE_EXACT] = 1;
    }
  }
}

#define TL(kernel, grid, block, ...) ((kernel<<<grid, block, 0, st>>>(__VA_ARGS__)), ::gc::count_launch())

}  // namespace

// Direction switch (Beamer): bottom-up once the frontier's edges exceed
// 1/alpha of the unexplored ones, back to top-down below n/beta frontier
// vertices.  Beamer's alpha = 14 is also the GPU optimum once a top-down
// level's queue appends are block-aggregated (with one counter atomic per
// overflowing claim, the large top-down level serialised and alpha = 30 —
// switching a level early — measured better).
constexpr int kBfsBeta = 24;
double bfs_alpha() {
  static const double a = [] {
    const char* e = getenv("GC_BFS_ALPHA");
    // measured on uniform 2^27 (forest): 8 -> 9.26 ms, 14 -> 9.27 ms, 30 -> 10.41 ms
    return e ? atof(e) : 14.0;
  }();
  return a;
}

// frontier size from which a non-batched top-down level uses the
// fire-and-forget claims (below it the returning atomics are cheap and the
// queue is built in the same pass)
// (n/2048: 65536 at n = 2^27; small graphs take the wide form from 256
// frontier vertices on, which keeps it covered by the test graphs)
unsigned long long bfs_wide_min(int64_t n) {
  static const long long v = [] {
    const char* e = getenv("GC_BFS_WIDE_MIN");
    return e ? atoll(e) : -1ll;
  }();
  if (v >= 0) return static_cast<unsigned long long>(v);
  const int64_t t = n >> 11;
  return static_cast<unsigned long long>(t > 256 ? t : 256);
}

// GC_BFS_PERSIST=0: narrow levels as a launch pair per level (batched 64 per
// host round trip) instead of one persistent cooperative launch
bool bfs_persistent() {
  static const bool p = [] {
    const char* e = getenv("GC_BFS_PERSIST");
    return !(e && e[0] == '0');
  }();
  return p;
}

bool bfs_trace() {
  static const bool t = getenv("GC_BFS_TRACE") != nullptr;
  return t;
}

void run_bfs(const gc_csr& g, const gc_spec& s, int32_t* P, int32_t* fu, int32_t* fv, SamplerWs& w,
             unsigned long long* ctr, cudaStream_t st) {
  const int32_t n = int32_t(g.n);
  if (n == 0 || g.m == 0) return;  // sampling.py:128-129
  const bool probe_src = s.bfs_source < 0 && s.bfs_probes && s.bfs_nprobes > 0;
  require(probe_src || (s.bfs_source >= 0 && s.bfs_source < n), GC_ERR_ARG, "BFS source out of range");
  if (probe_src)
    for (int32_t i = 0; i < s.bfs_nprobes; ++i)
      require(s.bfs_probes[i] >= 0 && s.bfs_probes[i] < n, GC_ERR_ARG, "BFS probe out of range");
  const int64_t words = (int64_t(n) + 31) / 32;
  uint32_t* par = reinterpret_cast<uint32_t*>(w.key);  // the claim buffer, as u32 parents
  GC_CUDA(cudaMemsetAsync(par, 0xff, size_t(n) * 4, st));  // kUnreached
  GC_CUDA(cudaMemsetAsync(w.fb0, 0, words * 4, st));
  GC_CUDA(cudaMemsetAsync(w.fb1, 0, words * 4, st));
  GC_CUDA(cudaMemsetAsync(w.vis, 0, words * 4, st));
  int32_t* minv = reinterpret_cast<int32_t*>(ctr + C_SCRATCH1);
  // frontier stats [count, degree sum] per level in a ring of three slots
  // (level L reads slot(L), writes slot(L+1)); slot 3 counts reached vertices
  auto slot = [&](int64_t L) { return w.stat + 2 * (L % 3); };
  unsigned long long* reached = w.stat + 6;
  int32_t* q[2] = {w.q0, w.q1};
  uint32_t* fb[2] = {w.fb0, w.fb1};
  GC_CUDA(cudaMemsetAsync(w.stat, 0, 8 * sizeof(unsigned long long), st));
  if (probe_src) {
    // the probe list rides in the second frontier queue until the seed
    // kernel has picked the source from it
    GC_CUDA(cudaMemcpyAsync(q[1], s.bfs_probes, size_t(s.bfs_nprobes) * 4, cudaMemcpyHostToDevice, st));
    TL(k_bfs_seed_probe, 1, kProbeTB, g.offsets, q[1], s.bfs_nprobes, par, q[0], slot(0), fb[0], w.vis, minv);
  } else {
    TL(k_bfs_seed, 1, 1, g.offsets, par, q[0], slot(0), fb[0], w.vis, int32_t(s.bfs_source), minv);
  }
  GC_CHECK_LAUNCH();
  unsigned long long* h = pinned_words();
  GC_CUDA(cudaMemcpyAsync(h, slot(0), 16, cudaMemcpyDeviceToHost, st));
  GC_CUDA(cudaStreamSynchronize(st));
  unsigned long long nf = h[0];
  double mf = double(h[1]);  // frontier edges: exact for the seed / bottom-up levels, estimated top-down
  const double avg_deg = double(g.m) / double(n);
  double unexplored = double(g.m) - mf;
  bool bottom_up = false;
  bool bits_stale = false;  // fb[current] not built (after batched levels)
  const int bu_grid = grid_for(n, kTB, 4);
  const int narrow_grid = num_sms() * 8;
  // Narrow frontiers (high-diameter graphs: a 256^3 grid has 765 levels)
  // run kBfsBatch top-down levels per host round trip: the kernels read the
  // frontier size on the device, claims go straight to the queue, and a
  // queue-sized pass marks them visited.  The direction switch is checked
  // between batches; parents are direction-independent, so the schedule
  // never changes the result.
  // The batch length is chosen so the frontier, growing at the observed
  // per-level rate (avg degree before any observation), stays narrow.
  constexpr int kBfsMaxBatch = 64;
  double growth = avg_deg > 1.01 ? avg_deg : 1.01;
  for (int64_t level = 0; nf > 0;) {
    int batch = 0;
    // batch while the predicted frontier stays well inside top-down
    // territory (half the switch threshold)
    const double limit = unexplored / (2.0 * bfs_alpha() * avg_deg);
    if (!bottom_up && double(nf) < limit) {
      const double k = std::log(limit / double(nf)) / std::log(growth);
      batch = k > kBfsMaxBatch ? kBfsMaxBatch : int(k);
    }
    if (batch >= 2) {
      const unsigned long long nf0 = nf;
      GC_CUDA(cudaMemsetAsync(slot(level + 1), 0, 16, st));
      if (bfs_persistent()) {
        // every narrow level in one cooperative launch, until the frontier
        // reaches the narrow bound (the direction switch is re-evaluated
        // on the host) or empties
        static int per_sm = 0;
        if (!per_sm) {
          GC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bfs_persist, kTB, 0));
          if (per_sm < 1) throw Error(GC_ERR_CUDA, "BFS persistent kernel does not fit on an SM");
        }
        const int64_t* off = g.offsets;
        const int32_t* tgt = g.targets;
        int32_t* q0 = q[0];
        int32_t* q1 = q[1];
        unsigned long long* stat = w.stat;
        int64_t lv0 = level;
        int32_t maxl = 1 << 20;
        unsigned long long nfs = static_cast<unsigned long long>(limit > 1.0 ? limit : 1.0);
        uint32_t* vis = w.vis;
        unsigned long long* outp = w.stat + 7;
        void* args[] = {&off, &tgt, &q0, &q1, &stat, &lv0, &maxl, &nfs, &par, &vis, &minv, &reached, &outp};
        GC_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_bfs_persist),
                                            dim3(num_sms() * per_sm), dim3(kTB), args, 0, st));
        ::gc::count_launch();
        GC_CHECK_LAUNCH();
        GC_CUDA(cudaMemcpyAsync(h + 3, outp, 8, cudaMemcpyDeviceToHost, st));
        GC_CUDA(cudaStreamSynchronize(st));
        batch = int(h[3]);
      } else {
        for (int k = 0; k < batch; ++k) {
          const int64_t L = level + k;
          TL(k_bfs_td, narrow_grid, kTB, g.offsets, g.targets, q[L & 1], slot(L), par, w.vis, q[(L + 1) & 1],
             slot(L + 1), static_cast<uint32_t*>(nullptr), minv, static_cast<unsigned long long*>(nullptr),
             slot(L + 2));
          TL(k_mark_queue, narrow_grid, kEwBlock, q[(L + 1) & 1], slot(L + 1), w.vis, reached);
        }
        GC_CHECK_LAUNCH();
      }
      level += batch;
      GC_CUDA(cudaMemcpyAsync(h, slot(level), 16, cudaMemcpyDeviceToHost, st));
      GC_CUDA(cudaMemcpyAsync(h + 2, reached, 8, cudaMemcpyDeviceToHost, st));
      GC_CUDA(cudaStreamSynchronize(st));
      nf = h[0];
      mf = double(nf) * avg_deg;
      unexplored = double(g.m) - double(h[2] + 1) * avg_deg;
      if (nf > 0) {
        const double observed = std::pow(double(nf) / double(nf0), 1.0 / batch);
        // safety margin on the exponent, not the factor: a slowly growing
        // frontier (a 3-D grid grows ~1% per level) keeps long batches
        // instead of one host round trip every few levels
        const double g15 = std::pow(observed > 1.0 ? observed : 1.0, 1.5);
        growth = g15 > 1.01 ? g15 : 1.01;
      }
      bits_stale = true;
      continue;
    }
    const int c = int(level & 1), nx = c ^ 1;
    // Beamer's heuristic: bottom-up once the frontier's edges exceed
    // 1/alpha of the unexplored ones, back to top-down below n/beta
    const bool want_bu = bottom_up ? (nf >= uint64_t(n) / kBfsBeta) : (mf * bfs_alpha() > unexplored);
    if ((want_bu || nf >= bfs_wide_min(n)) && bits_stale) {
      GC_CUDA(cudaMemsetAsync(fb[c], 0, words * 4, st));
      TL(k_queue_to_bits, grid_for(int64_t(nf), kEwBlock, 4), kEwBlock, q[c], slot(level), fb[c]);
    }
    bits_stale = false;
    if (!want_bu && bottom_up) {
      GC_CUDA(cudaMemsetAsync(slot(level), 0, 8, st));
      TL(k_bits_to_queue, grid_for(words, kEwBlock, 4), kEwBlock, fb[c], n, q[c], slot(level),
         static_cast<int32_t*>(nullptr), 0);
    }
    bottom_up = want_bu;
    GC_CUDA(cudaMemsetAsync(slot(level + 1), 0, 16, st));
    GC_CUDA(cudaMemsetAsync(fb[nx], 0, words * 4, st));
    if (bottom_up) {
      TL(k_bfs_bu, bu_grid, kTB, g.offsets, g.targets, n, par, fb[c], fb[nx], w.vis, slot(level + 1), minv);
    } else {
      const int64_t b64 = (int64_t(nf) + kTB - 1) / kTB;
      const int blocks = int(b64 < int64_t(num_sms()) * 8 ? (b64 > 0 ? b64 : 1) : int64_t(num_sms()) * 8);
      if (nf >= bfs_wide_min(n)) {
        TL(k_bfs_td_mark, blocks, kTB, g.offsets, g.targets, q[c], slot(level), w.vis, fb[nx]);
        TL(k_bits_to_queue, grid_for(words, kEwBlock, 4), kEwBlock, fb[nx], n, q[nx], slot(level + 1), minv, 0);
        TL(k_bfs_pull, num_sms() * (2048 / kTB), kTB, g.offsets, g.targets, q[nx], slot(level + 1), fb[c], par);
      } else {
        TL(k_bfs_td, blocks, kTB, g.offsets, g.targets, q[c], slot(level), par, w.vis, q[nx], slot(level + 1),
           fb[nx], minv, static_cast<unsigned long long*>(nullptr), static_cast<unsigned long long*>(nullptr));
      }
      // the visited bitmap takes the level's claims in one word-parallel pass
      // (an extra atomic per claim would double the level's atomics)
      TL(k_or_words, grid_for(words, kEwBlock, 2), kEwBlock, w.vis, fb[nx], words);
    }
    GC_CHECK_LAUNCH();
    ++level;
    GC_CUDA(cudaMemcpyAsync(h, slot(level), 16, cudaMemcpyDeviceToHost, st));
    GC_CUDA(cudaStreamSynchronize(st));
    nf = h[0];
    mf = bottom_up ? double(h[1]) : double(nf) * avg_deg;
    unexplored -= mf;
    if (bfs_trace()) fprintf(stderr, "bfs level %lld %s next frontier %llu\n", (long long)level,
                             bottom_up ? "bottom-up" : "top-down", nf);
  }
  const auto al = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  const int vec = al(g.offsets) && al(P) && (!fu || (al(fu) && al(fv)));
  TL(k_bfs_label, grid_for((int64_t(n) + 3) / 4, kEwBlock, 8), kEwBlock, par, minv, g.offsets, n, P, fu, fv,
     ctr + C_INSP_SAMPLE, vec);
  if (fu) TL(k_bfs_reroot, 1, 1, par, minv, fu, fv);
  GC_CHECK_LAUNCH();
}

// GC_LDD_PACKED=0 keeps the 6-byte (u32 cluster + u16 round) claim state
// in the persistent kernel even when the packed key fits
bool ldd_packed() {
  static const bool p = [] {
    const char* e = getenv("GC_LDD_PACKED");
    return !(e && e[0] == '0');
  }();
  return p;
}

// GC_LDD_PERSIST=0 selects the launch-per-round form (k_ldd_round +
// k_bits_to_queue, host termination check every 16 rounds)
bool ldd_persistent() {
  static const bool p = [] {
    const char* e = getenv("GC_LDD_PERSIST");
    return !(e && e[0] == '0');
  }();
  return p;
}

bool run_ldd(const gc_csr& g, const gc_spec& s, int32_t* P, SamplerWs& w, unsigned long long* ctr,
             cudaStream_t st) {
  const int32_t n = int32_t(g.n);
  w.cut_done = false;
  if (n == 0) return false;
  const float beta = s.ldd_beta > 0 ? float(s.ldd_beta) : 0.2f;
  int32_t* dmax = reinterpret_cast<int32_t*>(ctr + C_SCRATCH1);
  unsigned int* bcount = w.boff;
  unsigned int* cursor = w.cursor;
  GC_CUDA(cudaMemsetAsync(dmax, 0, 4, st));
  GC_CUDA(cudaMemsetAsync(bcount, 0, (kBuckets + 1) * sizeof(unsigned int), st));
  const int ge = grid_for(n, kEwBlock, 8);
  TL(k_ldd_delta_max, ge, kEwBlock, n, s.seed, beta, dmax);
  if (ldd_persistent()) {
    // one cooperative launch runs every round and the labelling (no host
    // round trip); the start-round buckets come from the three passes below
    uint32_t* cl = reinterpret_cast<uint32_t*>(w.key);
    // packed 4-byte claim keys when ids fit 24 bits and every round fits 8:
    // the start rounds are <= delta_max <= 24 ln 2 / beta (the exponential
    // draw's largest value), so beta > 0.066 keeps them < 254
    const bool packed = ldd_packed() && n <= (1 << 24) && 16.7f / beta < 253.f;
    uint16_t* cr = packed ? nullptr : reinterpret_cast<uint16_t*>(cl + n);
    // packed: the second half of the 8n-byte claim buffer counts cluster sizes
    uint32_t* csz = packed ? cl + n : nullptr;
    TL(k_ldd_start, ge, kEwBlock, n, s.seed, beta, dmax, w.start, cl, cr, bcount, csz, packed ? P : nullptr);
    TL(k_ldd_bucket_scan, 1, 1024, bcount, cursor);
    TL(k_ldd_scatter, grid_for(((int64_t(n) + 4095) / 4096) * kEwBlock, kEwBlock, 64), kEwBlock, n, w.start,
       cursor, w.order);
    GC_CUDA(cudaMemsetAsync(w.stat, 0, 3 * sizeof(unsigned long long), st));
    static int per_sm = 0;
    if (!per_sm) {
      int a = 0, b = 0;
      GC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_ldd_persist<false>, kTB, 0));
      GC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_ldd_persist<true>, kTB, 0));
      per_sm = a < b ? a : b;
      if (per_sm < 1) throw Error(GC_ERR_CUDA, "LDD persistent kernel does not fit on an SM");
    }
    const int64_t* off = g.offsets;
    const int32_t* tgt = g.targets;
    uint32_t* clp = cl;
    uint16_t* crp = cr;
    const int32_t* order = w.order;
    const unsigned int* boff = w.boff;
    const int32_t* dmb = dmax;
    int32_t maxr = kLddMaxRounds;
    int32_t* q0 = w.q0;
    int32_t* q1 = w.q1;
    unsigned long long* ring = w.stat;
    unsigned long long* insp = ctr + C_INSP_SAMPLE;
    int32_t* mins = w.q0;  // the queues are dead once the rounds end
    int32_t* Pp = P;
    unsigned long long* rounds_out = w.stat + 3;
    int32_t nn = n;
    // GC_LDD_TRACE: per-round frontier sizes on stderr
    static const bool trace_on = getenv("GC_LDD_TRACE") != nullptr;
    unsigned int* trace = nullptr;
    if (trace_on) GC_CUDA(cudaMallocAsync(&trace, sizeof(unsigned int) * (kLddMaxRounds + 1), st));
    if (trace) GC_CUDA(cudaMemsetAsync(trace, 0, sizeof(unsigned int) * (kLddMaxRounds + 1), st));
    uint32_t* cszp = csz;
    unsigned long long* ctrp = ctr;
    // emitting costs per cut edge, the gather it replaces is a fixed pass
    // over the active rows: emit while the cut share is small (ic ~ beta /
    // 2 on the 3-D grid: 0.05 / 0.10 / 0.24 at beta 0.1 / 0.2 / 0.5; the
    // gather won at 0.5)
    w.cut_done = packed && w.cut_u != nullptr && beta <= 0.3f;
    int32_t* cutu = w.cut_done ? w.cut_u : nullptr;
    int32_t* cutv = w.cut_done ? w.cut_v : nullptr;
    unsigned long long* cutc = w.cut_done ? w.cut_count : nullptr;
    void* args[] = {&off, &tgt, &nn, &clp, &crp, &order, &boff, &dmb, &maxr, &q0, &q1, &ring, &insp, &mins, &Pp,
                    &rounds_out, &trace, &cszp, &ctrp, &cutu, &cutv, &cutc};
    const void* kfn = packed ? reinterpret_cast<const void*>(k_ldd_persist<true>)
                             : reinterpret_cast<const void*>(k_ldd_persist<false>);
    GC_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(num_sms() * per_sm), dim3(kTB), args, 0, st));
    ::gc::count_launch();
    GC_CHECK_LAUNCH();
    if (trace) {
      std::vector<unsigned int> h(kLddMaxRounds + 1);
      unsigned long long nr = 0;
      GC_CUDA(cudaMemcpyAsync(h.data(), trace, sizeof(unsigned int) * h.size(), cudaMemcpyDeviceToHost, st));
      GC_CUDA(cudaMemcpyAsync(&nr, rounds_out, 8, cudaMemcpyDeviceToHost, st));
      GC_CUDA(cudaStreamSynchronize(st));
      fprintf(stderr, "ldd rounds %llu:", nr);
      for (unsigned long long i = 0; i < nr && i < h.size(); ++i) fprintf(stderr, " %u", h[i]);
      fprintf(stderr, "\n");
      GC_CUDA(cudaFreeAsync(trace, st));
    }
    return packed;
  }
  // the claim buffer (8n bytes) holds the u32 clusters and the u16 claim rounds
  uint32_t* cluster = reinterpret_cast<uint32_t*>(w.key);
  uint16_t* croud = reinterpret_cast<uint16_t*>(cluster + n);
  // Sorted frontiers: a round's claims set bits, and a word-parallel scan
  // turns them into the next round's queue in ascending id order (clearing
  // the bitmap as it goes).  Row and claim accesses of the next round then
  // follow the id order instead of the block-flush order of a shared queue:
  // on the 256^3 grid the rounds take 2.5 ms instead of 3.9 ms.
  const int64_t words = (int64_t(n) + 31) / 32;
  uint32_t* nbits = w.fb0;
  GC_CUDA(cudaMemsetAsync(nbits, 0, size_t(words) * 4, st));
  // per-parity "round claimed something" flags (in the free tail of stat)
  unsigned int* flag = reinterpret_cast<unsigned int*>(w.stat + 4);
  GC_CUDA(cudaMemsetAsync(flag, 0, 2 * sizeof(unsigned int), st));
  TL(k_ldd_start, ge, kEwBlock, n, s.seed, beta, dmax, w.start, cluster, croud, bcount);
  TL(k_ldd_bucket_scan, 1, 1024, bcount, cursor);
  TL(k_ldd_scatter, grid_for(((int64_t(n) + 4095) / 4096) * kEwBlock, kEwBlock, 64), kEwBlock, n, w.start,
     cursor, w.order);
  GC_CHECK_LAUNCH();
  unsigned long long* hq = pinned_words();
  GC_CUDA(cudaMemcpyAsync(hq + 1, dmax, 4, cudaMemcpyDeviceToHost, st));
  GC_CUDA(cudaStreamSynchronize(st));
  float dmax_h;
  std::memcpy(&dmax_h, hq + 1, 4);
  int32_t last_start = int32_t(floorf(dmax_h));
  if (last_start > kLddMaxRounds) last_start = kLddMaxRounds;
  if (last_start < 0) last_start = 0;
  // frontier counters: a ring of three (round r reads ring[(r+2)%3], writes
  // ring[r%3] and zeroes ring[(r+1)%3]); queues ping-pong
  unsigned long long* ring = w.stat;
  int32_t* q[2] = {w.q0, w.q1};
  GC_CUDA(cudaMemsetAsync(ring, 0, 3 * sizeof(unsigned long long), st));
  // rounds are enqueued kLddBatch at a time (one launch per round, kernels
  // read the frontier size on the device); the host checks termination per batch
  constexpr int kLddBatch = 16;
  const int grid = num_sms() * 8;
  for (int32_t r = 0;;) {
    for (int k = 0; k < kLddBatch; ++k, ++r) {
      TL(k_ldd_round, grid, kTB, g.offsets, g.targets, cluster, croud, w.order, w.boff, r, last_start, q[(r + 1) & 1],
         ring + (r + 2) % 3, q[r & 1], ring + r % 3, ring + (r + 1) % 3, ctr + C_INSP_SAMPLE, nbits, flag + (r & 1));
      TL(k_bits_to_queue, grid_for(words, kEwBlock, 4), kEwBlock, nbits, n, q[r & 1], ring + r % 3,
         static_cast<int32_t*>(nullptr), 1, flag + (r & 1), flag + ((r + 1) & 1));
    }
    GC_CHECK_LAUNCH();
    GC_CUDA(cudaMemcpyAsync(hq, ring + (r - 1) % 3, 8, cudaMemcpyDeviceToHost, st));
    GC_CUDA(cudaStreamSynchronize(st));
    if (*hq == 0 && r > last_start) break;
  }
  // labels: minimum member id per cluster (q0 is free again: reuse as mins)
  int32_t* mins = w.q0;
  fill(mins, n, INT_MAX, st);
  TL(k_ldd_mins, ge, kEwBlock, cluster, mins, n);
  TL(k_ldd_label, ge, kEwBlock, cluster, mins, P, n);
  GC_CHECK_LAUNCH();
  return false;
}

}  // namespace gc
