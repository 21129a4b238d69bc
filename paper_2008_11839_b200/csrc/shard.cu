// shard.cu — the compact label exchange of the sharded pipeline.
//
// After gc_shard_sample every rank holds the partition induced by the
// sampled edges of its own rows.  Exchanging it edge by edge costs one pair
// per sampled row.  Instead each rank describes its partition by
//   * one large class as an n-bit bitmap plus that class's label, and
//   * a pair (v, root) for every other non-singleton vertex,
// and the exchange runs in two rounds:
//   A. bitmaps of the local giants only; every rank absorbs all of them into
//      its local partition (giants sharing a vertex are one class; every
//      member is unioned with its class representative), so local fragments
//      that touch any giant join it;
//   B. bitmaps of the now-dominant class plus the remainder pairs, which are
//      few (fragments that touch no giant anywhere); gc_shard_join rebuilds
//      the join of every rank's partition from them.
// The result is exactly the partition of all sampled edges, so L_max, cov,
// the active set and the finish inspections equal the single-GPU pipeline's.
#include <climits>

#include "internal.h"
#include "pipeline.cuh"

namespace gc {

namespace {

constexpr int kMaxRanks = 8;  // one NVSwitch box; the overlap matrix is one u64

// the bitmap class: the root of the hint vertex, else the probe's candidate
// (any class gives an exact summary; a large one makes it compact)
__global__ void k_pick_class(const int32_t* P, const int32_t* hint, unsigned long long* ctr, int64_t* label_out) {
  int32_t g = int32_t(ctr[C_CAND]);
  if (hint) {
    g = *hint;
    int32_t y;
    while ((y = P[g]) != g) g = y;
  }
  ctr[C_LMAX] = static_cast<unsigned long long>(g);
  *label_out = g;
}

// bitmap words + block-aggregated remainder pairs (P compressed).  Four
// vertices per thread (one 16-byte load): a warp covers 128 vertices = four
// bitmap words, each OR-reduced over the eight lanes that hold it.
// COMPRESS: the labels are first resolved to their roots and written back
// (the compress pass fused in: round A's parents come straight from the
// sampler; the class was picked by the probe, which walks to roots itself)
template <bool COMPRESS>
__global__ void __launch_bounds__(kEwBlock)
k_summary(int32_t* __restrict__ P, int32_t n, const unsigned long long* ctr, uint32_t* bits,
          int32_t* out_u, int32_t* out_v, unsigned long long* out_count) {
  constexpr int kWarps = kEwBlock / 32;
  __shared__ unsigned warp_n[kWarps];
  __shared__ unsigned long long block_pos;
  const int32_t g = int32_t(ctr[C_LMAX]);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t nq = (int64_t(n) + 3) / 4;
  const int64_t words = (int64_t(n) + 31) / 32;
  // the trip count is uniform per block (base is), so the barriers are safe
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < nq; base += stride) {
    const int64_t q = base + threadIdx.x;
    const int64_t v0 = 4 * q;
    int32_t lab[4] = {0, 0, 0, 0};
    if (v0 + 3 < n) {
      const int4 p = reinterpret_cast<const int4*>(P)[q];
      lab[0] = p.x, lab[1] = p.y, lab[2] = p.z, lab[3] = p.w;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) lab[k] = v0 + k < n ? P[v0 + k] : g;
    }
    if constexpr (COMPRESS) {
      // first hops of the four walks together; only labels that moved walk on
      int32_t hop[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) hop[k] = (v0 + k < n && lab[k] != int32_t(v0 + k)) ? ld_weak(P + lab[k]) : lab[k];
      bool dirty = false;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (v0 + k >= n || hop[k] == lab[k]) continue;
        int32_t r = hop[k], y;
        while ((y = ld_weak(P + r)) != r) r = y;
        lab[k] = r;
        dirty = true;
      }
      if (dirty) {
        if (v0 + 3 < n) reinterpret_cast<int4*>(P)[q] = make_int4(lab[0], lab[1], lab[2], lab[3]);
        else
          for (int k = 0; k < 4; ++k)
            if (v0 + k < n) P[v0 + k] = lab[k];
      }
    }
    unsigned nib = 0, pairs = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool in_g = lab[k] == g && v0 + k < n;
      nib |= unsigned(in_g) << k;
      pairs |= unsigned(!in_g && v0 + k < n && lab[k] != int32_t(v0 + k)) << k;
    }
    unsigned word = nib << (4 * (lane & 7));
    word |= __shfl_xor_sync(0xffffffffu, word, 1);
    word |= __shfl_xor_sync(0xffffffffu, word, 2);
    word |= __shfl_xor_sync(0xffffffffu, word, 4);
    if ((lane & 7) == 0 && (v0 >> 5) < words) bits[v0 >> 5] = word;
    if (!out_u) continue;  // bitmap only (round A)
    // one counter atomic per block: small fragments are spread over most
    // blocks, and a per-warp atomic on the one counter serialised the pass
    const unsigned mine = __popc(pairs);
    unsigned incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_n[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned tot = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) tot += warp_n[w];
      block_pos = tot ? atomicAdd(out_count, static_cast<unsigned long long>(tot)) : 0ull;
    }
    __syncthreads();
    if (pairs) {
      unsigned long long i = block_pos + incl - mine;
      for (int w = 0; w < warp; ++w) i += warp_n[w];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (pairs & (1u << k)) {
          out_u[i] = int32_t(v0 + k);
          out_v[i] = lab[k];
          ++i;
        }
    }
    __syncthreads();  // warp_n / block_pos are rewritten next iteration
  }
}


// overlap matrix: bit (r * 8 + s) set when giants r < s share a vertex
__global__ void __launch_bounds__(kEwBlock)
k_overlap(const uint32_t* __restrict__ bits, int64_t words, int32_t nranks, unsigned long long* mat) {
  unsigned long long m = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < words; w += stride) {
    uint32_t b[kMaxRanks];
#pragma unroll
    for (int r = 0; r < kMaxRanks; ++r) b[r] = r < nranks ? bits[int64_t(r) * words + w] : 0u;
#pragma unroll
    for (int r = 0; r < kMaxRanks; ++r)
#pragma unroll
      for (int s = r + 1; s < kMaxRanks; ++s)
        if (b[r] & b[s]) m |= 1ull << (r * 8 + s);
  }
  // one atomic per block (every warp of an overlapping region sets bits)
  __shared__ unsigned long long bm;
  if (threadIdx.x == 0) bm = 0;
  __syncthreads();
  for (int o = 16; o > 0; o >>= 1) m |= __shfl_xor_sync(0xffffffffu, m, o);
  if ((threadIdx.x & 31) == 0 && m) atomicOr(&bm, m);
  __syncthreads();
  if (threadIdx.x == 0 && bm) atomicOr(mat, bm);
}

// super-classes of the giants (tiny union-find over <= 8 nodes); rep[r] =
// smallest giant label in r's class
__global__ void k_giant_classes(const unsigned long long* mat, const int64_t* labels, int32_t nranks,
                                int32_t* rep, int32_t* single) {
  int par[kMaxRanks];
  for (int r = 0; r < kMaxRanks; ++r) par[r] = r;
  auto root = [&](int x) {
    while (par[x] != x) x = par[x];
    return x;
  };
  const unsigned long long m = *mat;
  for (int r = 0; r < nranks; ++r)
    for (int s = r + 1; s < nranks; ++s)
      if ((m >> (r * 8 + s)) & 1ull) {
        const int a = root(r), b = root(s);
        if (a != b) par[a > b ? a : b] = a < b ? a : b;
      }
  for (int r = 0; r < nranks; ++r) {
    int64_t best = LLONG_MAX;
    for (int s = 0; s < nranks; ++s)
      if (root(s) == root(r) && labels[s] < best) best = labels[s];
    rep[r] = int32_t(best);
  }
  if (single) {
    int one = 1;
    for (int r = 1; r < nranks; ++r) one &= rep[r] == rep[0];
    *single = one;
  }
}

// round A, streaming form (P compressed: P[v] is v's local root).
// Pass 1: every non-root member v of some giant marks its local root with
// the bit of the giant's class (one byte per root).  Local roots are never
// marked by themselves — at P ranks most bitmap members are local singletons
// (their rows live on other ranks), and marking those would be one random
// atomic per vertex; the apply pass reads a root's own bitmap class instead.
// A root whose class differs from a member's joins the two classes.
// Pass 2: every vertex whose local root carries a class points at that
// class's representative.
__device__ __forceinline__ int lowest_class(unsigned m) { return __ffs(int(m)) - 1; }

// class of v's first bitmap (-1: none).  All rank words are loaded up front:
// an early-exit loop would serialise up to eight dependent cache misses.
__device__ __forceinline__ int first_rank(const uint32_t* __restrict__ bits, int64_t words, int32_t nranks,
                                          int64_t v) {
  const int64_t w = v >> 5;
  uint32_t b[kMaxRanks];
#pragma unroll
  for (int q = 0; q < kMaxRanks; ++q) b[q] = q < nranks ? __ldg(bits + int64_t(q) * words + w) : 0u;
  unsigned hit = 0;
#pragma unroll
  for (int q = 0; q < kMaxRanks; ++q) hit |= ((b[q] >> (v & 31)) & 1u) << q;
  return hit ? __ffs(int(hit)) - 1 : -1;
}

__device__ __forceinline__ int bitmap_class(const uint32_t* __restrict__ bits, int64_t words, int32_t nranks,
                                            const int32_t* __restrict__ cls, int64_t v) {
  const int q = first_rank(bits, words, nranks, v);
  return q < 0 ? -1 : cls[q];
}

// the class (through cls) of each of the four vertices 4q..4q+3, from one
// load of every rank's bitmap word
__device__ __forceinline__ void quad_classes(const uint32_t* __restrict__ bits, int64_t words, int32_t nranks,
                                             const int32_t* __restrict__ cls, int64_t v0, int c[4]) {
  uint32_t b[kMaxRanks];
#pragma unroll
  for (int q = 0; q < kMaxRanks; ++q) b[q] = q < nranks ? __ldg(bits + int64_t(q) * words + (v0 >> 5)) : 0u;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    unsigned hit = 0;
#pragma unroll
    for (int q = 0; q < kMaxRanks; ++q) hit |= ((b[q] >> ((v0 + k) & 31)) & 1u) << q;
    c[k] = hit ? cls[__ffs(int(hit)) - 1] : -1;
  }
}

// Both passes take four vertices per thread per step (one 16-byte parent
// load, one bitmap word per rank): the one-vertex form issued two dependent
// DRAM round trips per vertex and ran latency-bound at ~1 TB/s.
__device__ __forceinline__ void mark_one(int32_t v, int32_t r, int c, const uint32_t* __restrict__ bits,
                                         int64_t words, int32_t nranks, const int32_t* __restrict__ cls,
                                         uint32_t* mark, unsigned long long* mat, int32_t& last_r, int& last_c) {
  if (r == v || c < 0 || (r == last_r && c == last_c)) return;
  last_r = r;
  last_c = c;
  const int cr = bitmap_class(bits, words, nranks, cls, r);
  if (cr >= 0 && cr != c) atomicOr(mat, 1ull << (cr * 8 + c));
  uint32_t* word = mark + (r >> 2);
  const uint32_t mine = (1u << c) << (8 * (r & 3));
  if (ld_weak(reinterpret_cast<const int32_t*>(word)) & mine) return;  // stale => one extra atomic
  const uint32_t old = (atomicOr(word, mine) >> (8 * (r & 3))) & 0xffu;
  if (old && !(old & (1u << c))) atomicOr(mat, 1ull << (lowest_class(old) * 8 + c));
}

__global__ void __launch_bounds__(kEwBlock)
k_absorb_mark(const int32_t* __restrict__ P, int32_t n, const uint32_t* __restrict__ bits, int64_t words,
              int32_t nranks, const int32_t* __restrict__ cls, uint32_t* mark, unsigned long long* mat,
              const int32_t* single) {
  if (*single) return;
  // a per-thread memo of the last (root, class) handled keeps the giant's
  // root word from being hit once per member
  int32_t last_r = -1;
  int last_c = -1;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t nq = n / 4;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nq; q += stride) {
    const int4 p = reinterpret_cast<const int4*>(P)[q];
    int c[4];
    quad_classes(bits, words, nranks, cls, 4 * q, c);
    const int32_t v = int32_t(4 * q);
    mark_one(v, p.x, c[0], bits, words, nranks, cls, mark, mat, last_r, last_c);
    mark_one(v + 1, p.y, c[1], bits, words, nranks, cls, mark, mat, last_r, last_c);
    mark_one(v + 2, p.z, c[2], bits, words, nranks, cls, mark, mat, last_r, last_c);
    mark_one(v + 3, p.w, c[3], bits, words, nranks, cls, mark, mat, last_r, last_c);
  }
  for (int64_t v = 4 * nq + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    mark_one(int32_t(v), P[v], bitmap_class(bits, words, nranks, cls, v), bits, words, nranks, cls, mark, mat,
             last_r, last_c);
}

// class bits of local root r: its mark byte plus its own bitmap class
__device__ __forceinline__ uint32_t root_classes(int32_t r, const uint32_t* __restrict__ mark,
                                                 const uint32_t* __restrict__ bits, int64_t words, int32_t nranks,
                                                 const int32_t* __restrict__ cls0) {
  uint32_t m = (__ldg(mark + (r >> 2)) >> (8 * (r & 3))) & 0xffu;
  const int cr = bitmap_class(bits, words, nranks, cls0, r);
  return cr >= 0 ? m | (1u << cr) : m;
}

__global__ void __launch_bounds__(kEwBlock)
k_absorb_apply(int32_t* P, int32_t n, const uint32_t* __restrict__ mark, const uint32_t* __restrict__ bits,
               int64_t words, int32_t nranks, const int32_t* __restrict__ cls0, const int32_t* __restrict__ cls_rep,
               const int32_t* single) {
  if (*single) return;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t nq = n / 4;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nq; q += stride) {
    int4 p = reinterpret_cast<int4*>(P)[q];
    // lookups for every distinct root of the quad, issued together (the
    // repeated ones - a giant's members - hit L1)
    const uint32_t m0 = root_classes(p.x, mark, bits, words, nranks, cls0);
    const uint32_t m1 = p.y == p.x ? m0 : root_classes(p.y, mark, bits, words, nranks, cls0);
    const uint32_t m2 = p.z == p.y ? m1 : root_classes(p.z, mark, bits, words, nranks, cls0);
    const uint32_t m3 = p.w == p.z ? m2 : root_classes(p.w, mark, bits, words, nranks, cls0);
    if (!(m0 | m1 | m2 | m3)) continue;
    if (m0) p.x = cls_rep[lowest_class(m0)];
    if (m1) p.y = cls_rep[lowest_class(m1)];
    if (m2) p.z = cls_rep[lowest_class(m2)];
    if (m3) p.w = cls_rep[lowest_class(m3)];
    reinterpret_cast<int4*>(P)[q] = p;
  }
  for (int64_t v = 4 * nq + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const uint32_t m = root_classes(P[v], mark, bits, words, nranks, cls0);
    if (m) P[v] = cls_rep[lowest_class(m)];
  }
}

// classes of the giants from a class matrix (bit i*8+j: i and j joined).
// pass 0: over ranks, from the bitmap overlaps.  pass 1: merges the pass-0
// classes that met at a shared local root.  Per rank: cls[r] = class index
// (a rank id), rep[r] = the class's smallest giant label; cls_rep[c] = rep for
// every class index c a mark byte can carry (pass-0 and merged ids alike).
__global__ void k_absorb_classes(const unsigned long long* mat, const int64_t* labels, int32_t nranks,
                                 int32_t* cls, int32_t* rep, int32_t* cls_rep, int pass, int32_t* single) {
  int par[kMaxRanks];
  for (int r = 0; r < kMaxRanks; ++r) par[r] = r;
  auto root = [&](int x) {
    while (par[x] != x) x = par[x];
    return x;
  };
  const unsigned long long m = *mat;
  for (int r = 0; r < kMaxRanks; ++r)
    for (int s = 0; s < kMaxRanks; ++s)
      if (r != s && ((m >> (r * 8 + s)) & 1ull)) {
        const int a = root(r), b = root(s);
        if (a != b) par[a > b ? a : b] = a < b ? a : b;
      }
  int c0[kMaxRanks];
  for (int r = 0; r < nranks; ++r) {
    c0[r] = pass == 0 ? r : cls[r];
    cls[r] = root(c0[r]);
  }
  for (int r = 0; r < nranks; ++r) {
    int64_t best = LLONG_MAX;
    for (int s = 0; s < nranks; ++s)
      if (cls[s] == cls[r] && labels[s] < best) best = labels[s];
    rep[r] = int32_t(best);
  }
  for (int r = 0; r < nranks; ++r) {
    cls_rep[c0[r]] = rep[r];
    cls_rep[cls[r]] = rep[r];
  }
  if (single) {
    int one = 1;
    for (int r = 1; r < nranks; ++r) one &= cls[r] == cls[0];
    *single = one;
  }
}

// One class (the usual case: every rank's giant is a piece of the one giant
// component).  Then the class matrix has nothing to record, a vertex's class
// is one bit of the OR of the bitmaps, and the per-root class byte shrinks to
// one bit: mark1 sets bit r for every local root r with a member in the
// class, apply1 points every vertex whose root is marked or in the class at
// the representative.  Four vertices per thread, one bitmap word per quad.
__device__ __forceinline__ bool bit_of(const uint32_t* __restrict__ b, int32_t x) {
  return (__ldg(b + (x >> 5)) >> (x & 31)) & 1u;
}

__global__ void __launch_bounds__(kEwBlock)
k_absorb_mark1(const int32_t* __restrict__ P, int32_t n, const uint32_t* __restrict__ any, uint32_t* mark,
               const int32_t* single) {
  if (!*single) return;
  int32_t last_r = -1;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t nq = (int64_t(n) + 3) / 4;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nq; q += stride) {
    const int64_t v0 = 4 * q;
    int32_t r[4];
    if (v0 + 3 < n) {
      const int4 p = reinterpret_cast<const int4*>(P)[q];
      r[0] = p.x, r[1] = p.y, r[2] = p.z, r[3] = p.w;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) r[k] = v0 + k < n ? P[v0 + k] : int32_t(v0 + k);
    }
    const uint32_t w = __ldg(any + (v0 >> 5)) >> (v0 & 31);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int32_t x = r[k];
      if (x == int32_t(v0 + k) || !((w >> k) & 1u) || x == last_r) continue;
      last_r = x;
      const uint32_t bit = 1u << (x & 31);
      if (ld_weak(reinterpret_cast<const int32_t*>(mark + (x >> 5))) & bit) continue;
      atomicOr(mark + (x >> 5), bit);
    }
  }
}

__global__ void __launch_bounds__(kEwBlock)
k_absorb_apply1(int32_t* P, int32_t n, const uint32_t* __restrict__ mark, const uint32_t* __restrict__ any,
                const int32_t* __restrict__ rep, const int32_t* single) {
  if (!*single) return;
  const int32_t r0 = rep[0];
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t nq = n / 4;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nq; q += stride) {
    int4 p = reinterpret_cast<int4*>(P)[q];
    const bool m0 = bit_of(mark, p.x) || bit_of(any, p.x);
    const bool m1 = p.y == p.x ? m0 : bit_of(mark, p.y) || bit_of(any, p.y);
    const bool m2 = p.z == p.y ? m1 : bit_of(mark, p.z) || bit_of(any, p.z);
    const bool m3 = p.w == p.z ? m2 : bit_of(mark, p.w) || bit_of(any, p.w);
    if (!(m0 | m1 | m2 | m3)) continue;
    if (m0) p.x = r0;
    if (m1) p.y = r0;
    if (m2) p.z = r0;
    if (m3) p.w = r0;
    reinterpret_cast<int4*>(P)[q] = p;
  }
  for (int64_t v = 4 * nq + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const int32_t x = P[v];
    if (bit_of(mark, x) || bit_of(any, x)) P[v] = r0;
  }
}

// one class (the usual case): OR the ranks' bitmaps once, word-parallel,
// then one bitmap test per vertex (the general path tests up to 8)
__global__ void __launch_bounds__(kEwBlock)
k_or_bitmaps(const uint32_t* __restrict__ bits, int64_t words, int32_t nranks, uint32_t* out,
             const int32_t* single) {
  if (!*single) return;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < words; w += stride) {
    uint32_t x = 0;
    for (int q = 0; q < nranks; ++q) x |= bits[int64_t(q) * words + w];
    out[w] = x;
  }
}

__global__ void __launch_bounds__(kEwBlock)
k_join_init_one(int32_t* P, int32_t n, const uint32_t* __restrict__ any, const int32_t* __restrict__ rep,
                const int32_t* single) {
  if (!*single) return;
  const int32_t r0 = rep[0];
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t nq = n / 4;  // four vertices per thread, one 16-byte store
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nq; q += stride) {
    const int32_t v = int32_t(4 * q);
    const uint32_t w = __ldg(any + (v >> 5)) >> (v & 31);
    reinterpret_cast<int4*>(P)[q] = make_int4(w & 1u ? r0 : v, w & 2u ? r0 : v + 1, w & 4u ? r0 : v + 2,
                                              w & 8u ? r0 : v + 3);
  }
  for (int64_t v = 4 * nq + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    P[v] = (any[v >> 5] >> (v & 31)) & 1u ? r0 : int32_t(v);
}

__global__ void __launch_bounds__(kEwBlock)
k_join_init(int32_t* P, int32_t n, const uint32_t* __restrict__ bits, int64_t words, int32_t nranks,
            const int32_t* __restrict__ rep, const int32_t* single) {
  if (*single) return;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const int q = first_rank(bits, words, nranks, v);
    P[v] = q < 0 ? int32_t(v) : rep[q];
  }
}

}  // namespace

}  // namespace gc

using namespace gc;

extern "C" {

size_t gc_shard_summary_workspace(int64_t n) { (void)n; return 4096; }

int gc_shard_summary(int32_t* parent, int64_t n, const int32_t* giant_hint, uint32_t* giant_bits,
                     int64_t* giant_label, int32_t* out_u, int32_t* out_v, unsigned long long* out_count, void* ws,
                     size_t ws_bytes, void* stream) {
  return guarded([&] {
    require(n >= 0 && n < (int64_t(1) << 31), GC_ERR_MALFORMED, "bad length");
    require(giant_label && (n == 0 || (parent && giant_bits)), GC_ERR_ARG, "null argument");
    require((out_u == nullptr) == (out_v == nullptr) && (out_u == nullptr || out_count), GC_ERR_ARG,
            "pairs need u, v and a count");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Arena a(ws, ws_bytes);
    unsigned long long* ctr = a.take<unsigned long long>(C_COUNT_);
    GC_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * C_COUNT_, st));
    if (out_count) GC_CUDA(cudaMemsetAsync(out_count, 0, sizeof(unsigned long long), st));
    const int32_t nn = int32_t(n);
    if (nn == 0) {
      GC_CUDA(cudaMemsetAsync(giant_label, 0, sizeof(int64_t), st));
      return;
    }
    // round B (a hint) follows gc_shard_absorb, which leaves every vertex
    // pointing at its root: the compress pass would read 4n bytes plus one
    // hop per vertex for nothing (P = 8 model at s27: 0.2 ms per rank)
    // the probe walks to roots itself, so it runs before the compress, which
    // is fused into the summary pass (round A); round B's parents are
    // compressed already
    if (!giant_hint) (k_mode_probe<<<1, 1024, 0, st>>>(parent, nn, ctr, 1), count_launch());
    (k_pick_class<<<1, 1, 0, st>>>(parent, giant_hint, ctr, giant_label), count_launch());
    // a null pair output summarises the bitmap class only (round A)
    const int gs = grid_for((int64_t(nn) + 3) / 4, kEwBlock, 8);
    if (giant_hint)
      (k_summary<false><<<gs, kEwBlock, 0, st>>>(parent, nn, ctr, giant_bits, out_u, out_v, out_count),
       count_launch());
    else
      (k_summary<true><<<gs, kEwBlock, 0, st>>>(parent, nn, ctr, giant_bits, out_u, out_v, out_count),
       count_launch());
    GC_CHECK_LAUNCH();
  });
}

int gc_shard_absorb(int32_t* parent, int64_t n, const uint32_t* bits, const int64_t* giant_labels,
                    int32_t nranks, int32_t* main_rep, void* ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    require(n >= 0 && n < (int64_t(1) << 31), GC_ERR_MALFORMED, "bad length");
    require(nranks >= 1 && nranks <= kMaxRanks, GC_ERR_ARG, "1..8 ranks supported");
    require(main_rep != nullptr, GC_ERR_ARG, "null representative output");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Arena a(ws, ws_bytes);
    unsigned long long* mat = a.take<unsigned long long>(2);
    int32_t* cls = a.take<int32_t>(kMaxRanks);
    int32_t* rep = a.take<int32_t>(kMaxRanks);
    int32_t* cls_rep = a.take<int32_t>(kMaxRanks);
    int32_t* single = a.take<int32_t>(1);
    const int32_t nn = int32_t(n);
    if (nn == 0) return;
    const int64_t words = (n + 31) / 32;
    // one byte of class bits per local root (general path); its first
    // n/8 bytes double as the one-bit root marks of the single-class path
    uint32_t* mark = a.take<uint32_t>((n + 3) / 4);
    uint32_t* any = a.take<uint32_t>(words);
    GC_CUDA(cudaMemsetAsync(mat, 0, 16, st));
    GC_CUDA(cudaMemsetAsync(mark, 0, size_t((n + 3) / 4) * 4, st));
    // parent is compressed by the preceding gc_shard_summary
    const int gq = grid_for((n + 3) / 4, kEwBlock, 8);
    (k_overlap<<<grid_for(words, kEwBlock, 4), kEwBlock, 0, st>>>(bits, words, nranks, mat), count_launch());
    (k_absorb_classes<<<1, 1, 0, st>>>(mat, giant_labels, nranks, cls, rep, cls_rep, 0, single), count_launch());
    (k_or_bitmaps<<<grid_for(words, kEwBlock, 4), kEwBlock, 0, st>>>(bits, words, nranks, any, single),
     count_launch());
    (k_absorb_mark1<<<gq, kEwBlock, 0, st>>>(parent, nn, any, mark, single), count_launch());
    (k_absorb_mark<<<gq, kEwBlock, 0, st>>>(parent, nn, bits, words, nranks, cls, mark, mat + 1, single),
     count_launch());
    // classes joined through a shared local root (general path only)
    (k_absorb_classes<<<1, 1, 0, st>>>(mat + 1, giant_labels, nranks, cls, rep, cls_rep, 1, nullptr),
     count_launch());
    (k_absorb_apply1<<<gq, kEwBlock, 0, st>>>(parent, nn, mark, any, rep, single), count_launch());
    (k_absorb_apply<<<gq, kEwBlock, 0, st>>>(parent, nn, mark, bits, words, nranks, cls, cls_rep, single),
     count_launch());
    GC_CUDA(cudaMemcpyAsync(main_rep, rep, 4, cudaMemcpyDeviceToDevice, st));  // rank 0's class
    GC_CHECK_LAUNCH();
  });
}

int gc_shard_join(int32_t* parent, int64_t n, const uint32_t* bits, const int64_t* giant_labels, int32_t nranks,
                  const int32_t* us, const int32_t* vs, int64_t k, const gc_spec* spec, void* ws,
                  size_t ws_bytes, void* stream) {
  return guarded([&] {
    require(n >= 0 && n < (int64_t(1) << 31) && k >= 0, GC_ERR_MALFORMED, "bad length");
    require(nranks >= 1 && nranks <= kMaxRanks, GC_ERR_ARG, "1..8 ranks supported");
    require(spec != nullptr && spec->finish >= GC_FINISH_ASYNC && spec->finish <= GC_FINISH_JTB, GC_ERR_CONFIG,
            "join needs a union-find rule");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Arena a(ws, ws_bytes);
    unsigned long long* mat = a.take<unsigned long long>(1);
    int32_t* rep = a.take<int32_t>(kMaxRanks);
    int32_t* single = a.take<int32_t>(1);
    uint32_t* any = a.take<uint32_t>((n + 31) / 32);
    int32_t* aux = nullptr;
    const UFConfig c{spec->finish, spec->find, spec->splice};
    if (c.unite == GC_FINISH_HOOKS || c.unite == GC_FINISH_REM_LOCK) aux = a.take<int32_t>(n);
    const int32_t nn = int32_t(n);
    if (nn == 0) return;
    const int64_t words = (n + 31) / 32;
    GC_CUDA(cudaMemsetAsync(mat, 0, 8, st));
    (k_overlap<<<grid_for(words, kEwBlock, 4), kEwBlock, 0, st>>>(bits, words, nranks, mat), count_launch());
    (k_giant_classes<<<1, 1, 0, st>>>(mat, giant_labels, nranks, rep, single), count_launch());
    (k_or_bitmaps<<<grid_for(words, kEwBlock, 4), kEwBlock, 0, st>>>(bits, words, nranks, any, single),
     count_launch());
    (k_join_init_one<<<grid_for((n + 3) / 4, kEwBlock, 8), kEwBlock, 0, st>>>(parent, nn, any, rep, single),
     count_launch());
    (k_join_init<<<grid_for(nn, kEwBlock, 8), kEwBlock, 0, st>>>(parent, nn, bits, words, nranks, rep, single),
     count_launch());
    GC_CHECK_LAUNCH();
    if (aux) fill(aux, nn, c.unite == GC_FINISH_HOOKS ? nn : 0, st);
    if (k) {
      CooUnionArgs ca{parent, c.unite == GC_FINISH_HOOKS ? aux : nullptr, c.unite == GC_FINISH_REM_LOCK ? aux : nullptr,
                      spec->jtb_ranks, nullptr, nullptr, nn, us, vs, k, nullptr};
      launch_union_coo(c, false, ca, st);
    }
  });
}

}  // extern "C"
