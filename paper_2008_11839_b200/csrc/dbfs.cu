// dbfs.cu — distributed level-synchronous BFS sampling over row-sharded CSR
// (config 5, "BFS becomes a distributed level-synchronous BFS").
//
// The reference BFS (sampling.py:120-172) grows one frontier at a time from
// the probe source; a vertex reached at a level takes as parent its smallest
// frontier neighbour (the first discoverer in the ascending frontier), the
// reached set takes its minimum id, and the inspections are the frontier
// degree sums.  Sharded, every rank owns the rows [lo, hi) of the symmetric
// CSR and keeps the frontier F and the visited set V as replicated n-bit
// bitmaps.  A vertex's row lists all its neighbours, so the OWNER of x can
// decide x's parent alone: the first frontier vertex of x's ascending row —
// the same minimum as the single-GPU BFS.  One level:
//   * top-down (narrow frontiers): gc_dbfs_marks sets a mark bit for every
//     unvisited neighbour of the block's frontier rows and lists them; the
//     lists are all-gathered and merged (gc_dbfs_merge_marks), so every rank
//     holds the marks of all ranks; gc_dbfs_claim then lets each owner pull
//     the parent of its marked vertices;
//   * bottom-up (wide frontiers): gc_dbfs_claim with no marks scans every
//     unvisited owned row for its first frontier neighbour.
// The claimed bits of one rank lie in its own rows, so the next frontier is
// the all-reduce SUM of the ranks' next-bitmaps (disjoint bits: the sum is
// the OR), after which gc_dbfs_advance folds it into V and counts it.
// gc_dbfs_finish writes the labels (replicated), the block's tree edges
// (parent, v) and the degree sum of the block's reached rows (the reference
// counter summed over ranks).
#include <climits>
#include <cub/cub.cuh>

#include "internal.h"
#include "pipeline.cuh"

namespace gc {

namespace {

constexpr int kDB = 256;
constexpr uint32_t kNoParent = 0xffffffffu;

__device__ __forceinline__ bool bit(const uint32_t* b, int64_t x) { return (__ldg(b + (x >> 5)) >> (x & 31)) & 1u; }

__global__ void k_dbfs_init(uint32_t* F, uint32_t* V, uint32_t* par, int64_t s) {
  F[s >> 5] |= 1u << (s & 31);
  V[s >> 5] |= 1u << (s & 31);
  par[s] = kNoParent - 1;  // the source
}

// marks: unvisited neighbours of the block's frontier rows (red.or, no
// result needed).  A warp scans 32 frontier words per step and walks only
// the words with set bits (narrow top-down levels touch a sliver of the
// rows: scanning every row's bit cost ~0.3 ms per level at 2^27); a row
// with more than 32 entries is walked by the whole warp.
__device__ __forceinline__ uint32_t range_mask(int64_t w, int64_t lo, int64_t hi) {
  uint32_t m = ~0u;
  if (w == (lo >> 5)) m &= ~0u << (lo & 31);
  if (w == ((hi - 1) >> 5) && (hi & 31)) m &= (1u << (hi & 31)) - 1u;
  return m;
}

__global__ void __launch_bounds__(kDB)
k_dbfs_marks(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, int64_t lo, int64_t hi,
             const uint32_t* __restrict__ F, const uint32_t* __restrict__ V, uint32_t* M) {
  const int lane = threadIdx.x & 31;
  const int64_t w_lo = lo >> 5, w_hi = (hi + 31) >> 5;
  const int64_t gw = (int64_t(blockIdx.x) * kDB + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * kDB) >> 5;
  for (int64_t w0 = w_lo + gw * 32; w0 < w_hi; w0 += nw * 32) {
    const int64_t wl = w0 + lane;
    const uint32_t fw = wl < w_hi ? __ldg(F + wl) & range_mask(wl, lo, hi) : 0u;
    unsigned todo = __ballot_sync(0xffffffffu, fw != 0u);
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint32_t word = __shfl_sync(0xffffffffu, fw, src);
      const int64_t f = (w0 + src) * 32 + lane;
      int64_t b = 0, d = 0;
      if ((word >> lane) & 1u) {
        b = off[f];
        d = off[f + 1] - b;
      }
      const bool big = d > 32;
      if (!big)
        for (int64_t j = 0; j < d; ++j) {
          const int32_t x = tgt[b + j];
          if (!bit(V, x))
            asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(M + (x >> 5)), "r"(1u << (x & 31)) : "memory");
        }
      unsigned mask = __ballot_sync(0xffffffffu, big);
      while (mask) {
        const int s2 = __ffs(mask) - 1;
        mask &= mask - 1;
        const int64_t bb = __shfl_sync(0xffffffffu, b, s2);
        const int64_t dd = __shfl_sync(0xffffffffu, d, s2);
        for (int64_t j = lane; j < dd; j += 32) {
          const int32_t x = tgt[bb + j];
          if (!bit(V, x))
            asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(M + (x >> 5)), "r"(1u << (x & 31)) : "memory");
        }
      }
    }
  }
}

// bitmap -> ascending id list (block-scanned, one cursor atomic per block step)
__global__ void __launch_bounds__(kDB)
k_dbfs_list(const uint32_t* __restrict__ M, int64_t words, int32_t* out, unsigned long long* cnt) {
  using Scan = cub::BlockScan<int, kDB>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long base;
  for (int64_t w0 = int64_t(blockIdx.x) * kDB; w0 < words; w0 += int64_t(gridDim.x) * kDB) {
    const int64_t w = w0 + threadIdx.x;
    uint32_t word = w < words ? M[w] : 0u;
    int rank, total;
    Scan(tmp).ExclusiveSum(__popc(word), rank, total);
    if (threadIdx.x == 0) base = total ? atomicAdd(cnt, static_cast<unsigned long long>(total)) : 0ull;
    __syncthreads();
    unsigned long long p = base + rank;
    while (word) {
      const int b = __ffs(word) - 1;
      word &= word - 1;
      out[p++] = int32_t(w * 32 + b);
    }
    __syncthreads();
  }
}

__global__ void k_dbfs_merge(const int32_t* ids, int64_t k, int64_t n, uint32_t* M, unsigned int* bad) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < k; i += stride) {
    const int32_t x = ids[i];
    if (x < 0 || x >= n) {
      atomicOr(bad, 1u);
      continue;
    }
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(M + (x >> 5)), "r"(1u << (x & 31)) : "memory");
  }
}

// claim: a warp scans 32 words of the block's rows per step and walks the
// words holding candidates — unvisited vertices that are marked (top-down)
// or any unvisited vertex (bottom-up); a candidate takes the first frontier
// vertex of its row (the reference's smallest-discoverer rule)
__global__ void __launch_bounds__(kDB)
k_dbfs_claim(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, int64_t lo, int64_t hi,
             const uint32_t* __restrict__ F, const uint32_t* __restrict__ V, const uint32_t* __restrict__ M,
             uint32_t* par, uint32_t* N, unsigned long long* cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t w_lo = lo >> 5, w_hi = (hi + 31) >> 5;
  const int64_t gw = (int64_t(blockIdx.x) * kDB + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * kDB) >> 5;
  unsigned long long c = 0;
  for (int64_t w0 = w_lo + gw * 32; w0 < w_hi; w0 += nw * 32) {
    const int64_t wl = w0 + lane;
    uint32_t cand = 0u;
    if (wl < w_hi) cand = ~__ldg(V + wl) & (M ? __ldg(M + wl) : ~0u) & range_mask(wl, lo, hi);
    unsigned todo = __ballot_sync(0xffffffffu, cand != 0u);
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint32_t word = __shfl_sync(0xffffffffu, cand, src);
      const int64_t x = (w0 + src) * 32 + lane;
      bool found = false;
      if ((word >> lane) & 1u) {
        const int64_t b = off[x], e = off[x + 1];
        for (int64_t j = b; j < e; ++j) {
          const int32_t t = tgt[j];
          if (bit(F, t)) {
            par[x] = uint32_t(t);
            found = true;
            break;
          }
        }
      }
      const uint32_t got = __ballot_sync(0xffffffffu, found);
      if (lane == 0 && got) {
        N[w0 + src] = got;
        c += __popc(got);
      }
    }
  }
  block_add<kDB>(cnt, c);
}

// V |= N, F = N (separate buffers: F is overwritten), popcount(N)
__global__ void __launch_bounds__(kDB)
k_dbfs_advance(uint32_t* V, uint32_t* F, const uint32_t* N, int64_t words, unsigned long long* cnt) {
  unsigned long long c = 0;
  const int64_t stride = int64_t(gridDim.x) * kDB;
  for (int64_t w = int64_t(blockIdx.x) * kDB + threadIdx.x; w < words; w += stride) {
    const uint32_t x = N[w];
    F[w] = x;
    if (x) {
      V[w] |= x;
      c += __popc(x);
    }
  }
  block_add<kDB>(cnt, c);
}

__global__ void k_dbfs_min(const uint32_t* V, int64_t words, int32_t* mn) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int32_t best = INT_MAX;
  for (int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < words; w += stride) {
    const uint32_t x = V[w];
    if (x) {
      best = int32_t(w * 32 + __ffs(x) - 1);
      break;  // words ascend along this thread's stride
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const int32_t t = __shfl_xor_sync(0xffffffffu, best, o);
    best = t < best ? t : best;
  }
  if ((threadIdx.x & 31) == 0 && best != INT_MAX) atomicMin(mn, best);
}

// labels (every vertex), the block's tree edges and reached-row degree sum
__global__ void __launch_bounds__(kDB)
k_dbfs_finish(const int64_t* __restrict__ off, int64_t n, int64_t lo, int64_t hi, const uint32_t* __restrict__ V,
              const uint32_t* __restrict__ par, const int32_t* mn_p, int32_t* P, int32_t* fu, int32_t* fv,
              unsigned long long* fcnt, unsigned long long* insp) {
  // eight vertices per thread per step and one cursor atomic per block step
  // (a per-warp atomic on the one cursor serialised ~4M appends at 2^27)
  constexpr int kJ = 8;
  using Scan = cub::BlockScan<int, kDB>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long base;
  const int32_t mn = *mn_p;
  unsigned long long degs = 0;
  const int64_t step = int64_t(kDB) * kJ;
  for (int64_t b0 = int64_t(blockIdx.x) * step; b0 < n; b0 += int64_t(gridDim.x) * step) {
    uint32_t p[kJ];
    int c = 0;
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int64_t v = b0 + int64_t(j) * kDB + threadIdx.x;
      p[j] = kNoParent;
      if (v < n) {
        const bool r = bit(V, v);
        P[v] = r ? mn : int32_t(v);
        if (r && v >= lo && v < hi) {
          degs += static_cast<unsigned long long>(off[v + 1] - off[v]);
          p[j] = par[v];
          c += p[j] < kNoParent - 1;
        }
      }
    }
    int rank, total;
    Scan(tmp).ExclusiveSum(c, rank, total);
    if (threadIdx.x == 0) base = total ? atomicAdd(fcnt, static_cast<unsigned long long>(total)) : 0ull;
    __syncthreads();
    unsigned long long i = base + rank;
#pragma unroll
    for (int j = 0; j < kJ; ++j)
      if (p[j] < kNoParent - 1) {
        fu[i] = int32_t(p[j]);
        fv[i] = int32_t(b0 + int64_t(j) * kDB + threadIdx.x);
        ++i;
      }
    __syncthreads();
  }
  block_add<kDB>(insp, degs);
}

int gdb(int64_t work) { return grid_for(work, kDB, 8); }

void check_block(const gc_csr* g, int64_t lo, int64_t hi) {
  require(g != nullptr && g->n >= 0 && g->n < (int64_t(1) << 31), GC_ERR_MALFORMED, "bad graph");
  require(lo >= 0 && lo <= hi && hi <= g->n, GC_ERR_ARG, "row block outside [0, n]");
}

}  // namespace

}  // namespace gc

using namespace gc;

extern "C" {

int gc_dbfs_init(int64_t n, int64_t source, uint32_t* frontier, uint32_t* visited, uint32_t* parent,
                 void* stream) {
  return guarded([&] {
    require(n >= 0 && n < (int64_t(1) << 31), GC_ERR_MALFORMED, "bad length");
    require(source >= 0 && source < n, GC_ERR_ARG, "BFS source outside [0, n)");
    require(frontier && visited && parent, GC_ERR_ARG, "null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t words = (n + 31) / 32;
    GC_CUDA(cudaMemsetAsync(frontier, 0, words * 4, st));
    GC_CUDA(cudaMemsetAsync(visited, 0, words * 4, st));
    GC_CUDA(cudaMemsetAsync(parent, 0xff, n * 4, st));
    (k_dbfs_init<<<1, 1, 0, st>>>(frontier, visited, parent, source), count_launch());
    GC_CHECK_LAUNCH();
  });
}

int gc_dbfs_marks(const gc_csr* g, int64_t row_lo, int64_t row_hi, const uint32_t* frontier,
                  const uint32_t* visited, uint32_t* marks, int32_t* out_ids, unsigned long long* out_count,
                  void* stream) {
  return guarded([&] {
    check_block(g, row_lo, row_hi);
    require(frontier && visited && marks && out_ids && out_count, GC_ERR_ARG, "null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t words = (g->n + 31) / 32;
    GC_CUDA(cudaMemsetAsync(marks, 0, words * 4, st));
    GC_CUDA(cudaMemsetAsync(out_count, 0, 8, st));
    if (row_hi > row_lo)
      (k_dbfs_marks<<<gdb(row_hi - row_lo), kDB, 0, st>>>(g->offsets, g->targets, row_lo, row_hi, frontier, visited,
                                                          marks), count_launch());
    if (words) (k_dbfs_list<<<gdb(words), kDB, 0, st>>>(marks, words, out_ids, out_count), count_launch());
    GC_CHECK_LAUNCH();
  });
}

int gc_dbfs_merge_marks(int64_t n, const int32_t* ids, int64_t k, uint32_t* marks, unsigned int* bad,
                        void* stream) {
  return guarded([&] {
    require(k >= 0 && (k == 0 || (ids && marks && bad)), GC_ERR_ARG, "null argument");
    if (k == 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    (k_dbfs_merge<<<grid_for(k, 256, 8), 256, 0, st>>>(ids, k, n, marks, bad), count_launch());
    GC_CHECK_LAUNCH();
  });
}

int gc_dbfs_claim(const gc_csr* g, int64_t row_lo, int64_t row_hi, const uint32_t* frontier,
                  const uint32_t* visited, const uint32_t* marks, uint32_t* parent, uint32_t* next,
                  unsigned long long* count, void* stream) {
  return guarded([&] {
    check_block(g, row_lo, row_hi);
    require(frontier && visited && parent && next && count, GC_ERR_ARG, "null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t words = (g->n + 31) / 32;
    GC_CUDA(cudaMemsetAsync(next, 0, words * 4, st));
    GC_CUDA(cudaMemsetAsync(count, 0, 8, st));
    const int64_t w_lo = row_lo >> 5, w_hi = (row_hi + 31) >> 5;
    if (w_hi > w_lo)
      (k_dbfs_claim<<<gdb((w_hi - w_lo) * 32), kDB, 0, st>>>(g->offsets, g->targets, row_lo, row_hi, frontier,
                                                             visited, marks, parent, next, count), count_launch());
    GC_CHECK_LAUNCH();
  });
}

int gc_dbfs_merge_claim(const gc_csr* g, int64_t row_lo, int64_t row_hi, const uint32_t* frontier,
                        const uint32_t* visited, uint32_t* marks, const int32_t* ids, int64_t k, unsigned int* bad,
                        uint32_t* parent, uint32_t* next, unsigned long long* count, void* stream) {
  const int rc = gc_dbfs_merge_marks(g ? g->n : 0, ids, k, marks, bad, stream);
  if (rc != GC_OK) return rc;
  return gc_dbfs_claim(g, row_lo, row_hi, frontier, visited, marks, parent, next, count, stream);
}

int gc_dbfs_advance(int64_t n, uint32_t* visited, uint32_t* frontier, const uint32_t* next,
                    unsigned long long* count, void* stream) {
  return guarded([&] {
    require(visited && frontier && next && count, GC_ERR_ARG, "null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t words = (n + 31) / 32;
    GC_CUDA(cudaMemsetAsync(count, 0, 8, st));
    if (words) (k_dbfs_advance<<<gdb(words), kDB, 0, st>>>(visited, frontier, next, words, count), count_launch());
    GC_CHECK_LAUNCH();
  });
}

int gc_dbfs_finish(const gc_csr* g, int64_t row_lo, int64_t row_hi, const uint32_t* visited,
                   const uint32_t* parent, int32_t* labels, int32_t* out_u, int32_t* out_v,
                   unsigned long long* out_count, unsigned long long* insp, void* ws, size_t ws_bytes,
                   void* stream) {
  return guarded([&] {
    check_block(g, row_lo, row_hi);
    require(visited && parent && labels && out_u && out_v && out_count && insp, GC_ERR_ARG, "null argument");
    require(ws && ws_bytes >= 16, GC_ERR_OOM, "workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t n = g->n, words = (n + 31) / 32;
    int32_t* mn = static_cast<int32_t*>(ws);
    fill(mn, 1, INT_MAX, st);
    GC_CUDA(cudaMemsetAsync(out_count, 0, 8, st));
    GC_CUDA(cudaMemsetAsync(insp, 0, 8, st));
    if (words) (k_dbfs_min<<<gdb(words), kDB, 0, st>>>(visited, words, mn), count_launch());
    if (n)
      (k_dbfs_finish<<<gdb(n), kDB, 0, st>>>(g->offsets, n, row_lo, row_hi, visited, parent, mn, labels, out_u, out_v,
                                             out_count, insp), count_launch());
    GC_CHECK_LAUNCH();
  });
}

}  // extern "C"
