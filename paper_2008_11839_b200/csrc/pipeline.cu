// pipeline.cu — elementwise phases of the two-phase pipeline
// (driver.py:454-500): set initialisation, compression, most-frequent label,
// active gather, finalisation and canonical relabelling.
#include <atomic>

#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <cstdlib>

#include "pipeline.cuh"

namespace gc {

namespace cg = cooperative_groups;

__global__ void k_init_sets(int32_t* P, int32_t* H, int32_t* L, int32_t n, unsigned long long* stamps,
                            unsigned stamp_mask) {
  entry_stamp(stamps, stamp_mask);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  if (!H && !L && (reinterpret_cast<uintptr_t>(P) & 15) == 0) {
    // 16-byte stores, four vertices per thread
    const int64_t nq = int64_t(n) / 4;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nq; q += stride) {
      const int32_t v = int32_t(4 * q);
      reinterpret_cast<int4*>(P)[q] = make_int4(v, v + 1, v + 2, v + 3);
    }
    for (int64_t v = 4 * nq + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
      P[v] = int32_t(v);
    return;
  }
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    P[v] = int32_t(v);
    if (H) H[v] = n;
    if (L) L[v] = 0;
  }
}

__device__ __forceinline__ int32_t root_weak(const int32_t* P, int32_t x) {
  int32_t y;
  while ((y = ld_weak(P + x)) != x) x = y;
  return x;
}

__global__ void k_compress(int32_t* P, int32_t n) {
  // four vertices per thread; the first hop of the four walks is issued
  // together and only parents that moved keep walking
  const bool aligned = (reinterpret_cast<uintptr_t>(P) & 15) == 0;
  const int64_t nq = (int64_t(n) + 3) / 4;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nq; q += stride) {
    const int64_t v0 = 4 * q;
    int32_t p[4];
    if (aligned && v0 + 3 < n) {
      const int4 p4 = *reinterpret_cast<const int4*>(P + v0);
      p[0] = p4.x; p[1] = p4.y; p[2] = p4.z; p[3] = p4.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) p[j] = v0 + j < n ? ld_weak(P + v0 + j) : int32_t(v0 + j);
    }
    int32_t hop[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) hop[j] = (v0 + j < n && p[j] != int32_t(v0 + j)) ? ld_free(P + p[j]) : p[j];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (v0 + j >= n || hop[j] == p[j]) continue;  // a root, or already points at its root
      const int32_t r = root_weak(P, hop[j]);
      P[v0 + j] = r;
    }
  }
}

// Fused post-sampling pass (sampling.py:38-47 compress_all, :29-35 count of
// the probe's candidate, driver.py:473 active gather): each thread owns 4
// consecutive vertices (one 16-byte load), resolves their roots with
// L1-cacheable loads (the union kernel has finished: parents only shrink
// toward roots from here), writes them back, counts the candidate label and
// appends the vertices not carrying it to the active list with one global
// atomic per block.  If the candidate turns out not to be the mode, the
// histogram fallback re-gathers (k_gather_active).
#ifndef GC_PS_BLOCKS
#define GC_PS_BLOCKS 6  // resident 256-thread blocks per SM of k_post_sample (one wave)
#endif
template <bool COMPRESS>
__global__ void __launch_bounds__(kEwBlock, GC_PS_BLOCKS)
k_post_sample(int32_t* P, int32_t n, const int64_t* off, int32_t* list, unsigned long long* ctr) {
  // two 4-vertex quads per thread per step (eight first hops in flight; the
  // step's barriers are paid once per eight vertices)
  constexpr int kQ = 2;
  using Scan = cub::BlockScan<int, kEwBlock>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long base;
  const int32_t cand = int32_t(ctr[C_CAND]);
  unsigned long long ccount = 0, degsum = 0;
  const int64_t nq = (int64_t(n) + 3) / 4;
  for (int64_t q0 = int64_t(blockIdx.x) * kEwBlock * kQ; q0 < nq; q0 += int64_t(gridDim.x) * kEwBlock * kQ) {
    int32_t lab[kQ][4];
    int64_t v0[kQ];
#pragma unroll
    for (int h = 0; h < kQ; ++h) {
      const int64_t q = q0 + int64_t(h) * kEwBlock + threadIdx.x;
      v0[h] = q * 4;
#pragma unroll
      for (int j = 0; j < 4; ++j) lab[h][j] = cand;
      if (q < nq) {
        if (v0[h] + 3 < n) {
          const int4 p4 = *reinterpret_cast<const int4*>(P + v0[h]);
          lab[h][0] = p4.x; lab[h][1] = p4.y; lab[h][2] = p4.z; lab[h][3] = p4.w;
        } else {
          for (int j = 0; j < 4; ++j) if (v0[h] + j < n) lab[h][j] = P[v0[h] + j];
        }
      }
    }
    if (COMPRESS) {
      // first hop of all eight walks issued together (most labels are
      // already roots after the union kernel's halving); only labels that
      // moved continue walking
      int32_t hop[kQ][4];
#pragma unroll
      for (int h = 0; h < kQ; ++h)
#pragma unroll
        for (int j = 0; j < 4; ++j) hop[h][j] = v0[h] + j < n ? ld_free(P + lab[h][j]) : lab[h][j];
#pragma unroll
      for (int h = 0; h < kQ; ++h) {
        if (v0[h] >= n) continue;
        bool dirty = false;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (v0[h] + j >= n) continue;
          const int32_t r = hop[h][j] == lab[h][j] ? lab[h][j] : root_weak(P, hop[h][j]);
          dirty |= r != lab[h][j];
          lab[h][j] = r;
        }
        if (dirty) {
          if (v0[h] + 3 < n)
            *reinterpret_cast<int4*>(P + v0[h]) = make_int4(lab[h][0], lab[h][1], lab[h][2], lab[h][3]);
          else
            for (int j = 0; j < 4; ++j) if (v0[h] + j < n) P[v0[h] + j] = lab[h][j];
        }
      }
    }
    int act = 0;
#pragma unroll
    for (int h = 0; h < kQ; ++h)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (v0[h] + j >= n) continue;
        ccount += lab[h][j] == cand;
        act += lab[h][j] != cand;
      }
    int rank, total;
    Scan(tmp).ExclusiveSum(act, rank, total);
    if (threadIdx.x == 0) base = total ? atomicAdd(ctr + C_N_ACTIVE, static_cast<unsigned long long>(total)) : 0ull;
    __syncthreads();
    if (act) {
      unsigned long long pos = base + rank;
#pragma unroll
      for (int h = 0; h < kQ; ++h)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (v0[h] + j < n && lab[h][j] != cand) {
            list[pos++] = int32_t(v0[h] + j);
            degsum += static_cast<unsigned long long>(off[v0[h] + j + 1] - off[v0[h] + j]);
          }
        }
    }
    __syncthreads();
  }
  block_add<kEwBlock>(ctr + C_CAND_COUNT, ccount);
  block_add<kEwBlock>(ctr + C_INSP_FINISH, degsum);
}

constexpr int kProbe = 1024;

// walk = 1: P is a parent forest and each sample is resolved to its root
// (the probe runs before compression); walk = 0: P is a plain label array
// (the census of arbitrary labels, which need not be a forest — a label
// cycle would never end the walk)
__global__ void __launch_bounds__(kProbe) k_mode_probe(const int32_t* P, int32_t n,
                                                       unsigned long long* ctr, int walk, unsigned stamp_mask) {
  entry_stamp(ctr + C_STAMP0, stamp_mask);
  // sample labels counted in a shared-memory hash table (open addressing,
  // warp-aggregated adds: the dominant label is one add per warp)
  constexpr int kSlots = 2 * kProbe;
  __shared__ int32_t key_[kSlots];
  __shared__ unsigned cnt_[kSlots];
  __shared__ unsigned long long best;
  const int s = n < kProbe ? n : kProbe;
  const int i = threadIdx.x;
  for (int k = i; k < kSlots; k += kProbe) {
    key_[k] = -1;
    cnt_[k] = 0;
  }
  if (i == 0) best = 0ull;
  int32_t x = -1;
  if (i < s) {
    // walk to the root so the probe can run before compression
    x = ld_weak(P + (int64_t(i) * n) / s);
    int32_t y;
    if (walk)
      while ((y = ld_weak(P + x)) != x) x = y;
  }
  __syncthreads();
  int slot = -1;
  if (i < s) {
    const unsigned same = __match_any_sync(__activemask(), x);
    // multiplicative hash, high bits (the samples are evenly spaced ids, so
    // the low bits of x * K can all coincide)
    slot = int((uint32_t(x) * 2654435761u) >> (32 - 11));
    while (true) {
      const int32_t k = atomicCAS(&key_[slot], -1, x);
      if (k == -1 || k == x) break;
      slot = (slot + 1) % kSlots;
    }
    if ((i & 31) == __ffs(int(same)) - 1) atomicAdd(&cnt_[slot], __popc(same));
  }
  __syncthreads();
  if (i < s) {
    const unsigned long long key =
        (static_cast<unsigned long long>(cnt_[slot]) << 32) | (0xffffffffull - uint32_t(x));
    atomicMax(&best, key);
  }
  __syncthreads();
  if (i == 0) {
    ctr[C_CAND] = s ? (0xffffffffull - (best & 0xffffffffull)) : 0ull;
    ctr[C_CAND_COUNT] = 0;
  }
}

__global__ void k_count_eq(const int32_t* P, int32_t n, unsigned long long* ctr) {
  const int32_t cand = int32_t(ctr[C_CAND]);
  unsigned long long c = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    c += P[v] == cand;
  block_add<kEwBlock>(ctr + C_CAND_COUNT, c);
}

// the candidate is the mode: a strict majority, or a sampler that counted
// its classes exactly (C_MODE_EXACT)
__device__ __forceinline__ bool majority(const unsigned long long* ctr, int32_t n) {
  return ctr[C_MODE_EXACT] != 0 || 2ull * ctr[C_CAND_COUNT] > static_cast<unsigned long long>(n);
}

__device__ __forceinline__ void hist_zero_body(int32_t* hist, int32_t n, unsigned long long* ctr) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) hist[v] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctr[C_SCRATCH0] = 0;
    ctr[C_N_ACTIVE] = 0;      // the optimistic gather used a non-mode candidate
    ctr[C_INSP_FINISH] = 0;
  }
}

__global__ void k_hist_zero(int32_t* hist, int32_t n, unsigned long long* ctr) {
  if (majority(ctr, n)) return;
  hist_zero_body(hist, n, ctr);
}

__device__ __forceinline__ void hist_add_body(const int32_t* P, int32_t* hist, int32_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
    const int64_t v = base + threadIdx.x;
    const bool ok = v < n;
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    if (!ok) continue;
    const int32_t lab = P[v];
    // warp aggregation: one atomic per distinct label in the warp
    const unsigned same = __match_any_sync(act, lab);
    const int leader = __ffs(same) - 1;
    if ((threadIdx.x & 31) == leader) atomicAdd(hist + lab, __popc(same));
  }
}

__global__ void k_hist_add(const int32_t* P, int32_t* hist, int32_t n, unsigned long long* ctr) {
  if (majority(ctr, n)) return;
  hist_add_body(P, hist, n);
}

__device__ __forceinline__ void hist_argmax_body(const int32_t* hist, int32_t n, unsigned long long* ctr) {
  __shared__ unsigned long long best;
  if (threadIdx.x == 0) best = 0ull;
  __syncthreads();
  unsigned long long mine = 0ull;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const unsigned long long key = (static_cast<unsigned long long>(uint32_t(hist[v])) << 32) |
                                   (0xffffffffull - uint64_t(v));
    mine = key > mine ? key : mine;
  }
  atomicMax(&best, mine);
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(ctr + C_SCRATCH0, best);
}

__global__ void k_hist_argmax(const int32_t* hist, int32_t n, unsigned long long* ctr) {
  if (majority(ctr, n)) return;
  hist_argmax_body(hist, n, ctr);
}

__device__ __forceinline__ void mode_finish_body(int32_t n, unsigned long long* ctr) {
  if (n == 0) {
    ctr[C_LMAX] = 0;
    ctr[C_LMAX_COUNT] = 0;
  } else if (majority(ctr, n)) {
    ctr[C_LMAX] = ctr[C_CAND];
    ctr[C_LMAX_COUNT] = ctr[C_CAND_COUNT];
  } else {
    const unsigned long long k = ctr[C_SCRATCH0];
    ctr[C_LMAX] = 0xffffffffull - (k & 0xffffffffull);
    ctr[C_LMAX_COUNT] = k >> 32;
  }
}

__global__ void k_mode_finish(int32_t n, unsigned long long* ctr) { mode_finish_body(n, ctr); }

__device__ __forceinline__ void gather_active_body(const int32_t* P, int32_t n, const int64_t* off, int32_t* list,
                                                   unsigned long long* ctr) {
  // four vertices per thread (one 16-byte label load), one scan and one
  // global atomic per 1024 vertices
  using Scan = cub::BlockScan<int, kEwBlock>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long base;
  const int32_t lmax = int32_t(ctr[C_LMAX]);
  const bool aligned = (reinterpret_cast<uintptr_t>(P) & 15) == 0;
  unsigned long long degsum = 0;
  const int64_t nq = (int64_t(n) + 3) / 4;
  for (int64_t q0 = int64_t(blockIdx.x) * kEwBlock; q0 < nq; q0 += int64_t(gridDim.x) * kEwBlock) {
    const int64_t q = q0 + threadIdx.x;
    const int64_t v0 = q * 4;
    int32_t lab[4] = {lmax, lmax, lmax, lmax};
    if (q < nq) {
      if (aligned && v0 + 3 < n) {
        const int4 p4 = *reinterpret_cast<const int4*>(P + v0);
        lab[0] = p4.x; lab[1] = p4.y; lab[2] = p4.z; lab[3] = p4.w;
      } else {
        for (int j = 0; j < 4; ++j) if (v0 + j < n) lab[j] = P[v0 + j];
      }
    }
    int act = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) act += lab[j] != lmax;
    int rank, total;
    Scan(tmp).ExclusiveSum(act, rank, total);
    if (threadIdx.x == 0) base = total ? atomicAdd(ctr + C_N_ACTIVE, static_cast<unsigned long long>(total)) : 0ull;
    __syncthreads();
    if (act) {
      unsigned long long pos = base + rank;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (lab[j] != lmax) {
          list[pos++] = int32_t(v0 + j);
          degsum += static_cast<unsigned long long>(off[v0 + j + 1] - off[v0 + j]);
        }
      }
    }
    __syncthreads();
  }
  block_add<kEwBlock>(ctr + C_INSP_FINISH, degsum);
}

__global__ void __launch_bounds__(kEwBlock)
k_gather_active(const int32_t* P, int32_t n, const int64_t* off, int32_t* list,
                unsigned long long* ctr, int only_fallback) {
  if (only_fallback && majority(ctr, n)) return;
  gather_active_body(P, n, off, list, ctr);
}

// The exact-mode fallback of the post-sampling pass as ONE cooperative
// launch (histogram zero -> add -> arg-max -> L_max -> active re-gather,
// grid barriers between): on a strict majority of the probe's candidate —
// the usual case — it only publishes L_max and exits, one launch instead of
// five early-exit launches per pipeline.
__global__ void __launch_bounds__(kEwBlock)
k_mode_fallback(const int32_t* P, int32_t* hist, int32_t n, const int64_t* off, int32_t* list,
                unsigned long long* ctr) {
  if (majority(ctr, n)) {  // the same decision in every block (C_CAND_COUNT is final)
    if (blockIdx.x == 0 && threadIdx.x == 0) mode_finish_body(n, ctr);
    return;
  }
  cg::grid_group grid = cg::this_grid();
  hist_zero_body(hist, n, ctr);
  grid.sync();
  hist_add_body(P, hist, n);
  grid.sync();
  hist_argmax_body(hist, n, ctr);
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) mode_finish_body(n, ctr);
  grid.sync();
  gather_active_body(P, n, off, list, ctr);
}

// Finalize over the active list alone (union-find finishes after a
// sampler, driver.py:483-490): the finish links only trees outside L_max,
// so while L_max is still a root every vertex labelled L_max is final and
// only the active vertices can have moved.  Components = the list's roots
// + L_max.  When the finish linked L_max itself (under a smaller root),
// this kernel does nothing and the whole-array kernel after it runs.
__global__ void __launch_bounds__(kEwBlock)
k_finalize_list(int32_t* P, int32_t n, const int32_t* __restrict__ list, unsigned long long* ctr,
                unsigned stamp_mask) {
  entry_stamp(ctr + C_STAMP0, stamp_mask);
  const int32_t lmax = int32_t(ctr[C_LMAX]);
  if (ld_acq(P + lmax) != lmax) return;
  const int64_t cnt = int64_t(ctr[C_N_ACTIVE]);
  unsigned long long roots = (blockIdx.x == 0 && threadIdx.x == 0) ? 1ull : 0ull;  // L_max
  bool noncanon = false, cyc = false;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt; i += stride) {
    const int32_t v = __ldg(list + i);
    const int32_t lab = ld_weak(P + v);
    if (lab == v) {
      ++roots;
      continue;
    }
    int32_t r = lab, y;
    int64_t steps = 0;
    while ((y = ld_weak(P + r)) != r) {
      r = y;
      if (++steps > n) { cyc = true; break; }
    }
    if (r != lab) P[v] = r;
    noncanon |= r > v;
  }
  block_add<kEwBlock>(ctr + C_COMPONENTS, roots);
  if (__syncthreads_or(noncanon) && threadIdx.x == 0) ctr[C_NONCANON] = 1;
  if (cyc) ctr[C_CYCLE] = 1;
}

// list_mode: k_finalize_list ran first; skip when L_max stayed a root
__device__ __forceinline__ bool list_done(const int32_t* P, const unsigned long long* ctr, int list_mode) {
  if (!list_mode) return false;
  const int32_t lmax = int32_t(ctr[C_LMAX]);
  return ld_acq(P + lmax) == lmax;
}

__global__ void k_finalize(int32_t* P, int32_t n, unsigned long long* ctr, unsigned stamp_mask, int list_mode) {
  entry_stamp(ctr + C_STAMP0, stamp_mask);
  if (list_done(P, ctr, list_mode)) return;
  unsigned long long roots = 0;
  bool noncanon = false, cyc = false;
  const int64_t nq = (int64_t(n) + 3) / 4;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nq; q += stride) {
    const int64_t v0 = q * 4;
    int32_t lab[4];
    const bool full = v0 + 3 < n;
    if (full) {
      const int4 p4 = *reinterpret_cast<const int4*>(P + v0);
      lab[0] = p4.x; lab[1] = p4.y; lab[2] = p4.z; lab[3] = p4.w;
    } else {
      for (int j = 0; j < 4; ++j) lab[j] = v0 + j < n ? P[v0 + j] : int32_t(v0 + j);
    }
    bool dirty = false;
    // first hop of the four walks issued together (labels are mostly
    // compressed already); only labels whose parent moved keep walking
    int32_t hop[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int32_t v = int32_t(v0 + j);
      hop[j] = (v < n && lab[j] != v) ? ld_free(P + lab[j]) : lab[j];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int32_t v = int32_t(v0 + j);
      if (v >= n) continue;
      int32_t r = lab[j];
      if (r == v) {
        ++roots;
        continue;
      }
      if (hop[j] == r) {
        noncanon |= r > v;
        continue;  // already points at its root
      }
      r = hop[j];
      dirty = true;
      int64_t steps = 0;
      int32_t y;
      while ((y = ld_weak(P + r)) != r) {
        r = y;
        if (++steps > n) { cyc = true; break; }
      }
      dirty |= r != lab[j];
      lab[j] = r;
      noncanon |= r > v;
    }
    if (dirty) {
      if (full) *reinterpret_cast<int4*>(P + v0) = make_int4(lab[0], lab[1], lab[2], lab[3]);
      else for (int j = 0; j < 4; ++j) if (v0 + j < n) P[v0 + j] = lab[j];
    }
  }
  block_add<kEwBlock>(ctr + C_COMPONENTS, roots);
  if (__syncthreads_or(noncanon) && threadIdx.x == 0) ctr[C_NONCANON] = 1;
  if (cyc) ctr[C_CYCLE] = 1;
}

// k_finalize with its tiles staged by the TMA engine: 4096 labels (16 KB)
// per tile, two stages per block; thread 0 issues the bulk copies, every
// thread then takes four quads of the tile from shared memory.  Same
// per-vertex work as k_finalize (which handles the < 4-label tail).
constexpr int kFinTile = 4096;
constexpr int kFinStages = 2;

__global__ void __launch_bounds__(kEwBlock)
k_finalize_tma(int32_t* P, int32_t n, unsigned long long* ctr, unsigned stamp_mask, int list_mode) {
  entry_stamp(ctr + C_STAMP0, stamp_mask);
  if (list_done(P, ctr, list_mode)) return;
  __shared__ alignas(128) int32_t buf[kFinStages][kFinTile];
  __shared__ alignas(8) uint64_t bar[kFinStages];
  const int64_t n4 = (int64_t(n) / 4) * 4;  // bulk-copied part (16-byte multiple)
  const int64_t tiles = (n4 + kFinTile - 1) / kFinTile;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kFinStages; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int64_t t, int s) {
    const int64_t lo = t * kFinTile;
    const int64_t cnt = n4 - lo < kFinTile ? n4 - lo : kFinTile;
    mbar_expect_tx(&bar[s], uint32_t(cnt * 4));
    bulk_g2s(buf[s], P + lo, uint32_t(cnt * 4), &bar[s]);
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < kFinStages; ++s) {
      const int64_t t = blockIdx.x + int64_t(s) * gridDim.x;
      if (t < tiles) issue(t, s);
    }
  unsigned long long roots = 0;
  bool noncanon = false, cyc = false;
  int k = 0;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
    const int s = k % kFinStages;
    mbar_wait(&bar[s], uint32_t((k / kFinStages) & 1));
    const int64_t lo = t * kFinTile;
    const int64_t cnt = n4 - lo < kFinTile ? n4 - lo : kFinTile;
#pragma unroll
    for (int h = 0; h < kFinTile / 4 / kEwBlock; ++h) {
      const int qi = h * kEwBlock + threadIdx.x;
      if (int64_t(qi) * 4 >= cnt) break;
      const int4 p4 = reinterpret_cast<const int4*>(buf[s])[qi];
      int32_t lab[4] = {p4.x, p4.y, p4.z, p4.w};
      const int64_t v0 = lo + int64_t(qi) * 4;
      int32_t hop[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) hop[j] = lab[j] != int32_t(v0 + j) ? ld_free(P + lab[j]) : lab[j];
      bool dirty = false;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int32_t v = int32_t(v0 + j);
        int32_t r = lab[j];
        if (r == v) {
          ++roots;
          continue;
        }
        if (hop[j] == r) {
          noncanon |= r > v;
          continue;
        }
        r = hop[j];
        dirty = true;
        int64_t steps = 0;
        int32_t y;
        while ((y = ld_weak(P + r)) != r) {
          r = y;
          if (++steps > n) { cyc = true; break; }
        }
        lab[j] = r;
        noncanon |= r > v;
      }
      if (dirty) *reinterpret_cast<int4*>(P + v0) = make_int4(lab[0], lab[1], lab[2], lab[3]);
    }
    __syncthreads();  // every thread is done with stage s
    if (threadIdx.x == 0) {
      const int64_t tn = t + int64_t(kFinStages) * gridDim.x;
      if (tn < tiles) issue(tn, s);
    }
  }
  // the last n % 4 labels
  if (blockIdx.x == 0 && threadIdx.x < n - n4) {
    const int32_t v = int32_t(n4 + threadIdx.x);
    int32_t r = P[v];
    if (r == v) {
      ++roots;
    } else {
      int32_t y;
      int64_t steps = 0;
      const int32_t r0 = r;
      while ((y = ld_weak(P + r)) != r) {
        r = y;
        if (++steps > n) { cyc = true; break; }
      }
      if (r != r0) P[v] = r;
      noncanon |= r > v;
    }
  }
  block_add<kEwBlock>(ctr + C_COMPONENTS, roots);
  if (__syncthreads_or(noncanon) && threadIdx.x == 0) ctr[C_NONCANON] = 1;
  if (cyc) ctr[C_CYCLE] = 1;
}

__global__ void k_canon_init(int32_t* mins, int32_t n, const unsigned long long* ctr) {
  if (ctr[C_NONCANON] == 0) return;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    mins[v] = INT_MAX;
}

__global__ void k_canon_min(const int32_t* P, int32_t* mins, int32_t n,
                            const unsigned long long* ctr) {
  if (ctr[C_NONCANON] == 0) return;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    atomicMin(mins + P[v], int32_t(v));
}

__global__ void k_canon_apply(int32_t* P, const int32_t* mins, int32_t n,
                              const unsigned long long* ctr) {
  if (ctr[C_NONCANON] == 0) return;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    P[v] = mins[P[v]];
}

__global__ void k_ic_census(const int32_t* P, int32_t n, const int64_t* off, const int32_t* tgt,
                            const int32_t* list, unsigned long long* ctr) {
  const int32_t lmax = int32_t(ctr[C_LMAX]);
  const int64_t count = list ? int64_t(ctr[C_N_ACTIVE]) : int64_t(n);
  unsigned long long ic = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    const int32_t u = list ? list[i] : int32_t(i);
    const int32_t pu = P[u];
    for (int64_t j = off[u]; j < off[u + 1]; ++j) {
      const int32_t pt = P[tgt[j]];
      // over all rows: count crossing entries; over the active rows only,
      // the reverse entries from L_max-labelled rows are added back
      ic += list ? (pu != pt) + (pt == lmax) : (pu != pt);
    }
  }
  block_add<kEwBlock>(ctr + C_IC, ic);
}

__global__ void k_fill(int32_t* a, int64_t n, int32_t v) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) a[i] = v;
}

__global__ void k_count_ne(const int32_t* a, int64_t n, int32_t v, unsigned long long* out) {
  unsigned long long c = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    c += a[i] != v;
  block_add<kEwBlock>(out, c);
}

// Root bitmap: bit v set when P[v] == v (the snapshot a later
// k_root_transitions compares against — n/8 bytes instead of a parent copy).
// Four vertices per thread; the eight lanes holding one word OR it together.
__global__ void __launch_bounds__(kEwBlock) k_root_bitmap(const int32_t* __restrict__ P, int32_t n, uint32_t* bits) {
  const int lane = threadIdx.x & 31;
  const int64_t nq = (int64_t(n) + 3) / 4;
  const int64_t words = (int64_t(n) + 31) / 32;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < nq; base += stride) {
    const int64_t q = base + threadIdx.x;
    const int64_t v0 = 4 * q;
    unsigned nib = 0;
    if (v0 + 3 < n) {
      const int4 p = reinterpret_cast<const int4*>(P)[q];
      nib = unsigned(p.x == int32_t(v0)) | unsigned(p.y == int32_t(v0 + 1)) << 1 |
            unsigned(p.z == int32_t(v0 + 2)) << 2 | unsigned(p.w == int32_t(v0 + 3)) << 3;
    } else {
      for (int k = 0; k < 4; ++k)
        if (v0 + k < n) nib |= unsigned(P[v0 + k] == int32_t(v0 + k)) << k;
    }
    unsigned word = nib << (4 * (lane & 7));
    word |= __shfl_xor_sync(0xffffffffu, word, 1);
    word |= __shfl_xor_sync(0xffffffffu, word, 2);
    word |= __shfl_xor_sync(0xffffffffu, word, 4);
    if ((lane & 7) == 0 && (v0 >> 5) < words) bits[v0 >> 5] = word;
  }
}

// The same snapshot / transitions over the active list alone (a sampled
// sharded finish, driver.py:473): the finish can hook only roots of active
// trees or L_max itself — every other vertex carries label L_max and is no
// root — so one flag per list entry (slot `count` for L_max) stands in for
// the n-bit bitmap and both passes are O(active) instead of O(n).
__global__ void __launch_bounds__(kEwBlock)
k_root_flags_list(const int32_t* __restrict__ P, const int32_t* __restrict__ list, const unsigned long long* ctr,
                  uint8_t* flags) {
  const int64_t count = int64_t(ctr[C_N_ACTIVE]);
  const int32_t lmax = int32_t(ctr[C_LMAX]);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= count; i += stride) {
    const int32_t v = i < count ? __ldg(list + i) : lmax;
    flags[i] = P[v] == v;
  }
}

__global__ void __launch_bounds__(kEwBlock)
k_root_transitions_list(const int32_t* __restrict__ P, const int32_t* __restrict__ list,
                        const unsigned long long* ctr, const uint8_t* __restrict__ flags, int32_t* out_u,
                        int32_t* out_v, unsigned long long* out_count) {
  const int64_t count = int64_t(ctr[C_N_ACTIVE]);
  const int32_t lmax = int32_t(ctr[C_LMAX]);
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t b = int64_t(blockIdx.x) * blockDim.x; b <= count; b += stride) {
    const int64_t i = b + threadIdx.x;
    int32_t v = 0, p = 0;
    bool moved = false;
    if (i <= count && flags[i]) {
      v = i < count ? __ldg(list + i) : lmax;
      p = P[v];
      moved = p != v;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, moved);
    if (!bal) continue;
    unsigned long long pos = 0;
    if (lane == __ffs(int(bal)) - 1) pos = atomicAdd(out_count, static_cast<unsigned long long>(__popc(bal)));
    pos = __shfl_sync(0xffffffffu, pos, __ffs(int(bal)) - 1) + __popc(bal & ((1u << lane) - 1u));
    if (moved) {
      out_u[pos] = v;
      out_v[pos] = p;
    }
  }
}

// Root transitions of one phase: every v that was a root before it
// (before == nullptr: every vertex was) and is not one now emits (v, P[v]) —
// one pair per merge, all inside one component, so unioning them elsewhere
// reproduces the partition change whatever the linking rule.  Four vertices
// per thread, one counter atomic per block (a per-warp atomic on the single
// counter serialised the pass when merges are spread thinly).
__global__ void __launch_bounds__(kEwBlock)
k_root_transitions(const int32_t* __restrict__ P, const uint32_t* __restrict__ before, int32_t n, int32_t* out_u,
                   int32_t* out_v, unsigned long long* count) {
  constexpr int kWarps = kEwBlock / 32;
  __shared__ unsigned warp_n[kWarps];
  __shared__ unsigned long long block_pos;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nq = (int64_t(n) + 3) / 4;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < nq; base += stride) {
    const int64_t q = base + threadIdx.x;
    const int64_t v0 = 4 * q;
    int32_t p[4] = {0, 1, 2, 3};
    unsigned moved = 0;
    if (q < nq) {
      if (v0 + 3 < n) {
        const int4 x = reinterpret_cast<const int4*>(P)[q];
        p[0] = x.x, p[1] = x.y, p[2] = x.z, p[3] = x.w;
      } else {
        for (int k = 0; k < 4; ++k) p[k] = v0 + k < n ? P[v0 + k] : int32_t(v0 + k);
      }
      const unsigned was = before ? (__ldg(before + (v0 >> 5)) >> (v0 & 31)) & 0xfu : 0xfu;
#pragma unroll
      for (int k = 0; k < 4; ++k) moved |= unsigned(p[k] != int32_t(v0 + k) && ((was >> k) & 1u)) << k;
    }
    const unsigned mine = __popc(moved);
    if (!__syncthreads_or(mine != 0)) continue;
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
      block_pos = atomicAdd(count, static_cast<unsigned long long>(tot));
    }
    __syncthreads();
    if (moved) {
      unsigned long long i = block_pos + incl - mine;
      for (int w = 0; w < warp; ++w) i += warp_n[w];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (moved & (1u << k)) {
          out_u[i] = int32_t(v0 + k);
          out_v[i] = p[k];
          ++i;
        }
    }
    __syncthreads();
  }
}

namespace {
std::atomic<long long> g_launches{0};
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

long long launch_total() { return g_launches.load(); }

void add_launches(long long k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

unsigned long long* pinned_words() {
  static thread_local unsigned long long* p = nullptr;
  if (!p) GC_CUDA(cudaMallocHost(&p, 64 * sizeof(unsigned long long)));
  return p;
}

__global__ void k_set_ctr(unsigned long long* ctr, int idx, unsigned long long v) { ctr[idx] = v; }

__global__ void k_add_ctr(unsigned long long* ctr, int idx, unsigned long long v) { ctr[idx] += v; }

void set_ctr_add(unsigned long long* ctr, int idx, unsigned long long v, cudaStream_t st) {
  (k_add_ctr<<<1, 1, 0, st>>>(ctr, idx, v), ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

__global__ void k_zero_words(unsigned long long* a, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = 0;
}

// zero a few counter words with a kernel node: a captured memset node ahead
// of the first kernel of a graph replay measured ~20-50 us of idle time
void zero_ctr(unsigned long long* ctr, int words, cudaStream_t st) {
  (k_zero_words<<<1, 32, 0, st>>>(ctr, words), ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

// Phase timestamps as kernel nodes writing %globaltimer: captured event
// record nodes left 5-10 us of idle between the kernels around them in a
// plan replay; a one-thread kernel node costs ~1.5 us
__global__ void k_stamp(unsigned long long* slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *slot = t;
}

void stamp(unsigned long long* ctr, int i, cudaStream_t st) {
  (k_stamp<<<1, 1, 0, st>>>(ctr + C_STAMP0 + i), ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

// phase boundaries with no work between them share one stamp node
__global__ void k_stamp_mask(unsigned long long* ctr, unsigned mask) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  for (int i = 0; i < 10; ++i)
    if (mask & (1u << i)) ctr[C_STAMP0 + i] = t;
}

namespace {
thread_local unsigned t_pending_stamps = 0;
}

void stamp_defer(int i) { t_pending_stamps |= 1u << i; }

unsigned take_stamps() {
  const unsigned m = t_pending_stamps;
  t_pending_stamps = 0;
  return m;
}

void stamp_flush(unsigned long long* ctr, cudaStream_t st) {
  if (!t_pending_stamps) return;
  (k_stamp_mask<<<1, 1, 0, st>>>(ctr, t_pending_stamps), ::gc::count_launch());
  t_pending_stamps = 0;
  GC_CHECK_LAUNCH();
}

void set_ctr(unsigned long long* ctr, int idx, unsigned long long v, cudaStream_t st) {
  (k_set_ctr<<<1, 1, 0, st>>>(ctr, idx, v), ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

void fill(int32_t* a, int64_t n, int32_t v, cudaStream_t st) {
  if (n <= 0) return;
  (k_fill<<<grid_for(n, kEwBlock, 8), kEwBlock, 0, st>>>(a, n, v), ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

void run_mode(int32_t* P, int32_t n, int32_t* hist, unsigned long long* ctr, cudaStream_t st) {
  if (n > 0) {
    const int g = grid_for(n, kEwBlock, 8);
    (k_mode_probe<<<1, kProbe, 0, st>>>(P, n, ctr, 0), ::gc::count_launch());
    (k_count_eq<<<g, kEwBlock, 0, st>>>(P, n, ctr), ::gc::count_launch());
    (k_hist_zero<<<g, kEwBlock, 0, st>>>(hist, n, ctr), ::gc::count_launch());
    (k_hist_add<<<g, kEwBlock, 0, st>>>(P, hist, n, ctr), ::gc::count_launch());
    (k_hist_argmax<<<g, kEwBlock, 0, st>>>(hist, n, ctr), ::gc::count_launch());
  }
  (k_mode_finish<<<1, 1, 0, st>>>(n, ctr), ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

bool mode_coop() {
  static const bool on = [] {
    const char* e = getenv("GC_MODE_COOP");
    return !(e && e[0] == '0');
  }();
  return on;
}

void run_post_sample(int32_t* P, int32_t n, const int64_t* off, int32_t* list, int32_t* hist,
                     unsigned long long* ctr, bool compress, cudaStream_t st, bool exact_mode) {
  if (n > 0) {
    const int64_t nq = (int64_t(n) + 3) / 4;
    const int gq = grid_for(nq, kEwBlock, 1);
    // the fallback kernels usually exit at once: one resident wave keeps
    // their early exit cheap and still streams when they do run
    const int g = grid_for(n, kEwBlock, 1);
    // the sampler may have set the exact mode (C_CAND + C_MODE_EXACT)
    if (exact_mode) stamp_flush(ctr, st);
    else (k_mode_probe<<<1, kProbe, 0, st>>>(P, n, ctr, 1, take_stamps()), ::gc::count_launch());
    // one resident wave: six 256-thread blocks per SM, two quads per thread
    const int gps = grid_for((nq + 1) / 2, kEwBlock, 1) < num_sms() * GC_PS_BLOCKS
                        ? grid_for((nq + 1) / 2, kEwBlock, 1)
                        : num_sms() * GC_PS_BLOCKS;
    if (compress) (k_post_sample<true><<<gps, kEwBlock, 0, st>>>(P, n, off, list, ctr), ::gc::count_launch());
    else (k_post_sample<false><<<gps, kEwBlock, 0, st>>>(P, n, off, list, ctr), ::gc::count_launch());
    // exact-mode fallback: one cooperative launch that exits at once on a
    // strict majority (GC_MODE_COOP=0: the five separate early-exit kernels)
    if (mode_coop()) {
      static int per_sm = 0;
      if (!per_sm) GC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mode_fallback, kEwBlock, 0));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(num_sms() * (per_sm > 0 ? per_sm : 1));
      cfg.blockDim = dim3(kEwBlock);
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const int32_t* Pc = P;
      GC_CUDA(cudaLaunchKernelEx(&cfg, k_mode_fallback, Pc, hist, n, off, list, ctr));
      ::gc::count_launch();
      GC_CHECK_LAUNCH();
      return;
    }
    (k_hist_zero<<<g, kEwBlock, 0, st>>>(hist, n, ctr), ::gc::count_launch());
    (k_hist_add<<<g, kEwBlock, 0, st>>>(P, hist, n, ctr), ::gc::count_launch());
    (k_hist_argmax<<<g, kEwBlock, 0, st>>>(hist, n, ctr), ::gc::count_launch());
  }
  (k_mode_finish<<<1, 1, 0, st>>>(n, ctr), ::gc::count_launch());
  if (n > 0)
    (k_gather_active<<<grid_for((int64_t(n) + 3) / 4, kEwBlock, 1), kEwBlock, 0, st>>>(P, n, off, list, ctr, 1),
     ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

void run_gather(int32_t* P, int32_t n, const int64_t* off, int32_t* list, unsigned long long* ctr,
                cudaStream_t st) {
  if (n <= 0) return;
  (k_gather_active<<<grid_for((int64_t(n) + 3) / 4, kEwBlock, 4), kEwBlock, 0, st>>>(P, n, off, list, ctr, 0),
   ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

void run_finalize(int32_t* P, int32_t n, int32_t* mins, unsigned long long* ctr, cudaStream_t st,
                  bool maybe_noncanon, const int32_t* list) {
  if (n <= 0) return;
  const int g = grid_for(n, kEwBlock, 8);
  unsigned sm = 0;
  if (list) {
    (k_finalize_list<<<num_sms() * 8, kEwBlock, 0, st>>>(P, n, list, ctr, take_stamps()), ::gc::count_launch());
  } else {
    sm = take_stamps();
  }
  const int lm = list != nullptr;
  // TMA-staged form by default (ncu, s24: 23.5 vs 25.1 us per launch);
  // GC_FIN_TMA=0 selects the register-staged kernel
  static const bool tma = !(getenv("GC_FIN_TMA") && atoi(getenv("GC_FIN_TMA")) == 0);
  if (tma && reinterpret_cast<uintptr_t>(P) % 16 == 0) {
    const int64_t tiles = ((int64_t(n) / 4) * 4 + kFinTile - 1) / kFinTile;
    const int64_t cap = int64_t(num_sms()) * 6;  // 6 blocks x 33 KB of stages per SM
    (k_finalize_tma<<<int(tiles < cap ? (tiles > 0 ? tiles : 1) : cap), kEwBlock, 0, st>>>(P, n, ctr, sm, lm),
     ::gc::count_launch());
  } else
  (k_finalize<<<grid_for((int64_t(n) + 3) / 4, kEwBlock, 4), kEwBlock, 0, st>>>(P, n, ctr, sm, lm),
   ::gc::count_launch());
  if (!maybe_noncanon) {
    GC_CHECK_LAUNCH();
    return;
  }
  (k_canon_init<<<g, kEwBlock, 0, st>>>(mins, n, ctr), ::gc::count_launch());
  (k_canon_min<<<g, kEwBlock, 0, st>>>(P, mins, n, ctr), ::gc::count_launch());
  (k_canon_apply<<<g, kEwBlock, 0, st>>>(P, mins, n, ctr), ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

}  // namespace gc

extern "C" long long gc_launch_count(void) { return gc::launch_total(); }
