// common.cuh — shared device helpers for libgconn (sm_100a).
//
// Memory-model note.  The parent array P is shared by every thread of a
// kernel and mutated with atomicCAS while other threads walk it.  All reads
// of P therefore go through ld.relaxed.gpu (LDG.E.STRONG.GPU: served by L2,
// never a stale L1 line), the GPU analogue of the reference's "single list
// reads are atomic under the GIL" (parallel.py:3-8).  Read-only graph data
// (offsets / targets) uses the non-coherent path (ld.global.nc).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/gconn.h"

namespace gc {

constexpr int kWarp = 32;

__device__ __forceinline__ int32_t ld_acq(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// plain global load the compiler may schedule freely (several in flight);
// for reads where any stale value is acceptable
__device__ __forceinline__ int32_t ld_free(const int32_t* p) {
  int32_t v;
  asm("ld.global.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// plain global load (L1-cacheable), never hoisted across other memory ops
__device__ __forceinline__ int32_t ld_weak(const int32_t* p) {
  int32_t v;
  asm volatile("ld.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_rlx(int32_t* p, int32_t v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ bool cas(int32_t* p, int32_t expect, int32_t desired) {
  return atomicCAS(p, expect, desired) == expect;
}

// bitmap words that other threads set concurrently (plain L1-cacheable
// load: a stale word only misses bits, which every user tolerates)
__device__ __forceinline__ uint32_t ld_bits(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_or_bits(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// giant-filter bitmap accesses with an L2 eviction-priority hint (evict_last
// keeps the n/8-byte bitmap resident while the batch's random parent reads
// stream a parent array several times the L2 through the cache)
__device__ __forceinline__ uint32_t ld_bits(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_bits_nc(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void red_or_bits(uint32_t* p, uint32_t v, uint64_t pol) {
  asm volatile("red.relaxed.gpu.global.or.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ bool gbit(uint32_t w, int32_t x) { return (w >> (x & 31)) & 1u; }

// atomicMin on a word many warps update (a running minimum): skip the atomic
// when a plain read already shows a value <= v (the word only decreases, so
// a stale read is never below the true value) — tens of thousands of
// per-warp atomics on one word serialise at its L2 slice
__device__ __forceinline__ void atomic_min_if_lower(int32_t* p, int32_t v) {
  if (v < ld_weak(p)) atomicMin(p, v);
}

// fire-and-forget min (RED.MIN): the result is not needed by the caller
__device__ __forceinline__ void red_min(int32_t* p, int32_t v) {
  asm volatile("red.relaxed.gpu.global.min.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Streaming loads for graph data that is read once per pass: no L1
// allocation and L2 evict-first, so the stream does not push the parent
// array (kept persisting in L2) out of the cache.
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t evict_normal_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// policy for the giant-filter bitmap (keep: evict_last, else evict_normal)
__device__ __forceinline__ uint64_t bits_policy(bool keep) {
  return keep ? evict_last_policy() : evict_normal_policy();
}
__device__ __forceinline__ int32_t ld_weak_pol(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol) : "memory");
  return v;
}
__device__ __forceinline__ int32_t ld_acq_pol(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol) : "memory");
  return v;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int2 ld_stream2(const int32_t* p, uint64_t pol) {
  int2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;"
               : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int64_t ld_stream64(const int64_t* p, uint64_t pol) {
  int64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}

// L1-allocating read-only load with an L2 evict-first hint
__device__ __forceinline__ int32_t ld_l1_evict_first(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ int64_t ldg64(const int64_t* p) { return __ldg(p); }
__device__ __forceinline__ int32_t ldg32(const int32_t* p) { return __ldg(p); }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of a 64-bit counter, one atomicAdd per block.  The staging
// array is shared by every call in a kernel, so a call first waits until the
// previous call's reader (warp 0) is done with it (compute-sanitizer
// racecheck found the back-to-back calls racing).
template <int BLOCK>
__device__ __forceinline__ void block_add(unsigned long long* dst, unsigned long long v) {
  __shared__ unsigned long long part[BLOCK / kWarp];
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) part[wid] = v;
  __syncthreads();
  if (wid == 0) {
    unsigned long long s = lane < BLOCK / kWarp ? part[lane] : 0ull;
    s = warp_sum(s);
    if (lane == 0 && s) atomicAdd(dst, s);
  }
}

// Block-aggregated append to a global queue.  Warps stage their items in
// shared memory (one shared atomic per warp per push); flush() reserves the
// block's range with a single global atomic, so a frontier of F vertices
// costs F / blockDim global atomics instead of one per warp or per item.
// Items beyond the staging capacity go straight to the global queue.
// push() must be called by whole (converged) warps and flush() by the whole
// block.
template <int CAP>
struct BlockQueue {
  int32_t items[CAP];
  int count;
  unsigned long long base;

  __device__ __forceinline__ void init() {
    if (threadIdx.x == 0) count = 0;
    __syncthreads();
  }
  __device__ __forceinline__ void push(bool p, int32_t x, int32_t* q, unsigned long long* qc) {
    const unsigned bal = __ballot_sync(0xffffffffu, p);
    if (!bal) return;
    const int lane = threadIdx.x & 31;
    int pos = 0;
    if (lane == 0) pos = atomicAdd(&count, __popc(bal));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    const int mine = pos + __popc(bal & ((1u << lane) - 1u));
    if (p && mine < CAP) items[mine] = x;
    // staging full: the overflowing lanes append straight to the global
    // queue with one counter atomic per warp (one per item serialised large
    // frontiers on the single counter)
    const unsigned over = __ballot_sync(0xffffffffu, p && mine >= CAP);
    if (!over) return;
    unsigned long long gpos = 0;
    if (lane == __ffs(int(over)) - 1) gpos = atomicAdd(qc, static_cast<unsigned long long>(__popc(over)));
    gpos = __shfl_sync(0xffffffffu, gpos, __ffs(int(over)) - 1);
    if (p && mine >= CAP) q[gpos + __popc(over & ((1u << lane) - 1u))] = x;
  }
  // block-uniform call sites only (every thread of the block reaches it):
  // flush once the staging is at least `threshold` full, so big frontiers
  // rarely overflow
  __device__ __forceinline__ void maybe_flush(int32_t* q, unsigned long long* qc, int threshold) {
    __syncthreads();
    if (count >= threshold) flush(q, qc);
  }
  __device__ __forceinline__ void flush(int32_t* q, unsigned long long* qc) {
    __syncthreads();
    const int c = count < CAP ? count : CAP;
    if (threadIdx.x == 0) base = c ? atomicAdd(qc, static_cast<unsigned long long>(c)) : 0ull;
    __syncthreads();
    for (int i = threadIdx.x; i < c; i += blockDim.x) q[base + i] = items[i];
    __syncthreads();
    if (threadIdx.x == 0) count = 0;
    __syncthreads();
  }
};

// ---- 1-D bulk copies (TMA engine) into shared memory ---------------------
// Streaming passes over the label array stage their tiles through shared
// memory with cp.async.bulk: the copy engine keeps a whole tile per stage in
// flight without occupying registers, where per-thread 16-byte loads hold
// one quad per thread and stall on the dependent work that follows.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LAB_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LAB_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Phase timestamps taken at the entry of the next kernel: thread 0 of block
// 0 writes %globaltimer into every slot of `mask` (ctr[stamp_base + i]).  A
// separate one-thread stamp node between two kernels costs ~1.5 us of a plan
// replay; the next kernel's first block starts within ~1 us of the previous
// kernel's end, which is the same phase boundary.
__device__ __forceinline__ void entry_stamp(unsigned long long* slots, unsigned mask) {
  if (mask == 0u || blockIdx.x != 0 || threadIdx.x != 0) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  for (int i = 0; i < 10; ++i)
    if (mask & (1u << i)) slots[i] = t;
}

// Grid size for an elementwise kernel: enough CTAs to cover `work` items
// but capped at a whole number of waves over the 148 SMs.
inline int grid_for(int64_t work, int block, int max_waves = 32) {
  int64_t g = (work + block - 1) / block;
  int64_t cap = int64_t(148) * (2048 / block) * max_waves;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return int(g);
}

}  // namespace gc
