// kout_micro.cu — where does the k-out union kernel's time go?
// Variants over the same CSR (RMAT s24 built on the device by the package):
//   stream      : offsets + the first two targets of every row, no unions
//   rows        : replica of k_union_rows<Rem-CAS, halve, atomic splice>
//   make_pairs  : write (t0, t1) per row (coalesced int2)
//   union_pairs : the unions alone, fed by the coalesced pair array
//   rows_async  : rows with the offsets / row heads staged in shared memory
//                 by cp.async two tiles ahead (no registers held in flight)
// Built by profiles/micro/kout_micro.py with nvcc; not product code.
#include <cstdint>
#include <cuda_runtime.h>

#include "uf.cuh"

using namespace gc;
using R = Rule<GC_FINISH_REM_CAS, GC_FIND_HALVE, GC_SPLICE_ATOMIC, false>;

namespace {

__global__ void k_init(int32_t* P, int32_t n) {
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += int64_t(gridDim.x) * blockDim.x)
    P[v] = int32_t(v);
}

__global__ void __launch_bounds__(512) k_stream(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt,
                                                int32_t n, int32_t* sink) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (int64_t(blockIdx.x) * 512 + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * 512) >> 5;
  const uint64_t pol = evict_first_policy();
  int32_t acc = 0;
  for (int64_t base = warp0 * 32; base < n; base += nwarps * 32) {
    const int64_t u = base + lane;
    if (u < n) {
      const int64_t b = ld_stream64(off + u, pol), e = ld_stream64(off + u + 1, pol);
      const int64_t d = e - b;
      if (d > 0) acc ^= ldg32(tgt + b);
      if (d > 1) acc ^= ldg32(tgt + b + 1);
    }
  }
  if (acc == 0x7fffffff) sink[0] = acc;
}

__global__ void __launch_bounds__(512) k_rows(int32_t* P, const int64_t* __restrict__ off,
                                              const int32_t* __restrict__ tgt, int32_t n) {
  UFState s{P, nullptr, nullptr, nullptr, nullptr, nullptr, n};
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (int64_t(blockIdx.x) * 512 + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * 512) >> 5;
  const uint64_t pol = evict_first_policy();
  for (int64_t base = warp0 * 32; base < n; base += nwarps * 32) {
    const int64_t i = base + lane;
    if (i < n) {
      const int32_t u = int32_t(i);
      const int64_t b = ld_stream64(off + u, pol), e = ld_stream64(off + u + 1, pol);
      const int64_t d = e - b;
      const int32_t take = int32_t(d < 2 ? d : 2);
      const int32_t f0 = take > 0 ? ldg32(tgt + b) : 0;
      const int32_t f1 = take > 1 ? ldg32(tgt + b + 1) : 0;
      if (take > 0) R::unite(s, u, f0);
      if (take > 1) R::unite(s, u, f1);
    }
    __syncwarp();  // reconverge: the next rows' loads issue as one warp request
  }
}

__global__ void k_make_pairs(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, int32_t n,
                             int2* pairs) {
  for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < n; u += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = off[u], d = off[u + 1] - b;
    pairs[u] = make_int2(d > 0 ? tgt[b] : -1, d > 1 ? tgt[b + 1] : -1);
  }
}

__global__ void __launch_bounds__(512) k_union_pairs(int32_t* P, const int2* __restrict__ pairs, int32_t n) {
  UFState s{P, nullptr, nullptr, nullptr, nullptr, nullptr, n};
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t b0 = int64_t(blockIdx.x) * blockDim.x; b0 < n; b0 += stride) {
    const int64_t u = b0 + threadIdx.x;
    if (u < n) {
      const int2 p = __ldg(pairs + u);
      if (p.x >= 0) R::unite(s, int32_t(u), p.x);
      if (p.y >= 0) R::unite(s, int32_t(u), p.y);
    }
    __syncwarp();
  }
}

// ---- cp.async staging ------------------------------------------------------
template <bool HINT>
__device__ __forceinline__ void cp16(void* dst, const void* src, uint64_t pol) {
  if (HINT)
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "l"(pol) : "memory");
  else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int kAW = 16;  // warps per block (512 threads)

struct AsyncSmem {
  alignas(16) int64_t off[kAW][2][34];
  alignas(16) int32_t head[kAW][2][32][8];
};

// offsets of tile rows [r0, r0 + 32] into ob: 16 lanes x 16 B + one 8-byte tail entry
template <bool HINT>
__device__ __forceinline__ void issue_off(int64_t* ob, const int64_t* off, int64_t r0, int32_t n, int lane,
                                          uint64_t pol) {
  if (r0 >= n) return;
  if (lane < 16) {
    const int64_t e = r0 + 2 * lane;  // entries e, e + 1 (<= n needed)
    if (e + 1 <= n) cp16<HINT>(ob + 2 * lane, off + e, pol);
    else if (e <= n) cp8(ob + 2 * lane, off + e);
  } else if (lane == 16 && r0 + 32 <= n) {
    cp8(ob + 32, off + r0 + 32);
  }
}

// the first two targets of the lane's row into hb (two 16-byte chunks)
template <bool HINT>
__device__ __forceinline__ void issue_head(int32_t* hb, const int32_t* tgt, int64_t b, int32_t take, int64_t m,
                                           uint64_t pol) {
  if (take <= 0) return;
  const int64_t c0 = b & ~int64_t(3);
  if (c0 + 4 <= m) cp16<HINT>(hb, tgt + c0, pol);
  else for (int64_t j = b; j < b + take; ++j) cp4(hb + (j - c0), tgt + j);
  if (take > 1 && (b & 3) == 3) {
    const int64_t c1 = c0 + 4;
    if (c1 + 4 <= m) cp16<HINT>(hb + 4, tgt + c1, pol);
    else cp4(hb + 4, tgt + c1);
  }
}

template <bool HINT>
__global__ void __launch_bounds__(kAW * 32) k_rows_async(int32_t* P, const int64_t* __restrict__ off,
                                                         const int32_t* __restrict__ tgt, int32_t n, int64_t m) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  AsyncSmem& sm = *reinterpret_cast<AsyncSmem*>(smem_raw);
  UFState s{P, nullptr, nullptr, nullptr, nullptr, nullptr, n};
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t gw = (int64_t(blockIdx.x) * kAW * 32 + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * kAW * 32) >> 5;
  auto tile_r0 = [&](int64_t k) { return (gw + k * nw) * 32; };
  const uint64_t pol = evict_first_policy();
  // prologue: offsets of tiles 0 and 1, heads of tile 0
  issue_off<HINT>(sm.off[w][0], off, tile_r0(0), n, lane, pol);
  cp_commit();
  issue_off<HINT>(sm.off[w][1], off, tile_r0(1), n, lane, pol);
  cp_commit();
  cp_wait<1>();
  __syncwarp();
  int32_t take_cur = 0;
  int64_t b_cur = 0;
  {
    const int64_t r0 = tile_r0(0);
    if (r0 + lane < n) {
      b_cur = sm.off[w][0][lane];
      const int64_t d = sm.off[w][0][lane + 1] - b_cur;
      take_cur = int32_t(d < 2 ? d : 2);
      issue_head<HINT>(sm.head[w][0][lane], tgt, b_cur, take_cur, m, pol);
    }
  }
  cp_commit();
  for (int64_t k = 0; tile_r0(k) < n; ++k) {
    const int cur = int(k & 1), nxt = cur ^ 1;
    cp_wait<0>();  // offsets of tile k + 1 and heads of tile k have landed
    __syncwarp();
    // heads of tile k + 1
    int32_t take_nxt = 0;
    int64_t b_nxt = 0;
    const int64_t r1 = tile_r0(k + 1);
    if (r1 + lane < n) {
      b_nxt = sm.off[w][nxt][lane];
      const int64_t d = sm.off[w][nxt][lane + 1] - b_nxt;
      take_nxt = int32_t(d < 2 ? d : 2);
      issue_head<HINT>(sm.head[w][nxt][lane], tgt, b_nxt, take_nxt, m, pol);
    }
    cp_commit();
    __syncwarp();  // every lane has read sm.off[w][nxt]... and sm.off[w][cur] is free
    issue_off<HINT>(sm.off[w][cur], off, tile_r0(k + 2), n, lane, pol);
    cp_commit();
    // unions of tile k
    const int64_t u = tile_r0(k) + lane;
    if (u < n && take_cur > 0) {
      const int32_t* hb = sm.head[w][cur][lane];
      const int o = int(b_cur & 3);
      const int32_t f0 = hb[o];
      const int32_t f1 = take_cur > 1 ? hb[o + 1] : 0;
      R::unite(s, int32_t(u), f0);
      if (take_cur > 1) R::unite(s, int32_t(u), f1);
    }
    take_cur = take_nxt;
    b_cur = b_nxt;
  }
  cp_wait<0>();
}

// ---- per-warp bulk-copy (TMA engine) staging -------------------------------
// Each warp stages its own tiles: lane 0 bulk-copies the offsets of tile
// k + 2 and, once tile k + 1's offsets have landed, the contiguous window of
// targets its 32 rows start in (capped at kWin bytes; rows past the window
// read their heads from global).  The copies run on the TMA engine, off the
// LSU / L1 path the union chains use; lanes copy their heads into registers
// and release the stage before their unions.
constexpr int kBW = 16;
constexpr int kWin = 1024;  // bytes per window stage

struct BulkSmem {
  alignas(16) int64_t off[kBW][2][34];
  alignas(16) int32_t win[kBW][2][kWin / 4];
  alignas(8) uint64_t boff[kBW][2];
  alignas(8) uint64_t bwin[kBW][2];
};

__device__ __forceinline__ void win_bounds(const int64_t* o, int64_t r0, int32_t n, int64_t m, int64_t& ws,
                                           int64_t& we) {
  const int64_t last = r0 + 32 <= n ? r0 + 32 : n;
  const int64_t lo = o[0], hi = o[last - r0];
  ws = lo & ~int64_t(3);
  int64_t e = (hi + 3) & ~int64_t(3);
  if (e > ws + kWin / 4) e = ws + kWin / 4;
  const int64_t mfloor = m & ~int64_t(3);
  if (e > mfloor) e = mfloor > ws ? mfloor : ws;
  we = e;
}

__global__ void __launch_bounds__(kBW * 32) k_rows_bulk(int32_t* P, const int64_t* __restrict__ off,
                                                      const int32_t* __restrict__ tgt, int32_t n, int64_t m) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BulkSmem& sm = *reinterpret_cast<BulkSmem*>(smem_raw);
  UFState s{P, nullptr, nullptr, nullptr, nullptr, nullptr, n};
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t gw = (int64_t(blockIdx.x) * kBW * 32 + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * kBW * 32) >> 5;
  auto tile_r0 = [&](int64_t k) { return (gw + k * nw) * 32; };
  // offsets of tile k into stage st: entries r0 .. min(r0 + 33, n + 1) (16-byte multiple)
  auto issue_off = [&](int64_t k, int st) {
    const int64_t r0 = tile_r0(k);
    if (r0 >= n) return;
    int64_t cnt = (n + 1) - r0;
    if (cnt > 34) cnt = 34;
    cnt &= ~int64_t(1);  // 16-byte multiple; the odd last entry is read from global
    mbar_expect_tx(&sm.boff[w][st], uint32_t(cnt * 8));
    bulk_g2s(sm.off[w][st], off + r0, uint32_t(cnt * 8), &sm.boff[w][st]);
  };
  auto off_at = [&](int st, int64_t r0, int i) -> int64_t {
    // entry r0 + i of the offsets: from the stage unless it is the odd tail
    const int64_t avail = ((n + 1) - r0) < 34 ? (((n + 1) - r0) & ~int64_t(1)) : 34;
    return i < avail ? sm.off[w][st][i] : __ldg(off + r0 + i);
  };
  auto issue_win = [&](int64_t k, int st) {
    const int64_t r0 = tile_r0(k);
    if (r0 >= n) return;
    int64_t o[33];
    (void)o;
    const int64_t last = r0 + 32 <= n ? r0 + 32 : n;
    const int64_t lo = off_at(st, r0, 0), hi = off_at(st, r0, int(last - r0));
    int64_t ws = lo & ~int64_t(3);
    int64_t e = (hi + 3) & ~int64_t(3);
    if (e > ws + kWin / 4) e = ws + kWin / 4;
    const int64_t mfloor = m & ~int64_t(3);
    if (e > mfloor) e = mfloor > ws ? mfloor : ws;
    const uint32_t bytes = uint32_t((e - ws) * 4);
    mbar_expect_tx(&sm.bwin[w][st], bytes);
    if (bytes) bulk_g2s(sm.win[w][st], tgt + ws, bytes, &sm.bwin[w][st]);
  };
  if (lane == 0) {
    for (int st = 0; st < 2; ++st) {
      mbar_init(&sm.boff[w][st], 1);
      mbar_init(&sm.bwin[w][st], 1);
    }
    mbar_fence_init();
  }
  __syncwarp();
  if (lane == 0) {
    issue_off(0, 0);
    issue_off(1, 1);
    if (tile_r0(0) < n) {
      mbar_wait(&sm.boff[w][0], 0);
      issue_win(0, 0);
    }
  }
  __syncwarp();
  for (int64_t k = 0; tile_r0(k) < n; ++k) {
    const int st = int(k & 1);
    const uint32_t ph = uint32_t((k >> 1) & 1);
    const int64_t r0 = tile_r0(k);
    // the next tile's window, as soon as its offsets are in
    if (lane == 0 && tile_r0(k + 1) < n) {
      mbar_wait(&sm.boff[w][st ^ 1], uint32_t(((k + 1) >> 1) & 1));
      issue_win(k + 1, st ^ 1);
    }
    mbar_wait(&sm.boff[w][st], ph);
    mbar_wait(&sm.bwin[w][st], ph);
    const int64_t u = r0 + lane;
    int32_t take = 0, f0 = 0, f1 = 0;
    if (u < n) {
      const int64_t b = off_at(st, r0, lane), e = off_at(st, r0, lane + 1);
      const int64_t d = e - b;
      take = int32_t(d < 2 ? d : 2);
      const int64_t last = r0 + 32 <= n ? r0 + 32 : n;
      const int64_t lo = off_at(st, r0, 0), hi = off_at(st, r0, int(last - r0));
      int64_t ws = lo & ~int64_t(3);
      int64_t we = (hi + 3) & ~int64_t(3);
      if (we > ws + kWin / 4) we = ws + kWin / 4;
      const int64_t mfloor = m & ~int64_t(3);
      if (we > mfloor) we = mfloor > ws ? mfloor : ws;
      if (take > 0) f0 = b < we ? sm.win[w][st][b - ws] : ldg32(tgt + b);
      if (take > 1) f1 = b + 1 < we ? sm.win[w][st][b + 1 - ws] : ldg32(tgt + b + 1);
    }
    __syncwarp();  // stage st fully read
    if (lane == 0) issue_off(k + 2, st);
    if (take > 0) R::unite(s, int32_t(u), f0);
    if (take > 1) R::unite(s, int32_t(u), f1);
    __syncwarp();
  }
}

}  // namespace

extern "C" {

int km_init(int32_t* P, int32_t n, cudaStream_t st) {
  k_init<<<148 * 8, 256, 0, st>>>(P, n);
  return int(cudaGetLastError());
}
int km_stream(const int64_t* off, const int32_t* tgt, int32_t n, int32_t* sink, cudaStream_t st) {
  k_stream<<<148 * 4, 512, 0, st>>>(off, tgt, n, sink);
  return int(cudaGetLastError());
}
int km_rows(int32_t* P, const int64_t* off, const int32_t* tgt, int32_t n, cudaStream_t st) {
  k_rows<<<148 * 4, 512, 0, st>>>(P, off, tgt, n);
  return int(cudaGetLastError());
}
int km_make_pairs(const int64_t* off, const int32_t* tgt, int32_t n, int2* pairs, cudaStream_t st) {
  k_make_pairs<<<148 * 8, 256, 0, st>>>(off, tgt, n, pairs);
  return int(cudaGetLastError());
}
int km_union_pairs(int32_t* P, const int2* pairs, int32_t n, cudaStream_t st) {
  k_union_pairs<<<148 * 4, 512, 0, st>>>(P, pairs, n);
  return int(cudaGetLastError());
}
int km_rows_async(int32_t* P, const int64_t* off, const int32_t* tgt, int32_t n, int64_t m, int blocks_per_sm,
                  int hint, cudaStream_t st) {
  const int bytes = int(sizeof(AsyncSmem));
  if (hint) {
    cudaFuncSetAttribute(k_rows_async<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    k_rows_async<true><<<148 * blocks_per_sm, kAW * 32, bytes, st>>>(P, off, tgt, n, m);
  } else {
    cudaFuncSetAttribute(k_rows_async<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    k_rows_async<false><<<148 * blocks_per_sm, kAW * 32, bytes, st>>>(P, off, tgt, n, m);
  }
  return int(cudaGetLastError());
}
int km_async_smem() { return int(sizeof(AsyncSmem)); }
int km_rows_bulk(int32_t* P, const int64_t* off, const int32_t* tgt, int32_t n, int64_t m, int blocks_per_sm,
                 cudaStream_t st) {
  const int bytes = int(sizeof(BulkSmem));
  cudaFuncSetAttribute(k_rows_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  k_rows_bulk<<<148 * blocks_per_sm, kBW * 32, bytes, st>>>(P, off, tgt, n, m);
  return int(cudaGetLastError());
}
int km_bulk_smem() { return int(sizeof(BulkSmem)); }
}
