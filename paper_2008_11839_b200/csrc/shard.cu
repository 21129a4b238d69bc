// shard.cu — the compact label exchange of the sharded pipeline.
//
// After gc_shard_sample every rank holds the partition induced by the
// sampled edges of its own rows.  Exchanging it edge by edge costs one pair
// per sampled row; but almost every sampled vertex sits in the rank's most
// frequent class (the local giant), so the summary is
//   * the giant as an n-bit bitmap plus its label, and
//   * a pair (v, label) for every other non-singleton vertex,
// i.e. n/8 bytes plus the (small) non-giant remainder.  gc_shard_join
// rebuilds the join of all ranks' partitions exactly: giants that share a
// vertex are one class (an 8x8 overlap matrix reduced on the device), every
// giant member points at its class representative, and the remainder pairs
// are unioned with the spec's own rule.  The sampled partition — hence
// L_max, cov, the active set and the finish inspections — equals the
// single-GPU pipeline's.
#include <climits>

#include "internal.h"
#include "pipeline.cuh"

namespace gc {

namespace {

constexpr int kMaxRanks = 8;  // one NVSwitch box; the overlap matrix is one u64

// bitmap word per warp + block-aggregated remainder pairs
__global__ void __launch_bounds__(kEwBlock)
k_summary(const int32_t* __restrict__ P, int32_t n, const unsigned long long* ctr, uint32_t* bits,
          int32_t* out_u, int32_t* out_v, unsigned long long* out_count) {
  const int32_t g = int32_t(ctr[C_LMAX]);
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
    const int64_t v = base + threadIdx.x;
    int32_t lab = 0;
    bool in_g = false, pair = false;
    if (v < n) {
      lab = P[v];
      in_g = lab == g;
      pair = !in_g && lab != int32_t(v);
    }
    const unsigned word = __ballot_sync(0xffffffffu, in_g);
    if (lane == 0 && base + (threadIdx.x & ~31) < n) bits[(base + (threadIdx.x & ~31)) >> 5] = word;
    const unsigned bal = __ballot_sync(0xffffffffu, pair);
    if (!bal) continue;
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(out_count, static_cast<unsigned long long>(__popc(bal)));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (pair) {
      const unsigned long long i = pos + __popc(bal & ((1u << lane) - 1u));
      out_u[i] = int32_t(v);
      out_v[i] = lab;
    }
  }
}

__global__ void k_store_label(const unsigned long long* ctr, int64_t* label_out) {
  *label_out = int64_t(ctr[C_LMAX]);
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
  for (int o = 16; o > 0; o >>= 1) m |= __shfl_xor_sync(0xffffffffu, m, o);
  if ((threadIdx.x & 31) == 0 && m) atomicOr(mat, m);
}

// super-classes of the giants (tiny union-find over <= 8 nodes); rep[r] =
// smallest giant label in r's class
__global__ void k_giant_classes(const unsigned long long* mat, const int64_t* labels, int32_t nranks,
                                int32_t* rep) {
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
}

__global__ void __launch_bounds__(kEwBlock)
k_join_init(int32_t* P, int32_t n, const uint32_t* __restrict__ bits, int64_t words, int32_t nranks,
            const int32_t* __restrict__ rep) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const int64_t w = v >> 5;
    const uint32_t bit = 1u << (v & 31);
    int32_t p = int32_t(v);
    for (int r = 0; r < nranks; ++r)
      if (bits[int64_t(r) * words + w] & bit) {
        p = rep[r];
        break;
      }
    P[v] = p;
  }
}

}  // namespace

}  // namespace gc

using namespace gc;

extern "C" {

size_t gc_shard_summary_workspace(int64_t n) { return size_t(n > 0 ? n : 1) * 4 + 4096; }

int gc_shard_summary(int32_t* parent, int64_t n, uint32_t* giant_bits, int64_t* giant_label, int32_t* out_u,
                     int32_t* out_v, unsigned long long* out_count, void* ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    require(n >= 0 && n < (int64_t(1) << 31), GC_ERR_MALFORMED, "bad length");
    require(giant_label && out_count && (n == 0 || (parent && giant_bits && out_u && out_v)), GC_ERR_ARG,
            "null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Arena a(ws, ws_bytes);
    unsigned long long* ctr = a.take<unsigned long long>(C_COUNT_);
    int32_t* hist = a.take<int32_t>(n);
    GC_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * C_COUNT_, st));
    GC_CUDA(cudaMemsetAsync(out_count, 0, sizeof(unsigned long long), st));
    const int32_t nn = int32_t(n);
    if (nn) {
      (k_compress<<<grid_for(nn, kEwBlock, 8), kEwBlock, 0, st>>>(parent, nn), count_launch());
      run_mode(parent, nn, hist, ctr, st);  // the local giant: most frequent label, ties -> smaller
      (k_summary<<<grid_for(nn, kEwBlock, 8), kEwBlock, 0, st>>>(parent, nn, ctr, giant_bits, out_u, out_v,
                                                                out_count), count_launch());
    }
    (k_store_label<<<1, 1, 0, st>>>(ctr, giant_label), count_launch());
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
    int32_t* aux = nullptr;
    const UFConfig c{spec->finish, spec->find, spec->splice};
    if (c.unite == GC_FINISH_HOOKS || c.unite == GC_FINISH_REM_LOCK) aux = a.take<int32_t>(n);
    const int32_t nn = int32_t(n);
    if (nn == 0) return;
    const int64_t words = (n + 31) / 32;
    GC_CUDA(cudaMemsetAsync(mat, 0, 8, st));
    (k_overlap<<<grid_for(words, kEwBlock, 4), kEwBlock, 0, st>>>(bits, words, nranks, mat), count_launch());
    (k_giant_classes<<<1, 1, 0, st>>>(mat, giant_labels, nranks, rep), count_launch());
    (k_join_init<<<grid_for(nn, kEwBlock, 8), kEwBlock, 0, st>>>(parent, nn, bits, words, nranks, rep),
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
