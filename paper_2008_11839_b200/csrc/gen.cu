// gen.cu — device graph generators and CSR normalisation (graphs.py:90-121,
// 210-245) plus the host MT19937 used for JTB ranks (dset.py:372-374).
//
// gen_rmat reproduces numpy's Generator(PCG64).random() stream exactly: the
// reference draws, per recursion level, an (m,4) noise block and then m
// quadrant draws, so edge i at level L reads stream positions
//   L*5m + 4i + j  (noise, j < 4)   and   L*5m + 4m + i  (quadrant).
// Each thread jumps its PCG64 state there with the LCG jump-ahead and
// evaluates the same IEEE double expressions (no FMA contraction), giving the
// reference's edge list bit for bit without a host round trip.
#include <climits>
#include <cub/cub.cuh>

#include "pipeline.cuh"

namespace gc {
namespace {

typedef unsigned __int128 u128;

constexpr uint64_t kMulHi = 0x2360ED051FC65DA4ull;
constexpr uint64_t kMulLo = 0x4385DF649FCCF645ull;

__host__ __device__ __forceinline__ u128 mk(uint64_t hi, uint64_t lo) {
  return (u128(hi) << 64) | u128(lo);
}

struct Pcg {
  u128 s, inc;
  __device__ __forceinline__ uint64_t next() {
    s = s * mk(kMulHi, kMulLo) + inc;
    const uint64_t hi = uint64_t(s >> 64), lo = uint64_t(s);
    const unsigned rot = unsigned(s >> 122);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __device__ __forceinline__ double next_double() {
    return double(next() >> 11) * (1.0 / 9007199254740992.0);
  }
};

// affine map s -> a*s + c equal to `delta` LCG steps
struct Jump {
  u128 a, c;
};

__host__ __device__ Jump make_jump(uint64_t delta, u128 inc) {
  u128 am = 1, ap = 0, cm = mk(kMulHi, kMulLo), cp = inc;
  while (delta) {
    if (delta & 1) {
      am = am * cm;
      ap = ap * cm + cp;
    }
    cp = (cm + 1) * cp;
    cm = cm * cm;
    delta >>= 1;
  }
  return Jump{am, ap};
}

struct RmatArgs {
  int32_t scale;
  int64_t m;
  double base[4];
  uint64_t s_hi, s_lo, i_hi, i_lo;
  uint64_t jlev_a_hi, jlev_a_lo, jlev_c_hi, jlev_c_lo;  // jump by 5m
};

constexpr int kGenChunk = 16;

__global__ void k_rmat(RmatArgs a, int64_t* src, int64_t* dst) {
  const u128 inc = mk(a.i_hi, a.i_lo);
  const u128 s0 = mk(a.s_hi, a.s_lo);
  const u128 ja = mk(a.jlev_a_hi, a.jlev_a_lo), jc = mk(a.jlev_c_hi, a.jlev_c_lo);
  const int64_t chunks = (a.m + kGenChunk - 1) / kGenChunk;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < chunks; c += stride) {
    const int64_t e0 = c * kGenChunk;
    const Jump jn = make_jump(uint64_t(4 * e0), inc);
    const Jump jr = make_jump(uint64_t(4 * a.m + e0), inc);
    u128 sn0 = jn.a * s0 + jn.c;  // level-0 state before edge e's noise block
    u128 sr0 = jr.a * s0 + jr.c;  // level-0 state before edge e's quadrant draw
    const int64_t e1 = e0 + kGenChunk < a.m ? e0 + kGenChunk : a.m;
    for (int64_t e = e0; e < e1; ++e) {
      int64_t u = 0, v = 0;
      Pcg pn{sn0, inc}, pr{sr0, inc};
      for (int lev = 0; lev < a.scale; ++lev) {
        Pcg qn = pn, qr = pr;
        double p[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double r = qn.next_double();
          p[j] = __dmul_rn(a.base[j], __dadd_rn(0.9, __dmul_rn(0.2, r)));
        }
        const double sum = __dadd_rn(__dadd_rn(__dadd_rn(p[0], p[1]), p[2]), p[3]);
        double cut = 0.0;
        const double r = qr.next_double();
        int quad = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double pj = __ddiv_rn(p[j], sum);
          cut = j == 0 ? pj : __dadd_rn(cut, pj);
          quad += r >= cut;
        }
        quad = quad < 3 ? quad : 3;
        const int64_t bit = int64_t(1) << (a.scale - 1 - lev);
        u += bit * (quad >= 2);
        v += bit * (quad & 1);
        pn.s = ja * pn.s + jc;
        pr.s = ja * pr.s + jc;
      }
      src[e] = u;
      dst[e] = v;
      // next edge: 4 noise draws and 1 quadrant draw later
      {
        Pcg t{sn0, inc};
        t.next(); t.next(); t.next(); t.next();
        sn0 = t.s;
        Pcg t2{sr0, inc};
        t2.next();
        sr0 = t2.s;
      }
    }
  }
}

// numpy Generator.integers(0, 2^k, size=(K, 2), dtype=int64): 32-bit buffered
// Lemire draws without rejection (the threshold is 0 for a power of two);
// pair i consumes the low then the high half of raw draw i.
__global__ void k_uniform_pow2(int32_t log2n, int64_t k, uint64_t s_hi, uint64_t s_lo,
                               uint64_t i_hi, uint64_t i_lo, int64_t* src, int64_t* dst) {
  const u128 inc = mk(i_hi, i_lo);
  const u128 s0 = mk(s_hi, s_lo);
  const int64_t chunks = (k + kGenChunk - 1) / kGenChunk;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const unsigned sh = 32u - unsigned(log2n);
  for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < chunks; c += stride) {
    const int64_t e0 = c * kGenChunk;
    const Jump j = make_jump(uint64_t(e0), inc);
    Pcg p{j.a * s0 + j.c, inc};
    const int64_t e1 = e0 + kGenChunk < k ? e0 + kGenChunk : k;
    for (int64_t e = e0; e < e1; ++e) {
      const uint64_t x = p.next();
      src[e] = int64_t(uint32_t(x) >> sh);
      dst[e] = int64_t(uint32_t(x >> 32) >> sh);
    }
  }
}

// ------------------------------------------------------------- CSR build ---
int key_bits(int64_t n) {
  int b = 1;
  while ((int64_t(1) << b) < n) ++b;
  return b;
}

__global__ void k_sym_keys(const int64_t* src, const int64_t* dst, int64_t k, int64_t n, int bits,
                           unsigned long long* keys, unsigned long long* bad) {
  const unsigned long long dead = ~0ull;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < k; i += stride) {
    const int64_t u = src[i], v = dst[i];
    if (u < 0 || v < 0 || u >= n || v >= n) {
      atomicMin(bad, static_cast<unsigned long long>(i));
      keys[2 * i] = keys[2 * i + 1] = dead;
      continue;
    }
    if (u == v) {
      keys[2 * i] = keys[2 * i + 1] = dead;  // self-loops dropped (graphs.py:109-110)
      continue;
    }
    keys[2 * i] = (static_cast<unsigned long long>(u) << bits) | static_cast<unsigned long long>(v);
    keys[2 * i + 1] = (static_cast<unsigned long long>(v) << bits) | static_cast<unsigned long long>(u);
  }
}

__global__ void k_csr_fill(const unsigned long long* keys, int64_t m, int64_t n, int bits,
                           int64_t* off, int32_t* tgt) {
  const unsigned long long mask = (1ull << bits) - 1ull;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j <= m; j += stride) {
    const int64_t u = j < m ? int64_t(keys[j] >> bits) : n;
    const int64_t up = j > 0 ? int64_t(keys[j - 1] >> bits) : -1;
    for (int64_t w = up + 1; w <= u; ++w) off[w] = j;  // rows (up, u] start at j
    if (j < m) tgt[j] = int32_t(keys[j] & mask);
  }
}

struct CsrWs {
  unsigned long long* keys;
  unsigned long long* keys2;
  unsigned long long* uniq;
  unsigned long long* ctr;
  void* tmp;
  size_t tmp_bytes;
};

template <class A>
void csr_carve(A& a, CsrWs& w, int64_t n, int64_t k) {
  const int64_t kk = 2 * k;
  w.keys = a.template take<unsigned long long>(kk);
  w.keys2 = a.template take<unsigned long long>(kk);
  w.uniq = w.keys;  // unique output reuses the first buffer
  w.ctr = a.template take<unsigned long long>(8);
  size_t b1 = 0, b2 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, b1, static_cast<unsigned long long*>(nullptr),
                                 static_cast<unsigned long long*>(nullptr), kk, 0, 64);
  cub::DeviceSelect::Unique(nullptr, b2, static_cast<unsigned long long*>(nullptr),
                            static_cast<unsigned long long*>(nullptr),
                            static_cast<unsigned long long*>(nullptr), kk);
  w.tmp_bytes = b1 > b2 ? b1 : b2;
  w.tmp = a.template take<char>(int64_t(w.tmp_bytes));
  (void)n;
}

}  // namespace

}  // namespace gc

using namespace gc;

extern "C" {

int gc_gen_rmat(int32_t scale, int64_t num_pairs, const double* base_host, uint64_t state_hi,
                uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t* src, int64_t* dst,
                void* stream) {
  return guarded([&] {
    require(scale >= 1 && scale <= 31, GC_ERR_CONFIG, "scale must be in [1, 31]");
    require(num_pairs >= 0, GC_ERR_ARG, "negative pair count");
    if (num_pairs == 0) return;
    RmatArgs a{};
    a.scale = scale;
    a.m = num_pairs;
    for (int j = 0; j < 4; ++j) a.base[j] = base_host[j];
    a.s_hi = state_hi;
    a.s_lo = state_lo;
    a.i_hi = inc_hi;
    a.i_lo = inc_lo;
    const Jump jl = make_jump(uint64_t(5 * num_pairs), mk(inc_hi, inc_lo));
    a.jlev_a_hi = uint64_t(jl.a >> 64);
    a.jlev_a_lo = uint64_t(jl.a);
    a.jlev_c_hi = uint64_t(jl.c >> 64);
    a.jlev_c_lo = uint64_t(jl.c);
    const int64_t chunks = (num_pairs + kGenChunk - 1) / kGenChunk;
    (k_rmat<<<grid_for(chunks, 128, 16), 128, 0, static_cast<cudaStream_t>(stream)>>>(a, src, dst), ::gc::count_launch());
    GC_CHECK_LAUNCH();
  });
}

int gc_gen_uniform_pow2(int32_t log2n, int64_t num_pairs, uint64_t state_hi, uint64_t state_lo,
                        uint64_t inc_hi, uint64_t inc_lo, int64_t* src, int64_t* dst, void* stream) {
  return guarded([&] {
    require(log2n >= 1 && log2n <= 31, GC_ERR_CONFIG, "log2n must be in [1, 31]");
    if (num_pairs <= 0) return;
    const int64_t chunks = (num_pairs + kGenChunk - 1) / kGenChunk;
    (k_uniform_pow2<<<grid_for(chunks, 128, 16), 128, 0, static_cast<cudaStream_t>(stream)>>>(
        log2n, num_pairs, state_hi, state_lo, inc_hi, inc_lo, src, dst), ::gc::count_launch());
    GC_CHECK_LAUNCH();
  });
}

size_t gc_build_csr_workspace(int64_t n, int64_t k) {
  Sizer s;
  CsrWs w{};
  csr_carve(s, w, n, k);
  return s.used + 1024;
}

int gc_build_csr(int64_t n, const int64_t* src, const int64_t* dst, int64_t k, int64_t* offsets,
                 int32_t* targets, int64_t* m_out, void* ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    require(n >= 0 && n < (int64_t(1) << 31), GC_ERR_MALFORMED, "vertex count outside [0, 2^31)");
    require(k >= 0 && m_out != nullptr, GC_ERR_ARG, "bad arguments");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    *m_out = 0;
    if (n == 0) return;
    Arena a(ws, ws_bytes);
    CsrWs w{};
    csr_carve(a, w, n, k);
    const int bits = key_bits(n);
    const unsigned long long sentinel = ~0ull;
    GC_CUDA(cudaMemsetAsync(w.ctr, 0, 64, st));
    GC_CUDA(cudaMemcpyAsync(w.ctr, &sentinel, 8, cudaMemcpyHostToDevice, st));
    int64_t m = 0;
    if (k > 0) {
      (k_sym_keys<<<grid_for(k, 256, 16), 256, 0, st>>>(src, dst, k, n, bits, w.keys, w.ctr), ::gc::count_launch());
      GC_CHECK_LAUNCH();
      unsigned long long bad = 0;
      GC_CUDA(cudaMemcpyAsync(&bad, w.ctr, 8, cudaMemcpyDeviceToHost, st));
      GC_CUDA(cudaStreamSynchronize(st));
      require(bad == sentinel, GC_ERR_MALFORMED,
              "edge " + std::to_string(bad) + " has an endpoint outside [0, " + std::to_string(n) + ")");
      size_t tb = w.tmp_bytes;
      // sort all 64 bits: the dead sentinel keys (self-loops) land at the end
      GC_CUDA(cub::DeviceRadixSort::SortKeys(w.tmp, tb, w.keys, w.keys2, 2 * k, 0, 64, st));
      tb = w.tmp_bytes;
      GC_CUDA(cub::DeviceSelect::Unique(w.tmp, tb, w.keys2, w.keys, w.ctr + 1, 2 * k, st));
      unsigned long long nu = 0, last = 0;
      GC_CUDA(cudaMemcpyAsync(&nu, w.ctr + 1, 8, cudaMemcpyDeviceToHost, st));
      GC_CUDA(cudaStreamSynchronize(st));
      if (nu > 0) {
        GC_CUDA(cudaMemcpyAsync(&last, w.keys + (nu - 1), 8, cudaMemcpyDeviceToHost, st));
        GC_CUDA(cudaStreamSynchronize(st));
      }
      m = int64_t(nu) - (nu > 0 && last == sentinel ? 1 : 0);
    }
    (k_csr_fill<<<grid_for(m + 1, 256, 16), 256, 0, st>>>(w.keys, m, n, bits, offsets, targets), ::gc::count_launch());
    GC_CHECK_LAUNCH();
    GC_CUDA(cudaStreamSynchronize(st));
    *m_out = m;
  });
}

// MT19937 (Python's random.Random) continuing from a getstate() snapshot:
// out[i] = getrandbits(32) for i = 0..n-1.
int gc_mt19937_fill(const uint32_t* state624, int32_t index, uint32_t* out, int64_t n) {
  return guarded([&] {
    require(state624 && out && n >= 0, GC_ERR_ARG, "bad arguments");
    uint32_t mt[624];
    for (int i = 0; i < 624; ++i) mt[i] = state624[i];
    int mti = index;
    for (int64_t k = 0; k < n; ++k) {
      if (mti >= 624) {
        for (int i = 0; i < 624; ++i) {
          const uint32_t y = (mt[i] & 0x80000000u) | (mt[(i + 1) % 624] & 0x7fffffffu);
          mt[i] = mt[(i + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        mti = 0;
      }
      uint32_t y = mt[mti++];
      y ^= y >> 11;
      y ^= (y << 7) & 0x9d2c5680u;
      y ^= (y << 15) & 0xefc60000u;
      y ^= y >> 18;
      out[k] = y;
    }
  });
}

}  // extern "C"
