// comm.cu — the single-process multi-device C ABI (gc_comm_init
// plus sharded variants taking a gc_comm*).  The reference is threads only
// (parallel.py:39-63) and has no counterpart; this is the C caller's route
// to the sharded pipeline that distributed.py drives through
// torch.distributed: one communicator over N devices of one box
// (ncclCommInitAll, NVLink / NVSwitch), each device holding one CSR row block
// and a full-length parent replica, the two exchange points of the
// two-phase pipeline as NCCL all-gathers of merging-edge lists,
// and BFS sampling as the distributed level-synchronous traversal of
// dbfs.cu (frontier marks all-gathered, next frontiers all-reduced).
//
// A communicator whose device list repeats one device runs in loopback
// mode: the ranks share that device and every collective is a stream-ordered
// device copy.  That is how the orchestration is exercised on a one-GPU box;
// a list of distinct devices always goes through NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.h"
#include "pipeline.cuh"

struct gc_comm {
  int ndev = 0;
  bool loopback = false;
  std::vector<int> devs;
  std::vector<ncclComm_t> nccl;
  std::vector<cudaStream_t> st;
};

namespace gc {
namespace {

// NCCL is resolved at gc_comm_init time (dlopen of libnccl.so.2: the one
// torch already loaded, else the system's), so libgconn.so itself has no
// link-time NCCL dependency and loads on hosts without it.
struct Nccl {
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl t;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      t.CommInitAll = reinterpret_cast<decltype(t.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
      t.CommDestroy = reinterpret_cast<decltype(t.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
      t.GroupStart = reinterpret_cast<decltype(t.GroupStart)>(dlsym(h, "ncclGroupStart"));
      t.GroupEnd = reinterpret_cast<decltype(t.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
      t.AllGather = reinterpret_cast<decltype(t.AllGather)>(dlsym(h, "ncclAllGather"));
      t.AllReduce = reinterpret_cast<decltype(t.AllReduce)>(dlsym(h, "ncclAllReduce"));
      t.GetErrorString = reinterpret_cast<decltype(t.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    }
  }
  if (!t.CommInitAll || !t.AllGather || !t.AllReduce || !t.GroupStart || !t.GroupEnd)
    throw Error(GC_ERR_CUDA, "NCCL (libnccl.so.2) not found: multi-device communicators need it");
  return t;
}

#define GC_NCCL(x)                                                                                  \
  do {                                                                                              \
    ncclResult_t r_ = (x);                                                                          \
    if (r_ != ncclSuccess)                                                                          \
      throw Error(GC_ERR_CUDA, std::string("NCCL: ") +                                              \
                                   (nccl().GetErrorString ? nccl().GetErrorString(r_) : "error")); \
  } while (0)

void check(int status) {
  if (status != GC_OK) throw Error(status, gc_last_error());
}

// per-rank device scratch of one call (freed at the end).  cnt: 8 words —
// [0] list / claim counts, [1] sticky malformed-mark flag, [2] degree sum
// (gc_dbfs_finish)
struct RankBufs {
  void* ws = nullptr;
  size_t wsb = 0;
  int32_t* mu = nullptr;   // merging edges (capacity n)
  int32_t* mv = nullptr;
  int32_t* send = nullptr;  // padded exchange buffers
  int32_t* recv = nullptr;
  int32_t* aux = nullptr;   // hooks / locks
  unsigned long long* cnt = nullptr;
  int32_t* fu = nullptr;    // forest output (own + foreign merges)
  int32_t* fv = nullptr;
  int64_t fcount = 0;
  // dbfs
  uint32_t *F = nullptr, *V = nullptr, *M = nullptr, *N = nullptr, *par = nullptr;
  size_t xcap = 0;          // send / recv capacity (int32 entries)
};

struct Call {
  gc_comm* c;
  std::vector<RankBufs> b;
  explicit Call(gc_comm* cc) : c(cc), b(cc->ndev) {}
  ~Call() {
    for (int r = 0; r < c->ndev; ++r) {
      cudaSetDevice(c->devs[r]);
      // (fu / fv are the caller's forest outputs)
      for (void* p : {b[r].ws, (void*)b[r].mu, (void*)b[r].mv, (void*)b[r].send, (void*)b[r].recv,
                      (void*)b[r].aux, (void*)b[r].cnt, (void*)b[r].F, (void*)b[r].V, (void*)b[r].M,
                      (void*)b[r].N, (void*)b[r].par})
        if (p) cudaFree(p);
    }
  }
  void dev(int r) const { GC_CUDA(cudaSetDevice(c->devs[r])); }
  void sync_all() const {
    for (int r = 0; r < c->ndev; ++r) {
      dev(r);
      GC_CUDA(cudaStreamSynchronize(c->st[r]));
    }
  }
  void ensure_x(int r, size_t entries) {
    RankBufs& x = b[r];
    if (entries <= x.xcap) return;
    dev(r);
    if (x.send) cudaFree(x.send);
    if (x.recv) cudaFree(x.recv);
    x.send = x.recv = nullptr;
    GC_CUDA(cudaMalloc(&x.send, entries * 4));
    GC_CUDA(cudaMalloc(&x.recv, entries * 4 * size_t(c->ndev)));
    x.xcap = entries;
  }
  // all-gather `len` int32 per rank from send into recv (rank-major)
  void all_gather(size_t len) {
    if (len == 0) return;
    if (c->loopback) {
      dev(0);
      for (int r = 0; r < c->ndev; ++r)
        for (int s = 0; s < c->ndev; ++s)
          GC_CUDA(cudaMemcpyAsync(b[r].recv + size_t(s) * len, b[s].send, len * 4, cudaMemcpyDeviceToDevice,
                                  c->st[r]));
      // the ranks share the device: order every rank after every copy
      sync_all();
      return;
    }
    GC_NCCL(nccl().GroupStart());
    for (int r = 0; r < c->ndev; ++r)
      GC_NCCL(nccl().AllGather(b[r].send, b[r].recv, len, ncclInt32, c->nccl[r], c->st[r]));
    GC_NCCL(nccl().GroupEnd());
  }
  // all-reduce SUM of `len` int32 in place (buffer per rank)
  void all_reduce_sum(std::vector<int32_t*> bufs, size_t len) {
    if (len == 0) return;
    if (c->loopback) {
      // sum into rank 0's buffer, then copy back (one device, stream-ordered)
      sync_all();
      dev(0);
      for (int s = 1; s < c->ndev; ++s) launch_add(bufs[0], bufs[s], len, c->st[0]);
      for (int s = 1; s < c->ndev; ++s)
        GC_CUDA(cudaMemcpyAsync(bufs[s], bufs[0], len * 4, cudaMemcpyDeviceToDevice, c->st[0]));
      GC_CUDA(cudaStreamSynchronize(c->st[0]));
      return;
    }
    GC_NCCL(nccl().GroupStart());
    for (int r = 0; r < c->ndev; ++r)
      GC_NCCL(nccl().AllReduce(bufs[r], bufs[r], len, ncclInt32, ncclSum, c->nccl[r], c->st[r]));
    GC_NCCL(nccl().GroupEnd());
  }
  static void launch_add(int32_t* dst, const int32_t* src, size_t len, cudaStream_t st);
};

__global__ void k_add_i32(int32_t* dst, const int32_t* src, int64_t len) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < len; i += stride)
    dst[i] = int32_t(uint32_t(dst[i]) + uint32_t(src[i]));
}

void Call::launch_add(int32_t* dst, const int32_t* src, size_t len, cudaStream_t st) {
  (k_add_i32<<<grid_for(int64_t(len), 256, 4), 256, 0, st>>>(dst, src, int64_t(len)), count_launch());
  GC_CHECK_LAUNCH();
}

unsigned long long read_u64(const unsigned long long* d, cudaStream_t st) {
  unsigned long long h = 0;
  GC_CUDA(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st));
  GC_CUDA(cudaStreamSynchronize(st));
  return h;
}

// One exchange point: all-gather every rank's merging-edge list (mu, mv,
// count in cnt) and union the foreign lists into each replica, recording
// the edges that merged trees there when a forest is kept.
void exchange(Call& k, const gc_spec& s, int64_t n, std::vector<int32_t*>& parent, bool forest) {
  gc_comm* c = k.c;
  std::vector<int64_t> cnt(c->ndev);
  for (int r = 0; r < c->ndev; ++r) {
    k.dev(r);
    cnt[r] = int64_t(read_u64(k.b[r].cnt, c->st[r]));
  }
  const int64_t kmax = *std::max_element(cnt.begin(), cnt.end());
  if (kmax == 0) return;
  for (int r = 0; r < c->ndev; ++r) {
    k.ensure_x(r, size_t(2 * kmax));
    k.dev(r);
    RankBufs& x = k.b[r];
    GC_CUDA(cudaMemcpyAsync(x.send, x.mu, cnt[r] * 4, cudaMemcpyDeviceToDevice, c->st[r]));
    GC_CUDA(cudaMemcpyAsync(x.send + kmax, x.mv, cnt[r] * 4, cudaMemcpyDeviceToDevice, c->st[r]));
    if (forest && cnt[r]) {  // own merges are forest edges
      GC_CUDA(cudaMemcpyAsync(x.fu + x.fcount, x.mu, cnt[r] * 4, cudaMemcpyDeviceToDevice, c->st[r]));
      GC_CUDA(cudaMemcpyAsync(x.fv + x.fcount, x.mv, cnt[r] * 4, cudaMemcpyDeviceToDevice, c->st[r]));
      x.fcount += cnt[r];
    }
  }
  if (c->loopback) k.sync_all();
  k.all_gather(size_t(2 * kmax));
  for (int r = 0; r < c->ndev; ++r) {
    k.dev(r);
    RankBufs& x = k.b[r];
    for (int q = 0; q < c->ndev; ++q) {
      if (q == r || cnt[q] == 0) continue;
      const int32_t* us = x.recv + size_t(q) * 2 * kmax;
      const int32_t* vs = us + kmax;
      if (forest) {
        GC_CUDA(cudaMemsetAsync(x.cnt, 0, 8, c->st[r]));  // the list call accumulates into its count
        check(gc_union_edges_list(parent[r], n, us, vs, cnt[q], &s, x.aux, x.fu + x.fcount, x.fv + x.fcount,
                                  x.cnt, c->st[r]));
        x.fcount += int64_t(read_u64(x.cnt, c->st[r]));
      } else {
        check(gc_union_edges(parent[r], n, us, vs, cnt[q], &s, x.aux, nullptr, nullptr, c->st[r]));
      }
    }
  }
  if (c->loopback) k.sync_all();
}

// distributed BFS sampling (dbfs.cu) over the communicator; leaves the
// identical global labels in every parent[r] and, with a forest, the whole
// BFS tree in every rank's forest output
int64_t run_dbfs(Call& k, const gc_csr* shards, const int64_t* lo, const int64_t* hi, const gc_spec& s, int64_t n,
                 std::vector<int32_t*>& parent, bool forest) {
  gc_comm* c = k.c;
  const int64_t words = (n + 31) / 32;
  // global source: the probes' degrees summed over the owning ranks
  // (sampling.py:130-132); the probe ids come with the spec
  int64_t src = s.bfs_source;
  require(src >= 0 && src < n, GC_ERR_ARG, "BFS sampling needs spec->bfs_source (the probe vertex)");
  for (int r = 0; r < c->ndev; ++r) {
    k.dev(r);
    RankBufs& x = k.b[r];
    GC_CUDA(cudaMalloc(&x.F, words * 4));
    GC_CUDA(cudaMalloc(&x.V, words * 4));
    GC_CUDA(cudaMalloc(&x.M, words * 4));
    GC_CUDA(cudaMalloc(&x.N, words * 4));
    GC_CUDA(cudaMalloc(&x.par, n * 4));
    check(gc_dbfs_init(n, src, x.F, x.V, x.par, c->st[r]));
  }
  int64_t nf = 1, reached = 1;
  bool bottom_up = false;
  while (nf) {
    bottom_up = bottom_up ? nf >= n / 24 : nf * 14 > n - reached;  // Beamer, as distributed.py
    if (!bottom_up) {
      std::vector<int64_t> cnt(c->ndev);
      for (int r = 0; r < c->ndev; ++r) {
        k.dev(r);
        RankBufs& x = k.b[r];
        check(gc_dbfs_marks(&shards[r], lo[r], hi[r], x.F, x.V, x.M, x.mu, x.cnt, c->st[r]));
        cnt[r] = int64_t(read_u64(x.cnt, c->st[r]));
      }
      const int64_t kmax = *std::max_element(cnt.begin(), cnt.end());
      if (kmax) {
        for (int r = 0; r < c->ndev; ++r) {
          k.ensure_x(r, size_t(kmax));
          k.dev(r);
          GC_CUDA(cudaMemsetAsync(k.b[r].send, 0xff, kmax * 4, c->st[r]));
          GC_CUDA(cudaMemcpyAsync(k.b[r].send, k.b[r].mu, cnt[r] * 4, cudaMemcpyDeviceToDevice, c->st[r]));
        }
        if (c->loopback) k.sync_all();
        k.all_gather(size_t(kmax));
        for (int r = 0; r < c->ndev; ++r) {
          k.dev(r);
          for (int q = 0; q < c->ndev; ++q)
            if (q != r && cnt[q])
              check(gc_dbfs_merge_marks(n, k.b[r].recv + size_t(q) * kmax, cnt[q], k.b[r].M,
                                        reinterpret_cast<unsigned int*>(k.b[r].cnt + 1), c->st[r]));
        }
        if (c->loopback) k.sync_all();
      }
    }
    std::vector<int32_t*> nb(c->ndev);
    for (int r = 0; r < c->ndev; ++r) {
      k.dev(r);
      RankBufs& x = k.b[r];
      check(gc_dbfs_claim(&shards[r], lo[r], hi[r], x.F, x.V, bottom_up ? nullptr : x.M, x.par, x.N, x.cnt,
                          c->st[r]));
      nb[r] = reinterpret_cast<int32_t*>(x.N);
    }
    k.all_reduce_sum(nb, size_t(words));  // disjoint owned bits: SUM == OR
    for (int r = 0; r < c->ndev; ++r) {
      k.dev(r);
      check(gc_dbfs_advance(n, k.b[r].V, k.b[r].F, k.b[r].N, k.b[r].cnt, c->st[r]));
    }
    k.dev(0);
    nf = int64_t(read_u64(k.b[0].cnt, c->st[0]));
    reached += nf;
    if (!c->loopback) k.sync_all();
  }
  int64_t insp = 0;
  for (int r = 0; r < c->ndev; ++r) {
    k.dev(r);
    RankBufs& x = k.b[r];
    check(gc_dbfs_finish(&shards[r], lo[r], hi[r], x.V, x.par, parent[r], x.mu, x.mv, x.cnt, x.cnt + 2, x.ws,
                         x.wsb, c->st[r]));
    insp += int64_t(read_u64(x.cnt + 2, c->st[r]));
    require(read_u64(x.cnt + 1, c->st[r]) == 0, GC_ERR_MALFORMED, "a merged frontier mark lies outside [0, n)");
  }
  // the tree edges: every rank's own, gathered into every forest
  if (forest) {
    std::vector<int64_t> cnt(c->ndev);
    for (int r = 0; r < c->ndev; ++r) {
      k.dev(r);
      cnt[r] = int64_t(read_u64(k.b[r].cnt, c->st[r]));
    }
    const int64_t kmax = *std::max_element(cnt.begin(), cnt.end());
    if (kmax) {
      for (int r = 0; r < c->ndev; ++r) {
        k.ensure_x(r, size_t(2 * kmax));
        k.dev(r);
        GC_CUDA(cudaMemcpyAsync(k.b[r].send, k.b[r].mu, cnt[r] * 4, cudaMemcpyDeviceToDevice, c->st[r]));
        GC_CUDA(cudaMemcpyAsync(k.b[r].send + kmax, k.b[r].mv, cnt[r] * 4, cudaMemcpyDeviceToDevice, c->st[r]));
      }
      if (c->loopback) k.sync_all();
      k.all_gather(size_t(2 * kmax));
      for (int r = 0; r < c->ndev; ++r) {
        k.dev(r);
        RankBufs& x = k.b[r];
        for (int q = 0; q < c->ndev; ++q) {
          const int32_t* us = x.recv + size_t(q) * 2 * kmax;
          GC_CUDA(cudaMemcpyAsync(x.fu + x.fcount, us, cnt[q] * 4, cudaMemcpyDeviceToDevice, c->st[r]));
          GC_CUDA(cudaMemcpyAsync(x.fv + x.fcount, us + kmax, cnt[q] * 4, cudaMemcpyDeviceToDevice, c->st[r]));
          x.fcount += cnt[q];
        }
      }
    }
  }
  return insp;
}

void run_sharded(gc_comm* c, const gc_csr* shards, const int64_t* lo, const int64_t* hi, const gc_spec* spec,
                 int32_t* const* labels, int32_t* const* fu_out, int32_t* const* fv_out, int64_t* forest_count,
                 gc_stats* stats) {
  require(c && shards && lo && hi && spec && labels, GC_ERR_ARG, "null argument");
  const gc_spec& s = *spec;
  require(s.finish >= GC_FINISH_ASYNC && s.finish <= GC_FINISH_JTB, GC_ERR_CONFIG, "sharded connectivity needs a union-find finish");
  require(s.finish != GC_FINISH_JTB, GC_ERR_CONFIG, "JTB ranks are per-device state: not sharded");
  require(s.sample == GC_SAMPLE_NONE || s.sample == GC_SAMPLE_KOUT || s.sample == GC_SAMPLE_HB ||
              s.sample == GC_SAMPLE_BFS,
          GC_ERR_CONFIG, "sharded sampling supports none / k-out / hb / bfs");
  const bool forest = fu_out != nullptr;
  require(!forest || (fv_out && forest_count), GC_ERR_ARG, "forest needs fu, fv and a count");
  require(!forest || s.splice != GC_SPLICE_ATOMIC, GC_ERR_CONFIG,
          "the atomic splice is not root-based: no spanning forest");
  const int64_t n = shards[0].n;
  for (int r = 0; r < c->ndev; ++r) {
    require(shards[r].n == n, GC_ERR_ARG, "every shard spans the same vertex set");
    require(lo[r] >= 0 && lo[r] <= hi[r] && hi[r] <= n, GC_ERR_ARG, "row block outside [0, n]");
    require(labels[r] != nullptr || n == 0, GC_ERR_ARG, "null labels");
  }
  Call k(c);
  std::vector<int32_t*> parent(labels, labels + c->ndev);
  int64_t insp_s = 0, insp_f = 0;
  gc_stats st0{};
  if (n > 0) {
    for (int r = 0; r < c->ndev; ++r) {
      k.dev(r);
      RankBufs& x = k.b[r];
      x.wsb = gc_workspace_size(n, shards[r].m, spec);
      const size_t fin = size_t(n) * 4 + 8192;
      x.wsb = x.wsb > fin ? x.wsb : fin;
      GC_CUDA(cudaMalloc(&x.ws, x.wsb));
      GC_CUDA(cudaMalloc(&x.mu, n * 4));
      GC_CUDA(cudaMalloc(&x.mv, n * 4));
      GC_CUDA(cudaMalloc(&x.cnt, 64));
      GC_CUDA(cudaMemsetAsync(x.cnt, 0, 64, c->st[r]));
      if (s.finish == GC_FINISH_HOOKS || s.finish == GC_FINISH_REM_LOCK) GC_CUDA(cudaMalloc(&x.aux, n * 4));
      if (forest) {
        x.fu = fu_out[r];
        x.fv = fv_out[r];
      }
    }
    auto reset_aux = [&] {
      for (int r = 0; r < c->ndev; ++r)
        if (k.b[r].aux) {
          k.dev(r);
          fill(k.b[r].aux, n, s.finish == GC_FINISH_HOOKS ? int32_t(n) : 0, c->st[r]);
        }
    };
    // phase 1: sample (each rank its rows; BFS: one distributed traversal)
    if (s.sample == GC_SAMPLE_BFS) {
      insp_s = run_dbfs(k, shards, lo, hi, s, n, parent, forest);
    } else {
      for (int r = 0; r < c->ndev; ++r) {
        k.dev(r);
        gc_stats st{};
        check(gc_shard_sample(&shards[r], spec, lo[r], hi[r], parent[r], k.b[r].mu, k.b[r].mv, k.b[r].cnt, &st,
                              k.b[r].ws, k.b[r].wsb, c->st[r]));
        insp_s += st.insp_sample;
      }
      reset_aux();
      exchange(k, s, n, parent, forest);
    }
    // phase 2: finish over each rank's active rows, exchange again
    for (int r = 0; r < c->ndev; ++r) {
      k.dev(r);
      gc_stats st{};
      check(gc_shard_finish(&shards[r], spec, lo[r], hi[r], parent[r], k.b[r].mu, k.b[r].mv, k.b[r].cnt, &st,
                            k.b[r].ws, k.b[r].wsb, c->st[r]));
      insp_f += st.insp_finish;
      if (r == 0) st0 = st;
    }
    reset_aux();
    exchange(k, s, n, parent, forest);
    for (int r = 0; r < c->ndev; ++r) {
      k.dev(r);
      check(gc_label_finalization(parent[r], n, k.b[r].ws, k.b[r].wsb, c->st[r]));
    }
    k.sync_all();
  }
  if (forest)
    for (int r = 0; r < c->ndev; ++r) forest_count[r] = k.b[r].fcount;
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->insp_sample = insp_s;
    stats->insp_finish = insp_f;
    stats->l_max = st0.l_max;
    stats->lmax_count = st0.lmax_count;
    stats->n_active = st0.n_active;
  }
}

}  // namespace
}  // namespace gc

using namespace gc;

extern "C" {

int gc_comm_init(int ndev, const int* devs, gc_comm** out) {
  return guarded([&] {
    require(ndev >= 1 && devs && out, GC_ERR_ARG, "bad communicator arguments");
    gc_comm* c = new gc_comm();
    c->ndev = ndev;
    c->devs.assign(devs, devs + ndev);
    std::vector<int> sorted(c->devs);
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    const bool same = sorted.front() == sorted.back();
    try {
      require(distinct || same, GC_ERR_ARG, "devices must be all distinct (NCCL) or all one device (loopback)");
      c->loopback = ndev > 1 && same;
      c->st.resize(ndev);
      for (int r = 0; r < ndev; ++r) {
        GC_CUDA(cudaSetDevice(c->devs[r]));
        GC_CUDA(cudaStreamCreateWithFlags(&c->st[r], cudaStreamNonBlocking));
      }
      if (!c->loopback) {
        c->nccl.resize(ndev);
        GC_NCCL(nccl().CommInitAll(c->nccl.data(), ndev, c->devs.data()));
      }
    } catch (...) {
      gc_comm_destroy(c);
      throw;
    }
    *out = c;
  });
}

void gc_comm_destroy(gc_comm* c) {
  if (!c) return;
  for (auto& m : c->nccl)
    if (m) nccl().CommDestroy(m);
  for (int r = 0; r < int(c->st.size()); ++r)
    if (c->st[r]) {
      cudaSetDevice(c->devs[r]);
      cudaStreamDestroy(c->st[r]);
    }
  delete c;
}

int gc_comm_size(const gc_comm* c) { return c ? c->ndev : -1; }

int gc_comm_is_loopback(const gc_comm* c) { return c && c->loopback ? 1 : 0; }

int gc_comm_static_cc(gc_comm* c, const gc_csr* shards, const int64_t* row_lo, const int64_t* row_hi,
                      const gc_spec* spec, int32_t* const* labels, gc_stats* stats) {
  return guarded([&] { run_sharded(c, shards, row_lo, row_hi, spec, labels, nullptr, nullptr, nullptr, stats); });
}

int gc_comm_spanning_forest(gc_comm* c, const gc_csr* shards, const int64_t* row_lo, const int64_t* row_hi,
                            const gc_spec* spec, int32_t* const* labels, int32_t* const* fu, int32_t* const* fv,
                            int64_t* forest_count, gc_stats* stats) {
  return guarded([&] {
    require(fu && fv && forest_count, GC_ERR_ARG, "null forest outputs");
    run_sharded(c, shards, row_lo, row_hi, spec, labels, fu, fv, forest_count, stats);
  });
}

}  // extern "C"
