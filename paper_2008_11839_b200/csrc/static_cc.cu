// static_cc.cu — the two-phase static pipeline (driver.py:454-507) and its
// spanning-forest / finish-only / finalisation entry points.
//
//   sample  : init sets -> sampler (k-out / HB / BFS / LDD) -> compress
//             -> most-frequent label L_max                 (driver.py:465-471)
//   census  : optional post-sample copy + ic count, untimed (driver.py:495)
//   finish  : active gather -> union-find rows or min-label rounds
//                                                           (driver.py:473-481)
//   finalize: pointer jump + canonical labels              (driver.py:483-490)
//
// Every phase is a fixed kernel sequence on one stream with no host
// round-trip, except the round-based finishes which read a change flag per
// round (the reference's own fixpoint loop, minbased.py:124-304).
#include <climits>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "internal.h"
#include "pipeline.cuh"
#include "rounds.h"
#include "samplers.h"

namespace gc {

namespace {

struct EventSet {
  cudaEvent_t e[10];
  EventSet() {
    for (auto& x : e) GC_CUDA(cudaEventCreate(&x));
  }
  ~EventSet() {
    for (auto& x : e) cudaEventDestroy(x);
  }
};

// Keep the parent array resident in L2 for the duration of a pipeline: an
// access-policy window marks it persisting while CSR streams through with
// evict-first loads.  Released (and the persisting lines demoted) at the end.
struct L2Residency {
  cudaStream_t st;
  bool on = false;
  L2Residency(cudaStream_t s, void* base, size_t bytes) : st(s) {
    // opt-in only: on RMAT s24 it gains 1.5% (0.533 -> 0.525 ms), but a
    // captured plan keeps the lines persisting across replays, so they also
    // survive the benchmark's L2 flush between steps — not a fair default
    static const bool disabled = getenv("GC_L2_WINDOW") == nullptr;
    if (disabled) return;
    // not inside a stream capture: the persisting-cache reset at the end is
    // not a capturable operation (plans run without the window)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return;
    }
    static int max_persist = -1, max_window = 0;
    if (max_persist < 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
      cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
      if (max_persist > 0) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, size_t(max_persist));
      cudaGetLastError();
    }
    if (max_persist <= 0 || max_window <= 0 || bytes == 0) return;
    cudaStreamAttrValue a{};
    a.accessPolicyWindow.base_ptr = base;
    a.accessPolicyWindow.num_bytes = bytes < size_t(max_window) ? bytes : size_t(max_window);
    const double ratio = double(max_persist) / double(a.accessPolicyWindow.num_bytes);
    a.accessPolicyWindow.hitRatio = float(ratio < 1.0 ? ratio : 1.0);
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    on = cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a) == cudaSuccess;
    cudaGetLastError();
  }
  ~L2Residency() {
    if (!on) return;
    cudaStreamAttrValue a{};
    a.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a);
    cudaCtxResetPersistingL2Cache();
    cudaGetLastError();
  }
};


// Timing events: inside a stream capture they must become external event
// nodes of the graph; outside a capture the flag is rejected.
thread_local bool t_capturing = false;
cudaError_t rec(cudaEvent_t e, cudaStream_t st) {
  return t_capturing ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal) : cudaEventRecord(e, st);
}

bool is_union_finish(int f) { return f >= GC_FINISH_ASYNC && f <= GC_FINISH_JTB; }

UFConfig finish_cfg(const gc_spec& s) { return UFConfig{s.finish, s.find, s.splice}; }

// driver.py:96 — samplers use Async+Halve when the finish is not union-find
UFConfig sampler_cfg(const gc_spec& s) {
  if (is_union_finish(s.finish)) return finish_cfg(s);
  return UFConfig{GC_FINISH_ASYNC, GC_FIND_HALVE, GC_SPLICE_NONE};
}

void validate_spec(const gc_spec& s) {
  require(s.sample >= GC_SAMPLE_NONE && s.sample <= GC_SAMPLE_LDD, GC_ERR_CONFIG, "unknown sampler");
  require(s.finish >= GC_FINISH_ASYNC && s.finish <= GC_FINISH_LP, GC_ERR_CONFIG, "unknown finish");
  if (is_union_finish(s.finish))
    require(valid_uf(finish_cfg(s)), GC_ERR_CONFIG, "unsupported union-find combination");
  if (s.finish == GC_FINISH_LT) {
    require(s.lt_connect >= 0 && s.lt_connect <= 2 && s.lt_update >= 0 && s.lt_update <= 1 &&
                s.lt_shortcut >= 0 && s.lt_shortcut <= 1,
            GC_ERR_CONFIG, "invalid LT variant");
    require(!(s.lt_connect == GC_LT_CONNECT && !s.lt_alter), GC_ERR_CONFIG,
            "Connect requires the alter phase");
  }
  require(s.kout_k >= 1 || s.sample != GC_SAMPLE_KOUT, GC_ERR_CONFIG, "kout_k must be >= 1");
  if (s.finish == GC_FINISH_JTB || (s.sample == GC_SAMPLE_KOUT || s.sample == GC_SAMPLE_HB))
    require(sampler_cfg(s).unite != GC_FINISH_JTB || s.jtb_ranks != nullptr, GC_ERR_ARG,
            "JTB needs ranks");
}

void validate_csr(const gc_csr* g) {
  require(g != nullptr, GC_ERR_ARG, "null graph");
  require(g->n >= 0 && g->n < (int64_t(1) << 31), GC_ERR_MALFORMED, "vertex count outside [0, 2^31)");
  require(g->m >= 0, GC_ERR_MALFORMED, "negative edge count");
  require(g->n == 0 || g->offsets != nullptr, GC_ERR_ARG, "null offsets");
  require(g->m == 0 || g->targets != nullptr, GC_ERR_ARG, "null targets");
}

__global__ void k_split_pairs(const int2* __restrict__ pr, int32_t n, int32_t* fu, int32_t* fv,
                              unsigned long long* count) {
  unsigned long long c = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const int2 p = pr[v];
    fu[v] = p.x;
    fv[v] = p.y;
    c += p.x != -1;
  }
  block_add<kEwBlock>(count, c);
}

// Workspace layout shared by every static entry point.
// GC_LDD_CUT=0: rounds finishes after LDD gather their working COO from the
// active rows instead of taking the sampler's cut edges
bool ldd_cut_on() {
  static const bool on = [] {
    const char* e = getenv("GC_LDD_CUT");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class A>
struct Layout {
  unsigned long long* ctr = nullptr;
  int32_t* H = nullptr;
  int32_t* L = nullptr;
  int32_t* list = nullptr;
  int32_t* hist = nullptr;
  int2* fpair = nullptr;  // union-find forests of none / k-out / HB samplers
  RoundsWs rounds;
  SamplerWs samp;

  static bool pair_forest(const gc_spec& s) {
    return is_union_finish(s.finish) &&
           (s.sample == GC_SAMPLE_NONE || s.sample == GC_SAMPLE_KOUT || s.sample == GC_SAMPLE_HB);
  }

  void carve(A& a, int64_t n, int64_t m, const gc_spec& s, bool forest) {
    ctr = a.template take<unsigned long long>(C_COUNT_);
    if (forest && pair_forest(s)) fpair = a.template take<int2>(n);
    const UFConfig sc = sampler_cfg(s);
    const bool any_uf = is_union_finish(s.finish) || s.sample == GC_SAMPLE_KOUT || s.sample == GC_SAMPLE_HB;
    if (any_uf && sc.unite == GC_FINISH_HOOKS) H = a.template take<int32_t>(n);
    if (any_uf && sc.unite == GC_FINISH_REM_LOCK) L = a.template take<int32_t>(n);
    list = a.template take<int32_t>(n);
    hist = a.template take<int32_t>(n);
    if (!is_union_finish(s.finish)) rounds_carve(a, rounds, n, m, s, forest);
    sampler_carve(a, samp, n, m, s);
  }
};

struct Pipeline {
  const gc_csr& g;
  const gc_spec& s;
  int32_t* P;
  int32_t* fu;
  int32_t* fv;
  cudaStream_t st;
  Layout<Arena> ws;
  int32_t n;
  cudaEvent_t* kev = nullptr;  // [0,1] sampler kernel, [2,3] finish kernel
  bool timed_sample = false;
  int32_t* lu = nullptr;  // sharded drivers: merging edges of the union kernels
  int32_t* lv = nullptr;
  unsigned long long* lcount = nullptr;
  int64_t row_lo = 0, row_hi = -1;  // sharded drivers: the rows this block owns (-1: all)

  Pipeline(const gc_csr& g_, const gc_spec& s_, int32_t* P_, int32_t* fu_, int32_t* fv_,
           void* wsp, size_t wsb, cudaStream_t st_)
      : g(g_), s(s_), P(P_), fu(fu_), fv(fv_), st(st_), n(int32_t(g_.n)) {
    Arena a(wsp, wsb);
    ws.carve(a, g.n, g.m, s, fu != nullptr);
    zero_ctr(ws.ctr, C_COUNT_, st);
  }

  RowUnionArgs rows(const UFConfig& c) const {
    RowUnionArgs a{};
    a.P = P;
    a.H = c.unite == GC_FINISH_HOOKS ? ws.H : nullptr;
    a.L = c.unite == GC_FINISH_REM_LOCK ? ws.L : nullptr;
    a.R = s.jtb_ranks;
    a.fu = fu;
    a.fv = fv;
    a.fpair = fu ? ws.fpair : nullptr;
    a.n = n;
    a.off = g.offsets;
    a.tgt = g.targets;
    a.lu = lu;
    a.lv = lv;
    a.lcount = lcount;
    if (row_hi >= 0) {  // samplers walk only this block's rows
      a.row_base = row_lo;
      a.count_host = row_hi - row_lo;
    }
    return a;
  }

  void init_sets(const UFConfig& c) {
    if (n == 0) return;
    int32_t* H = c.unite == GC_FINISH_HOOKS ? ws.H : nullptr;
    int32_t* L = c.unite == GC_FINISH_REM_LOCK ? ws.L : nullptr;
    (k_init_sets<<<grid_for(n, kEwBlock, 8), kEwBlock, 0, st>>>(P, H, L, n, ws.ctr + C_STAMP0, take_stamps()),
     ::gc::count_launch());
    GC_CHECK_LAUNCH();
  }

  // ---- sampling phase (driver.py:378-403) -------------------------------
  void sample() {
    const UFConfig sc = sampler_cfg(s);
    if (s.sample == GC_SAMPLE_NONE) {
      init_sets(sc);
      return;  // l_max = n sentinel, set on host
    }
    if (s.sample == GC_SAMPLE_KOUT || s.sample == GC_SAMPLE_HB) {
      init_sets(sc);
      // the sampler kernel's span: taken at the entry of the union kernel
      // and of the mode probe that follows it (no stamp nodes)
      if (kev) stamp_defer(5);
      RowUnionArgs ra = rows(sc);
      ra.stamps = ws.ctr + C_STAMP0;
      if (s.sample == GC_SAMPLE_KOUT) {
        run_kout(g, s, sc, ra, fu != nullptr, ws.samp, ws.ctr, st);
      } else {
        run_hb(g, s, sc, ra, fu != nullptr, ws.samp, ws.ctr, st);
      }
      if (kev) stamp_defer(6);
      timed_sample = true;
      run_post_sample(P, n, g.offsets, ws.list, ws.hist, ws.ctr, true, st);
    } else if (s.sample == GC_SAMPLE_BFS) {
      // the BFS label pass writes every label (and forest slot) when it runs
      // (m > 0); the init is still needed for the hook / lock arrays
      if (g.m == 0 || sc.unite == GC_FINISH_HOOKS || sc.unite == GC_FINISH_REM_LOCK) init_sets(sc);
      if (kev) stamp(ws.ctr, 5, st);
      run_bfs(g, s, P, fu, fv, ws.samp, ws.ctr, st);
      if (kev) stamp(ws.ctr, 6, st);
      timed_sample = true;
      run_post_sample(P, n, g.offsets, ws.list, ws.hist, ws.ctr, false, st);
    } else {
      init_sets(sc);
      if (kev) stamp(ws.ctr, 5, st);
      // a labels-only rounds finish takes its working COO from the sampler
      // (the cut edges; GC_LDD_CUT=0 keeps the gather)
      if (!fu && !is_union_finish(s.finish) && ldd_cut_on()) {
        ws.samp.cut_u = ws.rounds.work.u;
        ws.samp.cut_v = ws.rounds.work.v;
        ws.samp.cut_count = ws.ctr + C_CUT;
      }
      const bool exact = run_ldd(g, s, P, ws.samp, ws.ctr, st);
      if (kev) stamp(ws.ctr, 6, st);
      timed_sample = true;
      run_post_sample(P, n, g.offsets, ws.list, ws.hist, ws.ctr, false, st, exact);
    }
  }

  void set_lmax_sentinel() {
    // driver.py:467-468: the sentinel n matches no vertex
    set_ctr(ws.ctr, C_LMAX, static_cast<unsigned long long>(n), st);
  }

  // ---- finish phase (driver.py:473-481) ----------------------------------
  // Returns the number of rounds (round-based finishes) and fills the active
  // list when the sampler left a dominant label.
  int64_t finish() {
    // the active list was gathered by the post-sampling pass (or by
    // run_gather for finish_phase)
    const bool all_active = s.sample == GC_SAMPLE_NONE;
    if (is_union_finish(s.finish)) {
      RowUnionArgs a = rows(finish_cfg(s));
      if (all_active) {
        // every vertex is active: each undirected edge is presented once
        // (t < u, a prefix of the sorted row); the reference inspection
        // count Σdeg is added analytically
        a.list = nullptr;
        a.count_dev = nullptr;
        a.row_base = row_hi >= 0 ? row_lo : 0;
        a.count_host = row_hi >= 0 ? row_hi - row_lo : n;
        a.take_max = INT_MAX;
        a.lower_only = 1;
        a.insp = nullptr;
        if (row_hi < 0) a.all_edges = g.m;
        set_ctr(ws.ctr, C_INSP_FINISH, static_cast<unsigned long long>(g.m), st);
      } else {
        a.list = ws.list;
        a.count_dev = ws.ctr + C_N_ACTIVE;
        a.row_base = 0;
        a.count_host = n;
        a.take_max = INT_MAX;
        a.lower_only = 0;
        a.insp = nullptr;  // counted by the gather
      }
      if (kev) stamp_defer(7);
      a.stamps = ws.ctr + C_STAMP0;  // the pending stamps are taken at the union kernel's entry
      launch_union_rows(finish_cfg(s), fu != nullptr, a, st);
      if (kev) stamp_defer(8);
      return 0;
    }
    if (kev) stamp_defer(7);
    stamp_flush(ws.ctr, st);
    const int64_t r = run_rounds_finish(g, s, P, all_active ? nullptr : ws.list, ws.ctr, fu, fv, ws.rounds, st,
                                        ws.samp.cut_done);
    if (kev) stamp_defer(8);
    return r;
  }
};

double ms(cudaEvent_t a, cudaEvent_t b) {
  float t = 0.f;
  GC_CUDA(cudaEventElapsedTime(&t, a, b));
  return double(t);
}

// Everything a static / forest run needs besides the caller's buffers.
struct RunState {
  EventSet ev;
  unsigned long long* host_ctr = nullptr;  // pinned copy of the device counters
  int64_t rounds = 0;
  bool timed_sample = false;
  RunState() { GC_CUDA(cudaMallocHost(&host_ctr, sizeof(unsigned long long) * C_COUNT_)); }
  ~RunState() { cudaFreeHost(host_ctr); }
};

// GC_FIN_LIST=0: always finalize the whole label array
bool finalize_list_on() {
  static const bool on = [] {
    const char* e = getenv("GC_FIN_LIST");
    return !(e && e[0] == '0');
  }();
  return on;
}

void check_static_args(const gc_csr* g, const gc_spec* spec, int32_t* labels) {
  validate_csr(g);
  require(spec != nullptr, GC_ERR_ARG, "null spec");
  validate_spec(*spec);
  require(g->n == 0 || labels != nullptr, GC_ERR_ARG, "null labels");
  require(reinterpret_cast<uintptr_t>(labels) % 16 == 0, GC_ERR_ARG, "labels must be 16-byte aligned");
}

// Stream-ordered body of a static / forest run.  Host synchronisation only
// happens inside the BFS / LDD samplers and the round finishes; for the
// union-find pipelines the sequence is sync-free and can be graph-captured.
void enqueue_static(const gc_csr* g, const gc_spec* spec, int32_t* labels, int32_t* post, int want_ic,
                    int32_t* fu, int32_t* fv, void* ws, size_t wsb, cudaStream_t st, RunState& rs) {
  const bool forest = fu != nullptr;
  if (forest) require(fv != nullptr, GC_ERR_ARG, "null forest array");
  Pipeline pl(*g, *spec, labels, fu, fv, ws, wsb, st);
  if (forest) {
    if (pl.ws.fpair) {
      fill(reinterpret_cast<int32_t*>(pl.ws.fpair), 2 * g->n, -1, st);  // pairs, split at the end
    } else if (!(spec->sample == GC_SAMPLE_BFS && g->m > 0)) {
      // a BFS sample over edges writes every slot itself (k_bfs_label)
      fill(fu, g->n, -1, st);
      fill(fv, g->n, -1, st);
    }
  }
  L2Residency keep_parents(st, labels, size_t(g->n) * 4);
  cudaEvent_t* ev = rs.ev.e;
  pl.kev = ev + 5;
  const int32_t n = pl.n;

  // union-find samplers start with the set init, which takes stamp 0 at its
  // entry; the traversal samplers stamp with a node
  if (spec->sample == GC_SAMPLE_NONE || spec->sample == GC_SAMPLE_KOUT || spec->sample == GC_SAMPLE_HB)
    stamp_defer(0);
  else
    stamp(pl.ws.ctr, 0, st);
  pl.sample();
  stamp_defer(1);  // shares a node with the finish-phase stamps when nothing runs between
  if (spec->sample == GC_SAMPLE_NONE) pl.set_lmax_sentinel();
  if (post && n) {
    stamp_flush(pl.ws.ctr, st);
    GC_CUDA(cudaMemcpyAsync(post, labels, size_t(n) * 4, cudaMemcpyDeviceToDevice, st));
  }
  if (want_ic && n && spec->sample != GC_SAMPLE_NONE) {
    stamp_flush(pl.ws.ctr, st);
    // every label-crossing edge has an endpoint outside L_max, so the census
    // only walks the active rows (Σ deg = the finish inspections), adding
    // back the reverse entries from L_max rows
    (k_ic_census<<<grid_for(n, kEwBlock, 8), kEwBlock, 0, st>>>(labels, n, g->offsets, g->targets,
                                                               pl.ws.list, pl.ws.ctr), ::gc::count_launch());
    GC_CHECK_LAUNCH();
  }
  stamp_defer(2);
  rs.rounds = pl.finish();
  stamp_defer(3);
  // finalize takes the pending stamps at its entry
  if (forest || n == 0) stamp_flush(pl.ws.ctr, st);
  if (!forest) {
    // after a sampler and a union-find finish only the active list can
    // have moved (k_finalize_list; the whole-array pass stays as the
    // fallback when the finish linked L_max itself)
    const bool uf_finish = spec->finish >= GC_FINISH_ASYNC && spec->finish <= GC_FINISH_REM_CAS;
    const bool list_ok = uf_finish && spec->sample != GC_SAMPLE_NONE && finalize_list_on();
    run_finalize(labels, n, pl.ws.hist, pl.ws.ctr, st, spec->finish == GC_FINISH_JTB,
                 list_ok ? pl.ws.list : nullptr);
  }
  if (forest && n) {
    // spanning_forest: component_count = n - |forest| (driver.py:535); the
    // pair form is split into fu / fv and counted in the same pass
    set_ctr(pl.ws.ctr, C_SCRATCH1, 0, st);
    if (pl.ws.fpair)
      (k_split_pairs<<<grid_for(n, kEwBlock, 8), kEwBlock, 0, st>>>(pl.ws.fpair, n, fu, fv,
                                                                   pl.ws.ctr + C_SCRATCH1), ::gc::count_launch());
    else
      (k_count_ne<<<grid_for(n, kEwBlock, 8), kEwBlock, 0, st>>>(fu, n, -1, pl.ws.ctr + C_SCRATCH1),
       ::gc::count_launch());
    GC_CHECK_LAUNCH();
  }
  stamp_defer(4);
  stamp_flush(pl.ws.ctr, st);
  GC_CUDA(cudaMemcpyAsync(rs.host_ctr, pl.ws.ctr, sizeof(unsigned long long) * C_COUNT_,
                          cudaMemcpyDeviceToHost, st));
  rs.timed_sample = pl.timed_sample;
}

// After the stream has drained: turn the counters and events into stats.
void collect_static(const gc_csr* g, const gc_spec* spec, bool forest, int want_ic, RunState& rs,
                    gc_stats* stats) {
  const unsigned long long* c = rs.host_ctr;
  const int64_t n = g->n;
  require(c[C_CYCLE] == 0, GC_ERR_MALFORMED, "label array contains a cycle");
  if (!stats) return;
  const auto span = [&](int a, int b) { return double(c[C_STAMP0 + b] - c[C_STAMP0 + a]) * 1e-6; };  // ns -> ms
  stats->t_sample_ms = span(0, 1);
  stats->t_finish_ms = span(2, 3);
  stats->t_finalize_ms = forest ? 0.0 : span(3, 4);
  stats->t_sample_kernel_ms = rs.timed_sample ? span(5, 6) : 0.0;
  stats->t_finish_kernel_ms = span(7, 8);
  stats->insp_sample = int64_t(c[C_INSP_SAMPLE]);
  stats->insp_finish = int64_t(c[C_INSP_FINISH]);
  stats->rounds = rs.rounds;
  stats->components = forest ? n - int64_t(c[C_SCRATCH1]) : int64_t(c[C_COMPONENTS]);
  if (spec->sample == GC_SAMPLE_NONE) {
    stats->l_max = n;
    stats->lmax_count = n ? 1 : 0;  // identity labels: every count is 1
    stats->n_active = n;
    stats->ic_count = g->m;  // every directed edge crosses identity labels
  } else {
    stats->l_max = int64_t(c[C_LMAX]);
    stats->lmax_count = int64_t(c[C_LMAX_COUNT]);
    stats->n_active = int64_t(c[C_N_ACTIVE]);
    stats->ic_count = want_ic ? int64_t(c[C_IC]) : -1;
  }
}

void run_static(const gc_csr* g, const gc_spec* spec, int32_t* labels, int32_t* post, int want_ic,
                int32_t* fu, int32_t* fv, gc_stats* stats, void* ws, size_t wsb, void* stream) {
  check_static_args(g, spec, labels);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static thread_local RunState rs;
  enqueue_static(g, spec, labels, post, want_ic, fu, fv, ws, wsb, st, rs);
  GC_CUDA(cudaStreamSynchronize(st));
  collect_static(g, spec, fu != nullptr, want_ic, rs, stats);
}

// Pipelines with no host round trip (union-find finish, none / k-out / HB
// sampling) can be captured once and replayed as one CUDA graph launch.
bool graph_capturable(const gc_spec& s) {
  return is_union_finish(s.finish) &&
         (s.sample == GC_SAMPLE_NONE || s.sample == GC_SAMPLE_KOUT || s.sample == GC_SAMPLE_HB);
}

}  // namespace

namespace {
thread_local std::string g_err;
}

void set_last_error(const char* msg) { g_err = msg; }

}  // namespace gc

using namespace gc;

extern "C" {

const char* gc_last_error(void) { return g_err.c_str(); }

const char* gc_version(void) { return "gconn-b200 0.1.0 (sm_100a, built " __DATE__ " " __TIME__ ")"; }

size_t gc_workspace_size(int64_t n, int64_t m, const gc_spec* spec) {
  if (!spec || n < 0 || m < 0) return 0;
  Sizer sz;
  Layout<Sizer> l;
  l.carve(sz, n, m, *spec, true);
  return sz.used + 4096;
}

struct gc_plan {
  gc_csr g;
  gc_spec s;
  int32_t* labels;
  void* ws;
  size_t wsb;
  cudaStream_t st;
  gc::RunState rs;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap = nullptr;  // private stream for capture (the caller's may be the legacy stream)
  bool capturable = false;
  long long kernels = 0;  // kernels per replay (for gc_launch_count)
};

int gc_plan_create(const gc_csr* g, const gc_spec* spec, int32_t* labels_out, void* ws,
                   size_t ws_bytes, void* stream, gc_plan** out) {
  return guarded([&] {
    require(out != nullptr, GC_ERR_ARG, "null plan out");
    check_static_args(g, spec, labels_out);
    require(ws_bytes >= gc_workspace_size(g->n, g->m, spec), GC_ERR_OOM, "workspace too small");
    gc_plan* p = new gc_plan();
    p->g = *g;
    p->s = *spec;
    p->labels = labels_out;
    p->ws = ws;
    p->wsb = ws_bytes;
    p->st = static_cast<cudaStream_t>(stream);
    p->capturable = graph_capturable(*spec) && getenv("GC_NO_GRAPH") == nullptr;
    num_sms();        // resolve device attributes before any capture
    pinned_words();
    *out = p;
  });
}

int gc_plan_run(gc_plan* p, gc_stats* stats) {
  return guarded([&] {
    require(p != nullptr, GC_ERR_ARG, "null plan");
    if (p->capturable && p->exec == nullptr) {
      cudaGraph_t graph = nullptr;
      if (!p->cap) GC_CUDA(cudaStreamCreateWithFlags(&p->cap, cudaStreamNonBlocking));
      GC_CUDA(cudaStreamBeginCapture(p->cap, cudaStreamCaptureModeThreadLocal));
      const long long l0 = launch_total();
      t_capturing = true;
      try {
        enqueue_static(&p->g, &p->s, p->labels, nullptr, 0, nullptr, nullptr, p->ws, p->wsb, p->cap, p->rs);
      } catch (...) {
        t_capturing = false;
        cudaStreamEndCapture(p->cap, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      t_capturing = false;
      GC_CUDA(cudaStreamEndCapture(p->cap, &graph));
      p->kernels = launch_total() - l0;
      add_launches(-p->kernels);  // captured, not yet executed
      const cudaError_t e = cudaGraphInstantiate(&p->exec, graph, 0);
      cudaGraphDestroy(graph);
      GC_CUDA(e);
    }
    if (p->exec) {
      GC_CUDA(cudaGraphLaunch(p->exec, p->st));
      add_launches(p->kernels);
    } else {
      enqueue_static(&p->g, &p->s, p->labels, nullptr, 0, nullptr, nullptr, p->ws, p->wsb, p->st, p->rs);
    }
    GC_CUDA(cudaStreamSynchronize(p->st));
    collect_static(&p->g, &p->s, false, 0, p->rs, stats);
  });
}

void gc_plan_destroy(gc_plan* p) {
  if (!p) return;
  if (p->exec) cudaGraphExecDestroy(p->exec);
  if (p->cap) cudaStreamDestroy(p->cap);
  delete p;
}

int gc_static_cc(const gc_csr* g, const gc_spec* spec, int32_t* labels_out, int32_t* post_sample_out,
                 int want_ic, gc_stats* stats, void* ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    run_static(g, spec, labels_out, post_sample_out, want_ic, nullptr, nullptr, stats, ws, ws_bytes,
               stream);
  });
}

int gc_spanning_forest(const gc_csr* g, const gc_spec* spec, int32_t* fu, int32_t* fv,
                       int32_t* parent_out, gc_stats* stats, void* ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    require(spec != nullptr, GC_ERR_ARG, "null spec");
    require(fu != nullptr && fv != nullptr, GC_ERR_ARG, "null forest arrays");
    const bool root_based =
        is_union_finish(spec->finish) ? spec->splice != GC_SPLICE_ATOMIC
        : spec->finish == GC_FINISH_SV ? true
        : spec->finish == GC_FINISH_LT ? spec->lt_update == GC_LT_UPDATE_ROOTS
                                       : false;
    require(root_based, GC_ERR_CONFIG, "spanning forest needs a root-based finish");
    // the parent buffer is the caller's, or lives in the workspace head
    const int64_t n = g ? g->n : 0;
    Arena a(ws, ws_bytes);
    int32_t* labels = parent_out ? parent_out : a.take<int32_t>(n);
    run_static(g, spec, labels, nullptr, 0, fu, fv, stats, static_cast<char*>(ws) + a.used,
               ws_bytes - a.used, stream);
  });
}

int gc_finish_phase(const gc_csr* g, const gc_spec* spec, int32_t* labels_io, int64_t l_max,
                    gc_stats* stats, void* ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    validate_csr(g);
    require(spec != nullptr, GC_ERR_ARG, "null spec");
    validate_spec(*spec);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the finish kernels use labels as parent indices (driver.py:440 copies
    // them into ds.p): an id outside [0, n) is malformed input, not a fault
    check_ids(labels_io, g->n, g->n, st, "finish_phase label");
    gc_spec s2 = *spec;
    s2.sample = GC_SAMPLE_KOUT;  // force the gather path (labels are given)
    Pipeline pl(*g, s2, labels_io, nullptr, nullptr, ws, ws_bytes, st);
    const int32_t n = pl.n;
    set_ctr(pl.ws.ctr, C_LMAX, static_cast<unsigned long long>(l_max), st);
    if (is_union_finish(spec->finish)) {
      UFConfig c = finish_cfg(*spec);
      if (n && (c.unite == GC_FINISH_HOOKS || c.unite == GC_FINISH_REM_LOCK)) {
        int32_t* buf = c.unite == GC_FINISH_HOOKS ? pl.ws.H : pl.ws.L;
        fill(buf, n, c.unite == GC_FINISH_HOOKS ? n : 0, st);
      }
    }
    static thread_local EventSet ev;
    GC_CUDA(rec(ev.e[0], st));
    run_gather(labels_io, n, g->offsets, pl.ws.list, pl.ws.ctr, st);
    const int64_t rounds = pl.finish();
    GC_CUDA(rec(ev.e[1], st));
    unsigned long long c[C_COUNT_];
    GC_CUDA(cudaMemcpyAsync(c, pl.ws.ctr, sizeof(c), cudaMemcpyDeviceToHost, st));
    GC_CUDA(cudaStreamSynchronize(st));
    if (stats) {
      std::memset(stats, 0, sizeof(*stats));
      stats->t_finish_ms = ms(ev.e[0], ev.e[1]);
      stats->insp_finish = int64_t(c[C_INSP_FINISH]);
      stats->rounds = rounds;
      stats->n_active = int64_t(c[C_N_ACTIVE]);
      stats->l_max = l_max;
    }
  });
}

int gc_label_finalization(int32_t* labels, int64_t n, void* ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    require(n >= 0 && n < (int64_t(1) << 31), GC_ERR_MALFORMED, "bad length");
    if (n == 0) return;
    require(reinterpret_cast<uintptr_t>(labels) % 16 == 0, GC_ERR_ARG, "labels must be 16-byte aligned");
    Arena a(ws, ws_bytes);
    unsigned long long* ctr = a.take<unsigned long long>(C_COUNT_);
    int32_t* mins = a.take<int32_t>(n);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    GC_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * C_COUNT_, st));
    run_finalize(labels, int32_t(n), mins, ctr, st);
    unsigned long long cyc = 0;
    GC_CUDA(cudaMemcpyAsync(&cyc, ctr + C_CYCLE, 8, cudaMemcpyDeviceToHost, st));
    GC_CUDA(cudaStreamSynchronize(st));
    require(cyc == 0, GC_ERR_MALFORMED, "label array contains a cycle");
  });
}

// ---- sharded two-phase building blocks ------------------------
namespace {

// finish = true: the labels come from any sharded sampler, including the
// distributed BFS (gc_dbfs_*), which has no gc_shard_sample form
void check_shard_spec(const gc_spec* spec, bool finish = false) {
  require(is_union_finish(spec->finish), GC_ERR_CONFIG, "sharded pipeline needs a union-find finish");
  require(spec->sample == GC_SAMPLE_NONE || spec->sample == GC_SAMPLE_KOUT || spec->sample == GC_SAMPLE_HB ||
              (finish && spec->sample == GC_SAMPLE_BFS),
          GC_ERR_CONFIG, finish ? "sharded sampling supports none / k-out / hb / bfs"
                                : "sharded sampling supports none / k-out / hb (bfs: gc_dbfs_*)");
  require(spec->sample != GC_SAMPLE_KOUT || spec->kout_mode == GC_KOUT_FIRST_K, GC_ERR_CONFIG,
          "sharded k-out needs FIRST_K (random offsets are drawn over the whole graph)");
}

void read_ctr(unsigned long long* dst, const unsigned long long* ctr, cudaStream_t st) {
  GC_CUDA(cudaMemcpyAsync(dst, ctr, sizeof(unsigned long long) * C_COUNT_, cudaMemcpyDeviceToHost, st));
  GC_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

int gc_shard_sample(const gc_csr* g, const gc_spec* spec, int64_t row_lo, int64_t row_hi, int32_t* parent,
                    int32_t* out_u, int32_t* out_v, unsigned long long* out_count, gc_stats* stats, void* ws,
                    size_t ws_bytes, void* stream) {
  return guarded([&] {
    check_static_args(g, spec, parent);
    check_shard_spec(spec);
    // NULL outputs: sample only (the compact summary exchange needs no list)
    const bool record = out_u != nullptr;
    require(!record || (out_v && out_count), GC_ERR_ARG, "null merging-edge output");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (record) GC_CUDA(cudaMemsetAsync(out_count, 0, sizeof(unsigned long long), st));
    require(row_lo >= 0 && row_lo <= row_hi && row_hi <= g->n, GC_ERR_ARG, "row block outside [0, n]");
    Pipeline pl(*g, *spec, parent, nullptr, nullptr, ws, ws_bytes, st);
    pl.row_lo = row_lo;
    pl.row_hi = row_hi;
    const bool edges = spec->splice != GC_SPLICE_ATOMIC;  // root-based: record real merging edges
    if (record && edges) {
      pl.lu = out_u;
      pl.lv = out_v;
      pl.lcount = out_count;
    }
    const UFConfig sc = sampler_cfg(*spec);
    pl.init_sets(sc);
    if (spec->sample == GC_SAMPLE_KOUT) run_kout(*g, *spec, sc, pl.rows(sc), false, pl.ws.samp, pl.ws.ctr, st);
    if (spec->sample == GC_SAMPLE_HB) run_hb(*g, *spec, sc, pl.rows(sc), false, pl.ws.samp, pl.ws.ctr, st);
    if (record && !edges && pl.n) {
      (k_root_transitions<<<grid_for((int64_t(pl.n) + 3) / 4, kEwBlock, 8), kEwBlock, 0, st>>>(
           parent, nullptr, pl.n, out_u, out_v, out_count), count_launch());
      GC_CHECK_LAUNCH();
    }
    unsigned long long c[C_COUNT_];
    read_ctr(c, pl.ws.ctr, st);
    if (stats) {
      std::memset(stats, 0, sizeof(*stats));
      stats->insp_sample = int64_t(c[C_INSP_SAMPLE]);
    }
  });
}

int gc_shard_finish(const gc_csr* g, const gc_spec* spec, int64_t row_lo, int64_t row_hi, int32_t* parent,
                    int32_t* out_u, int32_t* out_v, unsigned long long* out_count, gc_stats* stats, void* ws,
                    size_t ws_bytes, void* stream) {
  return guarded([&] {
    check_static_args(g, spec, parent);
    check_shard_spec(spec, true);
    require(out_u && out_v && out_count, GC_ERR_ARG, "null merging-edge output");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    GC_CUDA(cudaMemsetAsync(out_count, 0, sizeof(unsigned long long), st));
    require(row_lo >= 0 && row_lo <= row_hi && row_hi <= g->n, GC_ERR_ARG, "row block outside [0, n]");
    Pipeline pl(*g, *spec, parent, nullptr, nullptr, ws, ws_bytes, st);
    pl.row_lo = row_lo;
    pl.row_hi = row_hi;
    const bool edges = spec->splice != GC_SPLICE_ATOMIC;
    if (edges) {
      pl.lu = out_u;
      pl.lv = out_v;
      pl.lcount = out_count;
    }
    const UFConfig fc = finish_cfg(*spec);
    if (pl.n && (fc.unite == GC_FINISH_HOOKS || fc.unite == GC_FINISH_REM_LOCK))
      fill(fc.unite == GC_FINISH_HOOKS ? pl.ws.H : pl.ws.L, pl.n, fc.unite == GC_FINISH_HOOKS ? pl.n : 0, st);
    if (spec->sample == GC_SAMPLE_NONE) {
      pl.set_lmax_sentinel();
    } else {
      // the merged sampled partition is identical on every rank, so the
      // compressed labels, L_max and the active set are too
      run_post_sample(parent, pl.n, g->offsets, pl.ws.list, pl.ws.hist, pl.ws.ctr, true, st);
    }
    // non-root-based rules: snapshot which vertices are roots (a bitmap in
    // the histogram buffer, free after the mode) and emit root transitions
    // after the finish
    uint32_t* roots = reinterpret_cast<uint32_t*>(pl.ws.hist);
    const int gq = grid_for((int64_t(pl.n) + 3) / 4, kEwBlock, 8);
    // after a sampler only active roots and L_max can be hooked: snapshot
    // and compare over the active list (one flag per entry in the same
    // buffer) instead of the whole parent array
    const bool by_list = spec->sample != GC_SAMPLE_NONE;
    uint8_t* flags = reinterpret_cast<uint8_t*>(pl.ws.hist);
    if (!edges && pl.n) {
      if (by_list)
        (k_root_flags_list<<<grid_for(pl.n, kEwBlock, 2), kEwBlock, 0, st>>>(parent, pl.ws.list, pl.ws.ctr, flags),
         count_launch());
      else
        (k_root_bitmap<<<gq, kEwBlock, 0, st>>>(parent, pl.n, roots), count_launch());
    }
    pl.finish();
    if (!edges && pl.n) {
      if (by_list)
        (k_root_transitions_list<<<grid_for(pl.n, kEwBlock, 2), kEwBlock, 0, st>>>(
             parent, pl.ws.list, pl.ws.ctr, flags, out_u, out_v, out_count), count_launch());
      else
        (k_root_transitions<<<gq, kEwBlock, 0, st>>>(parent, roots, pl.n, out_u, out_v, out_count), count_launch());
      GC_CHECK_LAUNCH();
    }
    unsigned long long c[C_COUNT_];
    read_ctr(c, pl.ws.ctr, st);
    if (stats) {
      std::memset(stats, 0, sizeof(*stats));
      stats->insp_finish = int64_t(c[C_INSP_FINISH]);
      const bool none = spec->sample == GC_SAMPLE_NONE;
      stats->l_max = none ? g->n : int64_t(c[C_LMAX]);
      stats->lmax_count = none ? (g->n ? 1 : 0) : int64_t(c[C_LMAX_COUNT]);
      stats->n_active = none ? g->n : int64_t(c[C_N_ACTIVE]);
    }
  });
}

int gc_union_edges(int32_t* parent, int64_t n, const int32_t* us, const int32_t* vs, int64_t k,
                   const gc_spec* spec, int32_t* aux, int32_t* fu, int32_t* fv, void* stream) {
  return guarded([&] {
    require(spec != nullptr, GC_ERR_ARG, "null spec");
    require(is_union_finish(spec->finish), GC_ERR_CONFIG, "union_edges needs a union-find rule");
    UFConfig c = finish_cfg(*spec);
    require(valid_uf(c), GC_ERR_CONFIG, "unsupported union-find combination");
    require(c.unite != GC_FINISH_JTB || spec->jtb_ranks, GC_ERR_ARG, "JTB needs ranks");
    require((c.unite != GC_FINISH_HOOKS && c.unite != GC_FINISH_REM_LOCK) || aux, GC_ERR_ARG,
            "hooks / rem_lock need aux scratch");
    require(n >= 0 && n < (int64_t(1) << 31) && k >= 0, GC_ERR_ARG, "bad size");
    // endpoints index the parent array: reject out-of-range pairs up front
    check_ids(us, k, n, static_cast<cudaStream_t>(stream), "union endpoint");
    check_ids(vs, k, n, static_cast<cudaStream_t>(stream), "union endpoint");
    CooUnionArgs a{};
    a.P = parent;
    a.H = c.unite == GC_FINISH_HOOKS ? aux : nullptr;
    a.L = c.unite == GC_FINISH_REM_LOCK ? aux : nullptr;
    a.R = spec->jtb_ranks;
    a.fu = fu;
    a.fv = fv;
    a.n = int32_t(n);
    a.us = us;
    a.vs = vs;
    a.k = k;
    a.skip = nullptr;
    launch_union_coo(c, fu != nullptr, a, static_cast<cudaStream_t>(stream));
  });
}

int gc_union_edges_list(int32_t* parent, int64_t n, const int32_t* us, const int32_t* vs, int64_t k,
                        const gc_spec* spec, int32_t* aux, int32_t* out_u, int32_t* out_v,
                        unsigned long long* out_count, void* stream) {
  return guarded([&] {
    require(spec != nullptr && out_u && out_v && out_count, GC_ERR_ARG, "null argument");
    require(is_union_finish(spec->finish), GC_ERR_CONFIG, "union_edges needs a union-find rule");
    UFConfig c = finish_cfg(*spec);
    require(valid_uf(c), GC_ERR_CONFIG, "unsupported union-find combination");
    require(c.splice != GC_SPLICE_ATOMIC, GC_ERR_CONFIG,
            "atomic splice is not root-based: merging edges cannot be recorded");
    require(c.unite != GC_FINISH_JTB || spec->jtb_ranks, GC_ERR_ARG, "JTB needs ranks");
    require((c.unite != GC_FINISH_HOOKS && c.unite != GC_FINISH_REM_LOCK) || aux, GC_ERR_ARG,
            "hooks / rem_lock need aux scratch");
    require(n >= 0 && n < (int64_t(1) << 31) && k >= 0, GC_ERR_ARG, "bad size");
    check_ids(us, k, n, static_cast<cudaStream_t>(stream), "union endpoint");
    check_ids(vs, k, n, static_cast<cudaStream_t>(stream), "union endpoint");
    CooUnionArgs a{};
    a.P = parent;
    a.H = c.unite == GC_FINISH_HOOKS ? aux : nullptr;
    a.L = c.unite == GC_FINISH_REM_LOCK ? aux : nullptr;
    a.R = spec->jtb_ranks;
    a.n = int32_t(n);
    a.us = us;
    a.vs = vs;
    a.k = k;
    a.skip = nullptr;
    a.lu = out_u;
    a.lv = out_v;
    a.lcount = out_count;
    launch_union_coo(c, false, a, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
