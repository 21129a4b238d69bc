/*
 * gconn.h — C ABI of libgconn.so, the sm_100a implementation of the GConn
 * connectivity design space (arXiv 2008.11839).
 *
 * The reference (`connlab`, /root/reference/pkg/src/connlab) is a pure
 * Python package with no FFI; its drop-in surface is the Python driver API
 * (driver.py:99-725).  This header is the seam *under* that surface: the
 * Python package `paper_2008_11839_b200` mirrors the connlab names and binds
 * these entry points with ctypes (see INTEGRATION.md for the binding a
 * connlab maintainer would add).  Every entry point below names the
 * reference function it replaces.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers unless the parameter name ends
 *     in `_host`.  Vertex ids are int32 (graphs.py:11, VERTEX_LIMIT = 2^31),
 *     CSR offsets are int64 (graphs.py:47-51).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *     Calls are asynchronous with respect to the host unless documented
 *     otherwise; stats are written when the call returns (entry points that
 *     produce stats synchronize the stream once at the end).
 *   - Scratch memory is caller-owned: query gc_workspace_size() and pass a
 *     device buffer of at least that many bytes (the Python layer allocates
 *     it from the PyTorch caching allocator).
 *   - Return value: GC_OK or a GC_ERR_* status.  No C++ exception ever
 *     crosses the ABI; gc_last_error() returns a thread-local message.
 *     The Python layer maps GC_ERR_CONFIG -> connlab ConfigError and
 *     GC_ERR_MALFORMED -> MalformedInputError (errors.py:4-13).
 */
#ifndef GCONN_H_
#define GCONN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes -------------------------------------------------------*/
enum {
  GC_OK = 0,
  GC_ERR_CONFIG = 2,     /* invalid spec / combination (ConfigError)        */
  GC_ERR_MALFORMED = 3,  /* bad graph / endpoint out of range               */
  GC_ERR_CUDA = 4,       /* a CUDA runtime error                             */
  GC_ERR_OOM = 5,        /* workspace too small / allocation failed          */
  GC_ERR_ARG = 6         /* null pointer or negative size                    */
};

/* ---- spec enums (driver.py:65-82, dset.py:29-50, minbased.py:24-37) ------*/
enum gc_sample_kind { GC_SAMPLE_NONE = 0, GC_SAMPLE_KOUT = 1, GC_SAMPLE_HB = 2,
                      GC_SAMPLE_BFS = 3, GC_SAMPLE_LDD = 4 };
enum gc_finish_kind { GC_FINISH_ASYNC = 0, GC_FINISH_HOOKS = 1,
                      GC_FINISH_EARLY = 2, GC_FINISH_REM_LOCK = 3,
                      GC_FINISH_REM_CAS = 4, GC_FINISH_JTB = 5,
                      GC_FINISH_SV = 6, GC_FINISH_LT = 7,
                      GC_FINISH_STERGIOU = 8, GC_FINISH_LP = 9 };
enum gc_find_kind { GC_FIND_NAIVE = 0, GC_FIND_SPLIT = 1, GC_FIND_HALVE = 2,
                    GC_FIND_COMPRESS = 3, GC_FIND_TWO_TRY = 4 };
enum gc_splice_kind { GC_SPLICE_NONE = 0, GC_SPLICE_SPLIT_ONE = 1,
                      GC_SPLICE_HALVE_ONE = 2, GC_SPLICE_ATOMIC = 3 };
enum gc_lt_connect { GC_LT_CONNECT = 0, GC_LT_PARENT = 1, GC_LT_EXTENDED = 2 };
enum gc_lt_update { GC_LT_UPDATE_ALL = 0, GC_LT_UPDATE_ROOTS = 1 };
enum gc_lt_shortcut { GC_LT_SHORTCUT_ONE = 0, GC_LT_SHORTCUT_FULL = 1 };
enum gc_kout_mode { GC_KOUT_FIRST_K = 0, GC_KOUT_FIRST_PLUS_RANDOM = 1 };

/* A symmetrized CSR graph in device memory (graphs.py:43-87 `Graph`):
 * offsets[n+1] int64, targets[m] int32, rows sorted ascending, no
 * self-loops, no duplicates; m counts directed entries. */
typedef struct gc_csr {
  int64_t n;
  int64_t m;
  const int64_t* offsets;
  const int32_t* targets;
} gc_csr;

/* AlgorithmSpec (driver.py:99-110) flattened.  Host-side RNG-derived inputs
 * (BFS source, JTB ranks, k-out random offsets) are computed by the Python
 * layer with the reference's own generators and passed in, so runs are
 * reproducible against the oracle. */
typedef struct gc_spec {
  int32_t sample;        /* gc_sample_kind                                   */
  int32_t finish;        /* gc_finish_kind                                   */
  int32_t find;          /* gc_find_kind   (union-find finishes)             */
  int32_t splice;        /* gc_splice_kind (Rem finishes)                    */
  int32_t lt_connect;    /* gc_lt_connect  (LT finish)                       */
  int32_t lt_update;     /* gc_lt_update                                     */
  int32_t lt_shortcut;   /* gc_lt_shortcut                                   */
  int32_t lt_alter;      /* 0/1                                              */
  int32_t kout_k;        /* sampling.py:19 default 2                         */
  int32_t kout_mode;     /* gc_kout_mode                                     */
  int32_t hb_edges;      /* sampling.py:20 default 4                         */
  int32_t reserved0;
  int64_t bfs_source;    /* BFS sampler source vertex (sampling.py:130-132)  */
  uint64_t seed;         /* spec seed (driver.py:109)                        */
  double ldd_beta;       /* LDD sampler: exponential shift rate              */
  const uint32_t* jtb_ranks;          /* device, n entries, or NULL (dset.py:372-374) */
  const int32_t* kout_rand_offsets;   /* device, (#deg>0 vertices) x (k-1) row offsets */
  /* BFS sampler source chosen on the device (sampling.py:130-132): used when
   * bfs_source < 0 — host array of the sorted, distinct probe vertices; the
   * source is the first probe of maximum degree (np.argmax order) */
  const int32_t* bfs_probes;
  int32_t bfs_nprobes;
  int32_t reserved1;
} gc_spec;

/* RunStats (validate.py:20-43) as produced on device.  Times are CUDA-event
 * milliseconds per phase; inspection counts are computed analytically on
 * device with the reference's definitions. */
typedef struct gc_stats {
  double t_sample_ms;
  double t_finish_ms;
  double t_finalize_ms;
  int64_t insp_sample;
  int64_t insp_finish;
  int64_t rounds;
  int64_t components;
  int64_t l_max;          /* most frequent post-sample label (n for NONE)    */
  int64_t lmax_count;     /* its multiplicity (cov = lmax_count / n)         */
  int64_t n_active;       /* vertices the finish phase saw                   */
  int64_t ic_count;       /* directed edges with differing post-sample labels */
  double t_sample_kernel_ms; /* the sampler's union / traversal kernel alone */
  double t_finish_kernel_ms; /* the finish union kernel (or all rounds) alone */
} gc_stats;

/* ---- library ------------------------------------------------------------*/
const char* gc_last_error(void);
const char* gc_version(void);
/* Cumulative number of CUDA kernels libgconn has launched in this process
 * (bench.py reports the delta over its timed region as gpu_launches). */
long long gc_launch_count(void);
/* Scratch bytes needed by gc_static_cc / gc_spanning_forest / gc_finish_phase. */
size_t gc_workspace_size(int64_t n, int64_t m, const gc_spec* spec);

/* ---- static connectivity (driver.py:454-507 `_pipeline`,
 *      `static_connectivity`) -------------------------------------------------
 * labels_out[n] receives the finalized labels: each component's minimum
 * vertex id (driver.py:420-429 + validate.py:251-259).  If
 * `post_sample_out` is non-NULL it receives a copy of the post-sampling
 * labels (the `post_sample` array of driver.py:466) for the cov/ic census;
 * `want_ic` != 0 additionally counts label-crossing edges outside the timed
 * phases (driver.py:406-417). */
int gc_static_cc(const gc_csr* g, const gc_spec* spec, int32_t* labels_out,
                 int32_t* post_sample_out, int want_ic, gc_stats* stats,
                 void* ws, size_t ws_bytes, void* stream);

/* ---- reusable static plan -----------------------------------------------
 * Binds a graph, spec, output and workspace once; gc_plan_run repeats the
 * static pipeline.  Pipelines without host round trips (union-find finish
 * with none / k-out / HB sampling) are captured into a CUDA graph on the
 * first run and replayed as one launch afterwards. */
typedef struct gc_plan gc_plan;
int gc_plan_create(const gc_csr* g, const gc_spec* spec, int32_t* labels_out,
                   void* ws, size_t ws_bytes, void* stream, gc_plan** out);
int gc_plan_run(gc_plan* plan, gc_stats* stats);
void gc_plan_destroy(gc_plan* plan);

/* ---- spanning forest (driver.py:510-536) --------------------------------
 * Slot r of (fu, fv) holds the original edge recorded when r lost root
 * status; empty slots hold -1 (ForestEdges.edges None). */
int gc_spanning_forest(const gc_csr* g, const gc_spec* spec, int32_t* fu,
                       int32_t* fv, int32_t* parent_out, gc_stats* stats,
                       void* ws, size_t ws_bytes, void* stream);
/* parent_out (nullable) receives the unfinalised parent array — a valid
 * union-find state (P[v] <= v, roots are class minima) that the sharded
 * driver keeps merging into. */

/* ---- finish phase only (driver.py:432-446) -------------------------------
 * labels_io[n] holds the (possibly partial) input labels and receives the
 * unfinalized finish output. */
int gc_finish_phase(const gc_csr* g, const gc_spec* spec, int32_t* labels_io,
                    int64_t l_max, gc_stats* stats, void* ws, size_t ws_bytes,
                    void* stream);

/* ---- label finalization (driver.py:420-429) ------------------------------
 * In place: chase to the root, then relabel each class by its minimum
 * member (validate.py:251-259).  ws needs 4*n bytes. */
int gc_label_finalization(int32_t* labels, int64_t n, void* ws,
                          size_t ws_bytes, void* stream);

/* ---- batch union seam (dset.py:402-416 `union_edge_list`) ----------------
 * Applies the spec's union rule to k edge pairs over parent[n] (in place).
 * aux: 4*n bytes of zeroed scratch for HOOKS / REM_LOCK (else may be NULL).
 * Endpoints outside [0, n) -> GC_ERR_MALFORMED before any union runs (a
 * synchronous range check on the stream). */
int gc_union_edges(int32_t* parent, int64_t n, const int32_t* us,
                   const int32_t* vs, int64_t k, const gc_spec* spec,
                   int32_t* aux, int32_t* fu, int32_t* fv, void* stream);

/* Like gc_union_edges, but appends every edge whose union merged two trees
 * to (out_u, out_v) (capacity k) and counts them in *out_count (device).
 * Root-based rules only.  This is the exchange unit of the sharded drivers
 * (SURVEY 8e): the merging edges of a shard form a spanning forest of it. */
int gc_union_edges_list(int32_t* parent, int64_t n, const int32_t* us,
                        const int32_t* vs, int64_t k, const gc_spec* spec,
                        int32_t* aux, int32_t* out_u, int32_t* out_v,
                        unsigned long long* out_count, void* stream);

/* ---- sharded two-phase pipeline (multi-GPU building blocks) ----
 * The reference is single-process; these split `_pipeline`
 * (driver.py:454-500) at its two exchange points so a driver can run it over
 * edge-sharded CSR blocks (rows outside the block empty):
 *   [row_lo, row_hi) is the block's row range (rows outside it are empty in
 *   the block's CSR; the samplers and the unsampled finish walk only it).
 *   gc_shard_sample: parent := identity, then the sampler (none / k-out
 *     FIRST_K / HB) over the block's rows.  Every union that merged two trees
 *     appends its (u, v) to out_u/out_v (capacity n) and bumps *out_count
 *     (device).  stats->insp_sample = this block's sample inspections.
 *   -- exchange: all-gather the merging edges, union the foreign ones --
 *   gc_shard_finish (also after the distributed BFS sampler, gc_dbfs_*):
 *     compress, most-frequent label, active gather (identical
 *     on every rank once the sampled partitions are merged), then the
 *     union-find finish over the block's active rows, recording merging edges
 *     the same way.  stats: insp_finish (block), l_max, lmax_count, n_active.
 *   -- exchange again, union foreign edges, gc_label_finalization --
 * Union-find finishes only.  Root-based rules record the merging edges
 * themselves; the atomic splice (not root-based: it re-points non-roots)
 * records root transitions instead — every vertex that was a root before the
 * phase and is not one after emits (v, P[v]), one pair per merge, which
 * reproduces the partition change when unioned anywhere.  NULL outputs in
 * gc_shard_sample: sample only (the compact summary exchange). */
int gc_shard_sample(const gc_csr* g, const gc_spec* spec, int64_t row_lo,
                    int64_t row_hi, int32_t* parent, int32_t* out_u,
                    int32_t* out_v, unsigned long long* out_count,
                    gc_stats* stats, void* ws, size_t ws_bytes, void* stream);
int gc_shard_finish(const gc_csr* g, const gc_spec* spec, int64_t row_lo,
                    int64_t row_hi, int32_t* parent, int32_t* out_u,
                    int32_t* out_v, unsigned long long* out_count,
                    gc_stats* stats, void* ws, size_t ws_bytes, void* stream);

/* Compact phase-1 exchange for labels-only runs (no forest), in two rounds
 * (csrc/shard.cu):
 *   gc_shard_summary: compress parent in place and describe one class as an
 *     n-bit bitmap giant_bits[(n+31)/32] with its label (*giant_label,
 *     device): the class of *giant_hint (device vertex id) or, with a NULL
 *     hint, the probe's most frequent label.  With a hint (round B) parent
 *     must already be compressed, as gc_shard_absorb leaves it: the compress
 *     pass is skipped.  With out_u/out_v (capacity n)
 *     every other non-singleton vertex v also emits (v, root(v)), counted in
 *     *out_count (device); NULL pair outputs give the bitmap alone.
 *   gc_shard_absorb (round A): union every vertex of every rank's bitmap
 *     class with its class representative (bitmap classes sharing a vertex
 *     are one class); *main_rep (device) receives rank 0's class
 *     representative, the hint for round B's summary.
 *   gc_shard_join (round B): parent := the join of all ranks' partitions
 *     from their bitmaps + pairs (every bitmap member points at its class's
 *     smallest label, then the pairs are unioned with the spec's rule).
 * nranks <= 8.  ws: gc_shard_summary_workspace(n) bytes for the summary,
 * n + n/8 + 8192 for absorb, 5*n + 8192 for join. */
size_t gc_shard_summary_workspace(int64_t n);
int gc_shard_summary(int32_t* parent, int64_t n, const int32_t* giant_hint,
                     uint32_t* giant_bits, int64_t* giant_label, int32_t* out_u,
                     int32_t* out_v, unsigned long long* out_count, void* ws,
                     size_t ws_bytes, void* stream);
int gc_shard_absorb(int32_t* parent, int64_t n, const uint32_t* bits,
                    const int64_t* giant_labels, int32_t nranks,
                    int32_t* main_rep, void* ws, size_t ws_bytes, void* stream);
int gc_shard_join(int32_t* parent, int64_t n, const uint32_t* bits,
                  const int64_t* giant_labels, int32_t nranks,
                  const int32_t* us, const int32_t* vs, int64_t k,
                  const gc_spec* spec, void* ws, size_t ws_bytes, void* stream);

/* ---- distributed BFS sampling (csrc/dbfs.cu, BASELINE config 5)
 * The reference BFS (sampling.py:120-172) as a level-synchronous traversal
 * over row-sharded CSR.  Each rank owns rows [row_lo, row_hi); frontier,
 * visited, marks and next are n-bit bitmaps ((n+31)/32 words); the frontier
 * and visited bitmaps are replicated (identical on every rank).  parent is a
 * u32[n] (only the owned entries are meaningful).  A level is
 *   top-down: gc_dbfs_marks (unvisited neighbours of the block's frontier
 *     rows: marks bitmap + ascending id list out_ids, capacity n, count in
 *     *out_count, device) -> all-gather the id lists -> gc_dbfs_merge_marks
 *     for each foreign list -> gc_dbfs_claim(marks) (gc_dbfs_merge_claim:
 *     both in one call, the foreign lists concatenated);
 *   bottom-up: gc_dbfs_claim(marks = NULL).
 * gc_dbfs_claim: every unvisited (marked) vertex of the block takes the
 *   first frontier vertex of its ascending row as parent (the reference's
 *   smallest-discoverer rule) and sets its bit in next (zeroed first);
 *   *count (device) = vertices claimed.  The ranks' next bitmaps are
 *   disjoint, so their all-reduce SUM is their union; then
 * gc_dbfs_advance: visited |= next, frontier := next, *count = |next|.
 * gc_dbfs_finish: labels[v] = min reached id for reached v, else v (every
 *   vertex); the block's tree edges (parent[v], v) for reached v != source
 *   into out_u/out_v (capacity n, *out_count device); *insp (device) = degree
 *   sum of the block's reached rows (the reference's sample inspections,
 *   summed over ranks).  ws >= 16 bytes.  Malformed merged ids set *bad. */
int gc_dbfs_init(int64_t n, int64_t source, uint32_t* frontier, uint32_t* visited,
                 uint32_t* parent, void* stream);
int gc_dbfs_marks(const gc_csr* g, int64_t row_lo, int64_t row_hi,
                  const uint32_t* frontier, const uint32_t* visited,
                  uint32_t* marks, int32_t* out_ids,
                  unsigned long long* out_count, void* stream);
int gc_dbfs_merge_marks(int64_t n, const int32_t* ids, int64_t k, uint32_t* marks,
                        unsigned int* bad, void* stream);
int gc_dbfs_claim(const gc_csr* g, int64_t row_lo, int64_t row_hi,
                  const uint32_t* frontier, const uint32_t* visited,
                  const uint32_t* marks, uint32_t* parent, uint32_t* next,
                  unsigned long long* count, void* stream);
int gc_dbfs_merge_claim(const gc_csr* g, int64_t row_lo, int64_t row_hi,
                        const uint32_t* frontier, const uint32_t* visited, uint32_t* marks,
                        const int32_t* ids, int64_t k, unsigned int* bad,
                        uint32_t* parent, uint32_t* next, unsigned long long* count,
                        void* stream);
int gc_dbfs_advance(int64_t n, uint32_t* visited, uint32_t* frontier,
                    const uint32_t* next, unsigned long long* count, void* stream);
int gc_dbfs_finish(const gc_csr* g, int64_t row_lo, int64_t row_hi,
                   const uint32_t* visited, const uint32_t* parent, int32_t* labels,
                   int32_t* out_u, int32_t* out_v, unsigned long long* out_count,
                   unsigned long long* insp, void* ws, size_t ws_bytes, void* stream);

/* ---- single-process multi-device communicator (csrc/comm.cu)
 * gc_comm_init: one rank per listed device, NCCL over NVLink / NVSwitch
 *   (ncclCommInitAll) when the devices are distinct; a list that repeats one
 *   device gives a loopback communicator (ranks share it, collectives are
 *   device copies) for one-GPU hosts.  Mixed lists -> GC_ERR_ARG.
 * gc_comm_static_cc / gc_comm_spanning_forest: the two-phase sharded
 *   pipeline (gc_shard_sample -> all-gather merging edges -> gc_shard_finish
 *   -> all-gather -> gc_label_finalization), BFS sampling as the distributed
 *   traversal (gc_dbfs_*; spec->bfs_source must hold the probe source,
 *   sampling.py:130-132).  shards[r]: rank r's CSR row block [row_lo[r],
 *   row_hi[r]) resident on devs[r] (rows outside it empty, same n
 *   everywhere).  labels[r] (device, n int32, 16-byte aligned): the canonical
 *   labels, identical on every rank.  Forest: fu[r] / fv[r] (device, capacity
 *   n) receive a spanning forest of the whole graph on every rank,
 *   forest_count[r] (host) its edge count.  stats: sample / finish
 *   inspections summed over ranks, l_max / lmax_count / n_active.  Union-find
 *   finishes except JTB; samplers none / kout / hb / bfs. */
typedef struct gc_comm gc_comm;
int gc_comm_init(int ndev, const int* devs, gc_comm** out);
void gc_comm_destroy(gc_comm* comm);
int gc_comm_size(const gc_comm* comm);
int gc_comm_is_loopback(const gc_comm* comm);
int gc_comm_static_cc(gc_comm* comm, const gc_csr* shards, const int64_t* row_lo,
                      const int64_t* row_hi, const gc_spec* spec,
                      int32_t* const* labels, gc_stats* stats);
int gc_comm_spanning_forest(gc_comm* comm, const gc_csr* shards,
                            const int64_t* row_lo, const int64_t* row_hi,
                            const gc_spec* spec, int32_t* const* labels,
                            int32_t* const* fu, int32_t* const* fv,
                            int64_t* forest_count, gc_stats* stats);

/* Graph contract check (graphs.py:43-51) on device arrays: offsets start at
 * 0, never decrease and end at m; every target in [0, n) -> else
 * GC_ERR_MALFORMED.  One streaming pass; the Python layer runs it once per
 * Graph before the first kernel touches it (an out-of-range target would
 * otherwise be an out-of-bounds parent access). */
int gc_check_csr(const gc_csr* g, void* stream);

/* ---- DisjointSets probes and validation (dset.py:381-399,
 *      validate.py:178-259) -------------------------------------------------
 * gc_find_batch: roots_out[i] = find(xs[i]) with the given gc_find_kind,
 * applying its compaction writes to parent (DisjointSets.find_root); xs ==
 * NULL means xs[i] = i (k <= n).  GC_FIND_NAIVE is the read-only probe of
 * same_set / labels_array. */
int gc_find_batch(int32_t* parent, int64_t n, const int32_t* xs, int64_t k,
                  int32_t find_kind, int32_t* roots_out, void* stream);
/* canonical_labels (validate.py:251-259) in place: each label value becomes
 * the minimum index carrying it.  Values must lie in [0, n); ws needs
 * 4*n + 512 bytes. */
int gc_canonical_labels(int32_t* labels, int64_t n, void* ws, size_t ws_bytes,
                        void* stream);
/* The census of a labelling (validate.py:267-298 sampling_stats): out_host[0]
 * = most frequent label (ties -> smaller), [1] its multiplicity (cov =
 * [1] / n), [2] directed CSR entries whose endpoints carry different labels
 * (ic = [2] / m), [3] = -1, or with a non-NULL oracle labelling the smallest
 * vertex whose class (by `labels`) is not inside one oracle class — the
 * refinement check of validate.py:290-297.  Labels must lie in [0, n);
 * ws needs 4*n + 8192 bytes.  Synchronous. */
int gc_label_census(const gc_csr* g, const int32_t* labels, const int32_t* oracle,
                    int64_t* out_host, void* ws, size_t ws_bytes, void* stream);
/* check_forest clause (a) (validate.py:200-206): *first_missing (device)
 * receives the smallest i whose (us[i], vs[i]) is not in the CSR, or
 * UINT64_MAX when every edge exists. */
int gc_edges_exist(const gc_csr* g, const int32_t* us, const int32_t* vs,
                   int64_t k, unsigned long long* first_missing, void* stream);

/* ---- incremental (driver.py:567-725) -------------------------------------*/
typedef struct gc_incr gc_incr;
/* capacity = number of vertex slots; sentinel = capacity (driver.py:603). */
int gc_incr_create(int64_t capacity, const gc_spec* spec, void* stream,
                   gc_incr** out);
/* One batch: ops[i] = (us[i], vs[i]) is an insert if is_query[i]==0, else a
 * query.  Insert sub-phase, barrier, query sub-phase (driver.py:695-708);
 * racy != 0 interleaves them (driver.py:674-694).  bits_out receives one bit
 * per op packed LSB-first into ceil(len/32) words (bit i%32 of word i/32;
 * 1 = query answered connected, inserts read 0) — the reference's per-op
 * result bits (driver.py:658-668), written as one __ballot_sync word per 32
 * ops.  Times are accumulated into stats->t_sample_ms (insert) and
 * stats->t_finish_ms (query).
 * Endpoints must lie in [0, capacity): an op with an endpoint outside it is
 * skipped on the device (never touching the state) and the call returns
 * GC_ERR_MALFORMED (for gc_incr_insert_async: the next synchronising call
 * on the handle does). */
int gc_incr_batch(gc_incr* h, const int32_t* us, const int32_t* vs,
                  const uint8_t* is_query, int64_t len, uint32_t* bits_out,
                  int racy, gc_stats* stats);
/* Enqueue all later work of the handle on `stream` (ordered after the work
 * already enqueued on the previous stream).  The Python layer calls it so a
 * handle always runs on the caller's current stream. */
int gc_incr_set_stream(gc_incr* h, void* stream);
/* Columnar insert-only / query-only fast paths (no per-op flag array). */
int gc_incr_insert(gc_incr* h, const int32_t* us, const int32_t* vs,
                   int64_t len, gc_stats* stats);
/* As gc_incr_insert, but for union-find specs the batch is only enqueued on
 * the handle's stream (no synchronisation, no per-batch phase time): a stream
 * of inserts then runs back to back; gc_incr_query / gc_incr_labels /
 * gc_incr_state order after it.  Round finishes behave as gc_incr_insert. */
int gc_incr_insert_async(gc_incr* h, const int32_t* us, const int32_t* vs, int64_t len, gc_stats* stats);
/* Insert-only batch that also records the edges that merged two trees
 * (capacity len) — the per-batch exchange of the sharded incremental driver. */
int gc_incr_insert_list(gc_incr* h, const int32_t* us, const int32_t* vs,
                        int64_t len, int32_t* out_u, int32_t* out_v,
                        unsigned long long* out_count, gc_stats* stats);
/* Query-only batch; bits_out packed as in gc_incr_batch. */
int gc_incr_query(gc_incr* h, const int32_t* us, const int32_t* vs,
                  int64_t len, uint32_t* bits_out, gc_stats* stats);
/* Copy of the live state with the sentinel convention (driver.py:656,710). */
int gc_incr_state(gc_incr* h, int32_t* state_out);
/* The live state itself (driver.py:710-711 hands `on_batch` the live parent
 * list / label array): after synchronising the handle's stream, *state
 * receives the device pointer of the state array and *slots its length
 * (capacity, or capacity + 1 for SV / LT).  Valid until the next call that
 * mutates the handle; the caller must not write it. */
int gc_incr_state_view(gc_incr* h, int32_t** state, int64_t* slots);
/* Final labels (driver.py:715-725); returns the component count of the
 * initialized vertices in *components. */
int gc_incr_labels(gc_incr* h, int32_t* labels_out, int64_t* components);
int64_t gc_incr_capacity(gc_incr* h);
/* Pre-size the per-batch work buffers of the round finishes (SV / LT) for
 * batches of up to `batch_len` ops, so the first batch does not pay their
 * allocation.  No-op for union-find specs. */
int gc_incr_reserve(gc_incr* h, int64_t batch_len);
void gc_incr_destroy(gc_incr* h);

/* ---- graph generators + CSR build (graphs.py:90-121, 210-245, 297-308) ----
 * gc_gen_rmat reproduces numpy's PCG64 stream bit-for-bit: (state_hi,
 * state_lo, inc_hi, inc_lo) is `default_rng(seed).bit_generator.state`, and
 * base[4] = (a, b, c, d) exactly as the reference computes them.  Output:
 * src[ef*n], dst[ef*n] int64 pairs in the reference order. */
int gc_gen_rmat(int32_t scale, int64_t num_pairs, const double* base_host,
                uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                uint64_t inc_lo, int64_t* src, int64_t* dst, void* stream);
/* numpy Generator.integers(0, n, size=(k, 2), dtype=int64) for n = 2^log2n
 * (Lemire path without rejection). */
int gc_gen_uniform_pow2(int32_t log2n, int64_t num_pairs, uint64_t state_hi,
                        uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                        int64_t* src, int64_t* dst, void* stream);
/* Symmetrize, drop self-loops, dedupe, sort (build_csr semantics,
 * graphs.py:90-121).  targets must have capacity 2*k; *m_out (host) receives
 * the directed entry count.  An endpoint outside [0, n) -> GC_ERR_MALFORMED.
 * ws needs gc_build_csr_workspace(n, k) bytes. */
size_t gc_build_csr_workspace(int64_t n, int64_t k);
int gc_build_csr(int64_t n, const int64_t* src, const int64_t* dst, int64_t k,
                 int64_t* offsets, int32_t* targets, int64_t* m_out, void* ws,
                 size_t ws_bytes, void* stream);

/* Host helper: MT19937 continuing from Python random.Random().getstate()
 * (624 words + index): out[i] = getrandbits(32).  Used for the JTB ranks of
 * DisjointSets (dset.py:372-374). */
int gc_mt19937_fill(const uint32_t* state624, int32_t index, uint32_t* out,
                    int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* GCONN_H_ */
