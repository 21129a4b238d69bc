// rounds.h — min-label round finishes (minbased.py:124-304): Shiloach-
// Vishkin, the sixteen Liu-Tarjan variants, Stergiou and label propagation.
//
// Rounds are Jacobi exactly as in the reference (every read in a round sees
// the round's starting snapshot; writes are commutative atomic minima), so
// round counts and inspection counts match the oracle bit for bit.
#pragma once

#include "internal.h"

namespace gc {

// Working edge set in COO form.  Twin directed entries (u,t)/(t,u) of two
// active vertices are stored once with weight 2: every round rule here is
// symmetric in the endpoints, so the messages are identical, and the kept
// entry is the one with the smaller reference COO index (the row of the
// smaller endpoint), which preserves the forest tie-break
// (minbased.py:95-116).  Weighted counts reproduce the reference's per-round
// len(work) inspections.
struct Coo {
  int32_t* u = nullptr;
  int32_t* v = nullptr;
  int64_t* idx = nullptr;   // reference edge index (CSR position), forest only
  uint8_t* w = nullptr;     // 1 or 2
  int64_t len = 0;          // stored entries
  int64_t weight = 0;       // reference entries (sum of w)
};

struct RoundsWs {
  int32_t* a = nullptr;      // prev / snapshot
  int32_t* b = nullptr;      // cur / msg
  unsigned long long* win = nullptr;  // forest winner edge index per root
  int64_t* cnt = nullptr;    // gather cursor (one word)
  Coo work, spare;
  uint8_t* keep = nullptr;   // SV: per working edge, snapshot labels differ
  int64_t* chunks = nullptr; // SV: per-block chunk [start, len] tables
};

// upper bound of the edge-kernel grid (grid_for(.., 256, 8) on 148 SMs)
constexpr int64_t kMaxChunks = 148 * 8 * 8;


template <class A>
void rounds_carve(A& a, RoundsWs& w, int64_t n, int64_t m, const gc_spec& s, bool forest) {
  (void)s;
  w.a = a.template take<int32_t>(n + 1);
  w.b = a.template take<int32_t>(n + 1);
  if (forest) w.win = a.template take<unsigned long long>(n + 1);
  w.cnt = a.template take<int64_t>(2);
  for (Coo* c : {&w.work, &w.spare}) {
    c->u = a.template take<int32_t>(m);
    c->v = a.template take<int32_t>(m);
    c->w = a.template take<uint8_t>(m);
    if (forest) c->idx = a.template take<int64_t>(m);
  }
  if (s.finish == GC_FINISH_SV) {
    w.keep = a.template take<uint8_t>(m);
    w.chunks = a.template take<int64_t>(2 * kMaxChunks + 4);
  }
}

// Static / finish-phase driver: gathers the working COO of the active rows
// (all rows when list == nullptr) and runs the configured rounds on P.
// Returns the round count.
// cut_ready: work.u / work.v already hold every edge between two different
// labels once (LDD's cut edges, count in ctr[C_CUT]); they are oriented and
// weighted in place instead of gathered from the active rows.
int64_t run_rounds_finish(const gc_csr& g, const gc_spec& s, int32_t* P, const int32_t* list,
                          unsigned long long* ctr, int32_t* fu, int32_t* fv, RoundsWs& w,
                          cudaStream_t st, bool cut_ready = false);

// Incremental driver: rounds over an explicit batch COO on labels[nl]
// (nl = capacity + 1, minbased.py:124 / :163 with phase="insert").
int64_t run_rounds_coo(const gc_spec& s, int32_t* labels, int64_t nl, Coo& work, RoundsWs& w,
                       unsigned long long* ctr, int counter_slot, cudaStream_t st);

}  // namespace gc
