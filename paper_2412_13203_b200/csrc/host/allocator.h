// Workload Allocator, Algorithm 2 of the paper as the
// SPEC's workload_allocator module states it:
//
//   while any class improved:
//     for each class c:  t1 = measure(c, g_c); combine (g_c -> 2 g_c, capped);
//                        t2 = measure(c, 2 g_c); keep if t2 < t1 else revert
//
// Granularity g_c = work items fused into one warp task for class c (Combine
// "merges more basic computational units into a bigger one"; a work item is
// 32 contracted quartets, one per lane, each looping over its primitive
// quartets). Cap = min(task count, 4096). measure() returns the
// median of R repeated timings on a fixed sample (the class's work list) with
// the warm-up discarded; the spread is kept in the history.
// Header-only and device-free, so the loop itself is unit-tested on the CPU
// against the SPEC's mock-cost examples (eritile_alloc_simulate).
#pragma once
#include <utility>
#include <vector>

namespace eritile_b200 {

struct AllocMeasure {
  double median;  // seconds (or ms): what the loop compares
  double spread;  // max - min of the R repeats (reported, not compared)
};

struct AllocState {
  std::vector<int> g;       // granularity per class (>= 1)
  std::vector<int> cap;     // per class; cap <= 1 means "not tunable"
  std::vector<double> t;    // last accepted median per class
  struct Step {
    int g;
    double median, spread;
    bool accepted;
  };
  std::vector<std::vector<Step>> history;  // per class: every measured (g, t)
  int accepted = 0;  // accepted combines
  int sweeps = 0;    // sweeps run (the last one found no improvement if converged)

  void init(int ncls) {
    g.assign(ncls, 1);
    cap.assign(ncls, 1);
    t.assign(ncls, 0.0);
    history.assign(ncls, {});
    accepted = sweeps = 0;
  }
};

// combine: g -> 2g unless at the cap (returns false: capped, nothing changed)
inline bool alloc_combine(AllocState& s, int c) {
  if (2LL * s.g[c] > s.cap[c]) return false;
  s.g[c] *= 2;
  return true;
}
// revert the combine of this round
inline void alloc_revert(AllocState& s, int c) { s.g[c] /= 2; }

// One sweep over all classes; true if any class improved.
// measure(c, g) -> AllocMeasure for class c at granularity g.
template <class M>
bool alloc_sweep(AllocState& s, M&& measure) {
  bool improved = false;
  for (int c = 0; c < static_cast<int>(s.g.size()); ++c) {
    if (2LL * s.g[c] > s.cap[c]) continue;  // capped: combine is a no-op
    const AllocMeasure t1 = measure(c, s.g[c]);
    s.history[c].push_back({s.g[c], t1.median, t1.spread, true});
    alloc_combine(s, c);
    const AllocMeasure t2 = measure(c, s.g[c]);
    if (t2.median < t1.median) {
      s.history[c].push_back({s.g[c], t2.median, t2.spread, true});
      s.t[c] = t2.median;
      ++s.accepted;
      improved = true;
    } else {
      s.history[c].push_back({s.g[c], t2.median, t2.spread, false});
      alloc_revert(s, c);
      s.t[c] = t1.median;
    }
  }
  ++s.sweeps;
  return improved;
}

// The full loop: sweeps until one finds no improvement (terminates: every
// accepted step doubles some g_c, which is capped).
template <class M>
void alloc_tune(AllocState& s, M&& measure, int max_sweeps = 64) {
  while (s.sweeps < max_sweeps && alloc_sweep(s, measure)) {
  }
}

}  // namespace eritile_b200
