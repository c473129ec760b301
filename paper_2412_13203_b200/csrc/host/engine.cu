// eritile_gpu engine: host Block Constructor, screening, work lists, launch
// orchestration and the C ABI (include/eritile_gpu.h).
//
// Host Block Constructor (block.hpp:52-150 restated for the GPU):
//  * reference pair store: all S(S+1)/2 shell pairs i<=j with the kappa
//    screen of block.hpp:83-89, ordered by (Li+Lj, Li, Lj, i, j)
//    (block.hpp:94-101) — gives each pair its reference index `ref`;
//  * product pairs: the same pairs oriented A = higher-L shell, grouped by
//    (L_A+L_B, L_A, L_B, K) and, once Schwarz Q is known, sorted by Q
//    descending inside each group. Surviving kets of a bra are then a prefix
//    of every ket group, so quartet lists are (bra, ket range) work items;
//  * work items: one warp per (bra x, <=32 consecutive kets) of one ket
//    group, class-homogeneous and contraction-homogeneous (Permutation).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "allocator.h"
#include "../../../include/eritile_gpu.h"
#include "../jk_api.h"
#include "../jk_kernels.cuh"
#include "../jk_family.cuh"
#include "molecule.h"
#include "onee.h"

namespace eritile_b200 {

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};
struct StateError : std::runtime_error {
  explicit StateError(const std::string& m) : std::runtime_error(m) {}
};
struct ArgError : std::runtime_error {
  explicit ArgError(const std::string& m) : std::runtime_error(m) {}
};

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess)                                                                     \
      throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));                       \
  } while (0)

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    if (count <= n && p) return;
    release();
    if (count == 0) return;
    CK(cudaMalloc(&p, sizeof(T) * count));
    n = count;
  }
  // Stream-ordered and complete on return: a pageable cudaMemcpy may return
  // before its DMA lands, and kernels on a non-blocking stream would not wait
  // for it.
  void upload(const std::vector<T>& v, cudaStream_t st) {
    alloc(v.size());
    if (v.empty()) return;
    CK(cudaMemcpyAsync(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
  void download(T* dst, size_t count, cudaStream_t st) const {
    if (count == 0) return;
    CK(cudaMemcpyAsync(dst, p, sizeof(T) * count, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
};

// ------------------------------------------------------------ Boys table
// F_m(T_i) for T_i = i/16 by the convergent series
// F_m(T) = e^-T sum_k (2T)^k / ((2m+1)(2m+3)...(2m+2k+1)) in long double
// (all terms positive: no cancellation), stored as F_{M+k}(T_i)/k!, k<8,
// plus exp(-T_i) per row, for each slice M = 0..kBoysMmax.
static std::vector<double> make_boys_table() {
  const int mtop = kBoysMmax + 8;
  std::vector<long double> F(static_cast<size_t>(kBoysRows) * (mtop + 1));
  for (int i = 0; i < kBoysRows; ++i) {
    const long double T = static_cast<long double>(i) / 16.0L;
    const long double eT = expl(-T);
    for (int m = 0; m <= mtop; ++m) {
      long double term = 1.0L / (2 * m + 1), sum = term;
      for (int k = 0; k < 2000; ++k) {
        term *= 2.0L * T / (2 * m + 2 * k + 3);
        sum += term;
        if (term < 1e-22L * sum) break;
      }
      F[static_cast<size_t>(i) * (mtop + 1) + m] = eT * sum;
    }
  }
  std::vector<double> tab(static_cast<size_t>(kBoysMmax + 1) * kBoysRows * kBoysCols);
  const long double fact[8] = {1, 1, 2, 6, 24, 120, 720, 5040};
  for (int M = 0; M <= kBoysMmax; ++M)
    for (int i = 0; i < kBoysRows; ++i) {
      double* row = tab.data() + (static_cast<size_t>(M) * kBoysRows + i) * kBoysCols;
      for (int k = 0; k < 8; ++k)
        row[k] = static_cast<double>(F[static_cast<size_t>(i) * (mtop + 1) + M + k] / fact[k]);
      row[8] = static_cast<double>(expl(-static_cast<long double>(i) / 16.0L));
      row[9] = 0.0;
    }
  return tab;
}

// ------------------------------------------------------------- kernels
__global__ void k_prescale(const double* __restrict__ D, const double* __restrict__ s, double* __restrict__ Ds,
                           int N) {
  const size_t NN = static_cast<size_t>(N) * N;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < NN;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = e / N, c = e % N;
    Ds[e] = D[e] * (s[r] * s[c]);
  }
}

// true J = s_mu s_nu (Jacc + Jacc^T)/2, true K likewise (Appendix C).
// det: the accumulators hold int64 fixed point (kDetScale, red_add).
__global__ void k_finalize(const double* __restrict__ Jacc, const double* __restrict__ Kacc,
                           const double* __restrict__ s, double* __restrict__ J, double* __restrict__ K,
                           int N, int det) {
  const size_t NN = static_cast<size_t>(N) * N;
  const long long* Ji = reinterpret_cast<const long long*>(Jacc);
  const long long* Ki = reinterpret_cast<const long long*>(Kacc);
  const double inv = 1.0 / kDetScale;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < NN;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = e / N, c = e % N, t = c * N + r;
    const double f = 0.5 * (s[r] * s[c]);
    if (det) {
      J[e] = f * (static_cast<double>(Ji[e]) * inv + static_cast<double>(Ji[t]) * inv);
      K[e] = f * (static_cast<double>(Ki[e]) * inv + static_cast<double>(Ki[t]) * inv);
    } else {
      J[e] = f * (Jacc[e] + Jacc[t]);
      K[e] = f * (Kacc[e] + Kacc[t]);
    }
  }
}

template <int M>
__device__ void boys_one(double T, const double* tab, double* out) {
  double F[M + 1];
  boys_eval<M>(T, tab + static_cast<size_t>(M) * kBoysRows * kBoysCols, F);
  for (int m = 0; m <= M; ++m) out[m] = F[m];
}

// Device Boys values for tests (eritile_gpu_boys); table read from global.
__global__ void k_boys(int m_max, const double* __restrict__ T, int n, const double* __restrict__ tab,
                       double* __restrict__ F) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* o = F + static_cast<size_t>(i) * (m_max + 1);
  switch (m_max) {
    case 0: boys_one<0>(T[i], tab, o); break;
    case 1: boys_one<1>(T[i], tab, o); break;
    case 2: boys_one<2>(T[i], tab, o); break;
    case 3: boys_one<3>(T[i], tab, o); break;
    case 4: boys_one<4>(T[i], tab, o); break;
    case 5: boys_one<5>(T[i], tab, o); break;
    case 6: boys_one<6>(T[i], tab, o); break;
    case 7: boys_one<7>(T[i], tab, o); break;
    case 8: boys_one<8>(T[i], tab, o); break;
    case 9: boys_one<9>(T[i], tab, o); break;
    case 10: boys_one<10>(T[i], tab, o); break;
    case 11: boys_one<11>(T[i], tab, o); break;
    case 12: boys_one<12>(T[i], tab, o); break;
    case 13: boys_one<13>(T[i], tab, o); break;
    case 14: boys_one<14>(T[i], tab, o); break;
    case 15: boys_one<15>(T[i], tab, o); break;
    default: boys_one<16>(T[i], tab, o); break;
  }
}

// ---------------------------------------------------------------- context
struct Group {
  int la, lb, K;
  int first, count;  // product pair ids (units for unit groups)
  int nm = 1;        // unit groups: members per unit
};

// One class work list. The full (unsharded) list lives in all_items at
// [aoff, aoff + an); this rank's share (the LPT deal, eritile_gpu::deal) is
// [off, off + n) of the rank-local list. Unit classes keep their (1,1)
// (1,2) (2,1) (2,2) member segments contiguous in both (seg relative to off).
struct ClassWork {
  int cls;  // index into kClassTable
  bool fam; // items index units (shared-primitive kernels)
  long long aoff = 0, an = 0;
  long long aseg[5] = {0, 0, 0, 0, 0};
  long long aquartets = 0, aprim = 0;
  double cost_prim = 0.0, cost_q = 0.0;  // model FLOPs per primitive / contracted quartet
  // strips (csrc/jk_strip.cuh): per member segment sg, strips [asseg[sg],
  // asseg[sg+1]) of all_strips (from astrip_off) own the single-bra items
  // [aseg[sg], asitem[sg]); the packed multi-bra items follow up to aseg[sg+1]
  long long astrip_off = 0;
  long long asseg[5] = {0, 0, 0, 0, 0};
  long long asitem[4] = {0, 0, 0, 0};
  long long off = 0, n = 0;
  long long seg[5] = {0, 0, 0, 0, 0};
  long long strip_off = 0;
  long long sseg[5] = {0, 0, 0, 0, 0};
  long long sitem[4] = {0, 0, 0, 0};
  long long quartets = 0, prim_quartets = 0;
  double flops = 0.0;    // model FLOPs of this rank's launch
  double last_ms = 0.0;  // device time of the last launch (profiling mode)
  double full_flops() const { return cost_prim * static_cast<double>(aprim) + cost_q * static_cast<double>(aquartets); }
};

}  // namespace eritile_b200

using namespace eritile_b200;

struct eritile_gpu {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::string err;

  std::vector<Atom> atoms;
  std::vector<ShellData> shells;
  std::vector<int> bf_off;
  std::vector<double> bf_scale;
  int nbf = 0;
  bool have_mol = false;

  // reference pair store
  std::vector<int> ref_i, ref_j;
  // product pairs
  std::vector<PairMeta> pm;   // product order
  std::vector<PrimRec> prims;
  std::vector<PrimRec> kprims;  // group-transposed ket copy (build_ket_soa)
  std::vector<int> prod_of_ref;  // ref index -> product id
  std::vector<int> cls_of_pair;  // canonical pair class index per product pair
  std::vector<Group> groups;
  std::vector<double> Q;  // product order
  bool have_pairs = false, have_q = false, have_lists = false;
  int rank = 0, nranks = 1;
  double tau = 0.0;

  std::vector<WorkItem> all_items;        // every class list, unsharded
  std::vector<unsigned char> item_q;      // contracted quartets per item (all_items)
  std::vector<unsigned> item_p;           // primitive quartets per item (all_items)
  std::vector<WorkItem> items;            // this rank's items (nranks > 1)
  std::vector<Strip> all_strips, strips;  // strip tables (full lists / this rank)
  // compact K/D columns per ket class (L_C, L_D): list of the L_C functions
  // (++ the L_D functions when L_D != L_C); cpos per shell
  std::vector<int> shell_cpos, cols_all;
  int cols_off[8][8] = {}, cols_n[8][8] = {}, cols_nc[8][8] = {};
  DevBuf<int> d_cpos, d_cols;
  DevBuf<Strip> d_all_strips, d_strips;
  DevBuf<int> d_sctr;  // 4 strip hand-out counters per work entry (zeroed by each strip launch)
  std::vector<int> cnt;  // survivor counts per (group pair, bra) + sentinel
  std::vector<ClassWork> work;
  bool dealt = false;   // rank-local lists match the current variants and shard
  long long quartets = 0, prim_quartets = 0;
  double model_flops = 0.0;
  double last_build_ms = 0.0, last_schwarz_ms = 0.0;
  int launches_last = 0;

  DevBuf<PairMeta> d_pm;
  DevBuf<PrimRec> d_prims, d_kprims;
  DevBuf<double> d_boys, d_scale, d_Q;
  DevBuf<WorkItem> d_all_items, d_items;
  DevBuf<int> d_cnt;
  DevBuf<int> d_list;
  DevBuf<double> d_D, d_Ds, d_JK, d_J, d_K;

  // shared-primitive units (csrc/jk_family.cuh)
  bool families = true;
  std::vector<int> sib;                 // sibling id per shell (centre, L, exponents)
  std::vector<unsigned long long> fam_key_ref;  // per reference pair: prim-set signature
  std::vector<int> fam_sib_ref;         // per reference pair: sib(A) * nshell + sib(B)
  std::vector<UnitMeta> um;
  std::vector<Group> ugroups;
  std::vector<double> uQ;
  std::vector<double2> uw;
  std::vector<PrimRec> ukprims;
  std::vector<double2> ukw;
  DevBuf<UnitMeta> d_um;
  DevBuf<KetMeta> d_kmu, d_kmp;  // KetMeta per unit / per product pair
  DevBuf<double2> d_uw, d_ukw;
  DevBuf<PrimRec> d_ukprims;
  DevBuf<double> d_Qp;

  // Classes with unit ("fam_") variants get both work lists (pair items and
  // unit items); the chosen variant decides which one a build launches.
  bool fam_active(int c) const { return families && kClassTable[c].nfam > 0; }
  int var_lo(int) const { return 0; }
  int var_hi(int c) const { return fam_active(c) ? kClassTable[c].nvar : kClassTable[c].nvar - kClassTable[c].nfam; }
  bool uses_fam(int c) const { return fam_active(c) && variant(c) >= kClassTable[c].nvar - kClassTable[c].nfam; }
  bool active(const ClassWork& cw) const { return cw.fam == uses_fam(cw.cls); }
  // kernels one class launch issues: unit classes launch each non-empty
  // member segment separately
  int kernel_launches(const ClassWork& cw) const {
    if (!cw.fam) return 1;
    int k = 0;
    for (int i = 0; i < 4; ++i) k += cw.seg[i + 1] > cw.seg[i] ? 1 : 0;
    return k;
  }
  std::vector<int> active_work() const {
    std::vector<int> o;
    for (size_t w = 0; w < work.size(); ++w)
      if (active(work[w])) o.push_back(static_cast<int>(w));
    return o;
  }
  // totals over the launches a build makes
  void update_totals() {
    quartets = prim_quartets = 0;
    model_flops = 0.0;
    for (int w : active_work()) {
      quartets += work[w].quartets;
      prim_quartets += work[w].prim_quartets;
      model_flops += work[w].flops;
    }
  }

  // Workload Allocator state: kernel variant per class (kClassTable[c].var)
  // and the Alg. 2 granularity per class (allocator.h)
  std::vector<int> var_choice;
  AllocState alloc;
  int gran(int c) const { return alloc.g.empty() ? 1 : alloc.g[c]; }
  std::vector<double> tune_ms;  // per class launch x kMaxVariants: median ms (tune)

  bool profiling = false;
  bool det = false;  // deterministic reduction mode (fixed-point integer atomics)
  bool host_only = false;  // device < 0: block constructor / lists only
  std::vector<cudaEvent_t> prof_ev;

  static constexpr int kSide = 3;
  bool concurrent = true;
  cudaStream_t side[kSide] = {nullptr, nullptr, nullptr};
  cudaEvent_t side_ev[kSide] = {nullptr, nullptr, nullptr};
  cudaEvent_t fork_ev = nullptr;

  ~eritile_gpu() {
    for (int k = 0; k < kSide; ++k) {
      if (side[k]) cudaStreamDestroy(side[k]);
      if (side_ev[k]) cudaEventDestroy(side_ev[k]);
    }
    if (fork_ev) cudaEventDestroy(fork_ev);
    for (cudaEvent_t e : prof_ev) cudaEventDestroy(e);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
  }

  int variant(int c) const {
    const int v = var_choice.empty() ? -1 : var_choice[c];
    if (v >= var_lo(c) && v < var_hi(c)) return v;
    return kClassTable[c].def;
  }

  // Workload Allocator (Alg. 2): for every
  // class launch of this rank, time each kernel variant (median of R
  // launches, CUDA events) on the live density and keep the fastest. The
  // reference tunes a granularity g by doubling; here the tuned knob is the
  // variant (lane kernel residency / CTA-cooperative split), whose choice
  // cannot change results beyond atomic summation order.
  void tune(const double* dDs, int reps) {
    if (var_choice.empty()) {
      var_choice.resize(kNumClasses);
      for (int c = 0; c < kNumClasses; ++c) var_choice[c] = -1;
    }
    const size_t NN = static_cast<size_t>(nbf) * nbf;
    DevBuf<double> scratch;
    scratch.alloc(2 * NN);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    tune_ms.assign(static_cast<size_t>(kNumClasses) * kMaxVariants, 0.0);
    std::vector<int> pair_w(kNumClasses, -1), fam_w(kNumClasses, -1);
    for (size_t w = 0; w < work.size(); ++w) (work[w].fam ? fam_w : pair_w)[work[w].cls] = static_cast<int>(w);
    for (int c = 0; c < kNumClasses; ++c) {
      if (pair_w[c] < 0 && fam_w[c] < 0) continue;
      const ClassEntry& ce = kClassTable[c];
      double best = 1e300;
      int bestv = variant(c);
      for (int v = var_lo(c); v < var_hi(c); ++v) {
        const bool famv = v >= ce.nvar - ce.nfam;
        const int w = famv ? fam_w[c] : pair_w[c];
        if (w < 0) continue;
        std::vector<double> t;
        for (int r = 0; r < reps + 1; ++r) {
          LaunchArgs a = class_args(work[w], dDs, scratch.p, stream, true);
          CK(cudaEventRecord(e0, stream));
          ce.var[v](a);
          CK(cudaGetLastError());
          CK(cudaEventRecord(e1, stream));
          CK(cudaEventSynchronize(e1));
          if (r > 0) t.push_back(elapsed(e0, e1));  // first launch warms up
        }
        std::sort(t.begin(), t.end());
        const double med = t[t.size() / 2];
        tune_ms[static_cast<size_t>(c) * kMaxVariants + v] = med;
        if (med < best) {
          best = med;
          bestv = v;
        }
      }
      var_choice[c] = bestv;
    }
    dealt = false;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }

  // Work list of class c under its current variant (-1: no work).
  int chosen_work(int c) const {
    for (size_t w = 0; w < work.size(); ++w)
      if (work[w].cls == c && work[w].fam == uses_fam(c)) return static_cast<int>(w);
    return -1;
  }
  // Alg. 2 caps: min(task count, 4096) for classes whose variant takes the
  // granularity (lane, unit and strip kernels; the coop table kernels do not).
  void alloc_caps() {
    if (alloc.g.empty()) alloc.init(kNumClasses);
    for (int c = 0; c < kNumClasses; ++c) {
      const int w = chosen_work(c);
      const std::string vn = kClassTable[c].var_name[variant(c)];
      if (w < 0 || vn.rfind("coop", 0) == 0) {
        alloc.cap[c] = 1;
        alloc.g[c] = 1;
        continue;
      }
      alloc.cap[c] = static_cast<int>(std::min<long long>(work[w].an, 4096));
      if (alloc.g[c] > alloc.cap[c]) alloc.g[c] = 1;
    }
  }
  // measure(c, g): median (and spread) of R timed launches of class c's
  // chosen variant at granularity g on the full work list, warm-up discarded.
  AllocMeasure measure_class(int c, int g, const double* dDs, double* scratch, int reps, cudaEvent_t e0,
                             cudaEvent_t e1) {
    const int w = chosen_work(c);
    std::vector<double> t;
    for (int r = 0; r < reps + 1; ++r) {
      LaunchArgs a = class_args(work[w], dDs, scratch, stream, true);
      a.gran = g;
      CK(cudaEventRecord(e0, stream));
      kClassTable[c].var[variant(c)](a);
      check_launch(work[w]);
      CK(cudaEventRecord(e1, stream));
      CK(cudaEventSynchronize(e1));
      if (r > 0) t.push_back(elapsed(e0, e1));
    }
    std::sort(t.begin(), t.end());
    return AllocMeasure{t[t.size() / 2], t.back() - t.front()};
  }
  // Alg. 2 on the live density: one sweep (SCF interleave) or to convergence.
  // Returns true if the (last) sweep improved some class.
  bool tune_granularity(const double* dDs, int reps, int max_sweeps) {
    alloc_caps();
    const size_t NN = static_cast<size_t>(nbf) * nbf;
    DevBuf<double> scratch;
    scratch.alloc(2 * NN);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    bool improved = false;
    try {
      auto m = [&](int c, int g) { return measure_class(c, g, dDs, scratch.p, reps, e0, e1); };
      const int s0 = alloc.sweeps;
      while (alloc.sweeps - s0 < max_sweeps) {
        improved = alloc_sweep(alloc, m);
        if (!improved) break;
      }
    } catch (...) {
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      throw;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return improved;
  }

  // full = true: the class's whole (unsharded) list (the allocator times
  // those); else this rank's share.
  LaunchArgs class_args(const ClassWork& cw, const double* dDs, double* dJK, cudaStream_t st,
                        bool full = false) const {
    const size_t NN = static_cast<size_t>(nbf) * nbf;
    LaunchArgs a{};
    a.mode = 0;
    const bool use_all = full || nranks == 1;
    a.det = det ? 1 : 0;
    a.items = use_all ? d_all_items.p + cw.aoff : d_items.p + cw.off;
    a.nitems = full ? cw.an : cw.n;
    a.cnt = d_cnt.p;
    a.pm = d_pm.p;
    a.prims = d_prims.p;
    a.kprims = d_kprims.p;
    a.D = dDs;
    a.J = dJK;
    a.K = dJK + NN;
    a.N = nbf;
    a.boys_tab = d_boys.p;
    a.stream = st;
    a.block = 128;
    for (int k = 0; k < 5; ++k) a.seg[k] = full ? cw.aseg[k] : cw.seg[k];
    for (int k = 0; k < 5; ++k) a.sseg[k] = use_all ? cw.asseg[k] : cw.sseg[k];
    for (int k = 0; k < 4; ++k) a.sitem[k] = use_all ? cw.asitem[k] : cw.sitem[k];
    a.strips = use_all ? d_all_strips.p + cw.astrip_off : d_strips.p + cw.strip_off;
    a.sctr = d_sctr.p ? d_sctr.p + 4 * (&cw - work.data()) : nullptr;
    {
      const ClassEntry& ce = kClassTable[cw.cls];
      a.cols = d_cols.p + cols_off[ce.lc][ce.ld];
      a.ncols = cols_n[ce.lc][ce.ld];
      a.ncolC = cols_nc[ce.lc][ce.ld];
      a.cpos = d_cpos.p;
    }
    a.kmeta = cw.fam ? d_kmu.p : d_kmp.p;
    a.gran = gran(cw.cls);
    if (cw.fam) {
      a.um = d_um.p;
      a.uw = d_uw.p;
      a.ukprims = d_ukprims.p;
      a.ukw = d_ukw.p;
      a.Qp = d_Qp.p;
      a.tau = tau;
    }
    return a;
  }

  int class_index(int la, int lb, int lc, int ld) const {
    for (int c = 0; c < kNumClasses; ++c)
      if (kClassTable[c].la == la && kClassTable[c].lb == lb && kClassTable[c].lc == lc &&
          kClassTable[c].ld == ld)
        return c;
    throw ArgError("no generated kernel for class (" + std::to_string(la) + "," + std::to_string(lb) + "," +
                   std::to_string(lc) + "," + std::to_string(ld) + ")");
  }

  void set_molecule(std::vector<Atom> a, std::vector<ShellData> s) {
    for (const auto& sh : s)
      if (sh.L > kMaxL) throw ArgError("shell angular momentum exceeds compiled classes");
    if (s.empty()) throw ArgError("build_pairs: no shells");
    atoms = std::move(a);
    shells = std::move(s);
    bf_off.assign(shells.size() + 1, 0);
    bf_scale.clear();
    std::vector<std::array<int, 3>> comps;
    for (size_t i = 0; i < shells.size(); ++i) {
      bf_off[i + 1] = bf_off[i] + shells[i].nfunc();
      cart_components(shells[i].L, comps);
      for (auto& c : comps) bf_scale.push_back(component_scale(c[0], c[1], c[2]));
    }
    nbf = bf_off.back();
    // sibling shells: same centre, L and exponents (general contractions
    // written in segmented form, e.g. cc-pVDZ O 1s/2s)
    {
      std::map<std::vector<double>, int> ids;
      sib.assign(shells.size(), 0);
      for (size_t i = 0; i < shells.size(); ++i) {
        std::vector<double> k = {shells[i].c[0], shells[i].c[1], shells[i].c[2], static_cast<double>(shells[i].L)};
        k.insert(k.end(), shells[i].exps.begin(), shells[i].exps.end());
        auto it = ids.emplace(k, static_cast<int>(ids.size())).first;
        sib[i] = it->second;
      }
    }
    // compact columns for the strip kernels
    {
      std::vector<std::vector<int>> lists(kMaxL + 1);
      shell_cpos.assign(shells.size(), 0);
      for (size_t i = 0; i < shells.size(); ++i) {
        const int L = shells[i].L;
        shell_cpos[i] = static_cast<int>(lists[L].size());
        for (int f = 0; f < shells[i].nfunc(); ++f) lists[L].push_back(bf_off[i] + f);
      }
      cols_all.clear();
      for (int lc = 0; lc <= kMaxL; ++lc)
        for (int ld = 0; ld <= kMaxL; ++ld) {
          cols_off[lc][ld] = static_cast<int>(cols_all.size());
          cols_all.insert(cols_all.end(), lists[lc].begin(), lists[lc].end());
          if (ld != lc) cols_all.insert(cols_all.end(), lists[ld].begin(), lists[ld].end());
          cols_nc[lc][ld] = static_cast<int>(lists[lc].size());
          cols_n[lc][ld] = static_cast<int>(cols_all.size()) - cols_off[lc][ld];
        }
      if (!host_only) {
        d_cpos.upload(shell_cpos, stream);
        d_cols.upload(cols_all, stream);
      }
    }
    have_mol = true;
    have_pairs = have_q = have_lists = false;
    Q.clear();  // Q belongs to the previous pair store
    if (!host_only) d_scale.upload(bf_scale, stream);
  }

  // block.hpp:52-103 restated + product orientation and grouping.
  void build_pairs(double kappa_screen) {
    if (!have_mol) throw StateError("build_pairs before a molecule was loaded");
    const int S = static_cast<int>(shells.size());
    struct Tmp {
      int i, j, li, lj;
      std::vector<PrimRec> pr;
      unsigned long long sig = 1469598103934665603ull;  // FNV-1a of kept (k, l)
    };
    std::vector<Tmp> all;
    all.reserve(static_cast<size_t>(S) * (S + 1) / 2);
    const double u_const = std::sqrt(2.0) * std::pow(M_PI, 1.25);
    for (int i = 0; i < S; ++i)
      for (int j = i; j < S; ++j) {
        const ShellData& si = shells[i];
        const ShellData& sj = shells[j];
        // kappa and the screen use the reference's (i, j) orientation
        const double ABi[3] = {si.c[0] - sj.c[0], si.c[1] - sj.c[1], si.c[2] - sj.c[2]};
        const double ab2 = ABi[0] * ABi[0] + ABi[1] * ABi[1] + ABi[2] * ABi[2];
        const bool swap = sj.L > si.L;  // orient A = higher L
        const ShellData& A = swap ? sj : si;
        const ShellData& B = swap ? si : sj;
        Tmp t{i, j, si.L, sj.L, {}};
        for (int k = 0; k < si.K(); ++k)
          for (int l = 0; l < sj.K(); ++l) {
            const double alpha = si.exps[k], beta = sj.exps[l];
            const double p = alpha + beta;
            const double kappa = std::exp(-alpha * beta * ab2 / p);
            const double coef = si.coefs[k] * sj.coefs[l];
            if (kappa_screen > 0.0 && std::fabs(coef) * kappa < kappa_screen) continue;
            const double ea = swap ? beta : alpha, eb = swap ? alpha : beta;
            PrimRec r;
            r.p = p;
            r.Px = (ea * A.c[0] + eb * B.c[0]) / p;
            r.Py = (ea * A.c[1] + eb * B.c[1]) / p;
            r.Pz = (ea * A.c[2] + eb * B.c[2]) / p;
            r.PAx = r.Px - A.c[0];
            r.PAy = r.Py - A.c[1];
            r.PAz = r.Pz - A.c[2];
            r.U = u_const * kappa * coef / p;
            r.i2p = 0.5 / p;
            r.pad = 0.0;
            t.pr.push_back(r);
            t.sig = (t.sig ^ static_cast<unsigned long long>(k * 4096 + l)) * 1099511628211ull;
          }
        if (kappa_screen > 0.0 && t.pr.empty()) continue;
        all.push_back(std::move(t));
      }
    // reference order (block.hpp:94-101)
    std::vector<int> order(all.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
      const Tmp& a = all[x];
      const Tmp& b = all[y];
      return std::make_tuple(a.li + a.lj, a.li, a.lj, a.i, a.j) <
             std::make_tuple(b.li + b.lj, b.li, b.lj, b.i, b.j);
    });
    const int np = static_cast<int>(all.size());
    ref_i.resize(np);
    ref_j.resize(np);
    fam_key_ref.resize(np);
    fam_sib_ref.resize(np);
    std::vector<int> ref_of_tmp(np);
    for (int r = 0; r < np; ++r) {
      const Tmp& t = all[order[r]];
      ref_i[r] = t.i;
      ref_j[r] = t.j;
      ref_of_tmp[order[r]] = r;
      const bool sw = t.lj > t.li;
      const int A = sw ? t.j : t.i, B = sw ? t.i : t.j;
      fam_key_ref[r] = t.sig ^ (static_cast<unsigned long long>(t.pr.size()) << 48);
      fam_sib_ref[r] = sib[A] * static_cast<int>(shells.size()) + sib[B];
    }
    // product grouping: key (LA+LB, LA, LB, K), then reference index
    std::vector<int> pord(np);
    std::iota(pord.begin(), pord.end(), 0);
    auto gkey = [&](int t) {
      const Tmp& a = all[t];
      const int LA = std::max(a.li, a.lj), LB = std::min(a.li, a.lj);
      return std::make_tuple(LA + LB, LA, LB, static_cast<int>(a.pr.size()), ref_of_tmp[t]);
    };
    std::sort(pord.begin(), pord.end(), [&](int x, int y) { return gkey(x) < gkey(y); });
    pm.assign(np, PairMeta{});
    prims.clear();
    prod_of_ref.assign(np, -1);
    groups.clear();
    cls_of_pair.assign(np, 0);
    for (int g = 0; g < np; ++g) {
      const Tmp& t = all[pord[g]];
      const bool swap = t.lj > t.li;
      const int a = swap ? t.j : t.i, b = swap ? t.i : t.j;
      PairMeta m{};
      m.prim_off = static_cast<int>(prims.size());
      m.K = static_cast<int>(t.pr.size());
      m.sha = a;
      m.shb = b;
      m.bfa = bf_off[a];
      m.bfb = bf_off[b];
      m.ref = ref_of_tmp[pord[g]];
      m.ABx = shells[a].c[0] - shells[b].c[0];
      m.ABy = shells[a].c[1] - shells[b].c[1];
      m.ABz = shells[a].c[2] - shells[b].c[2];
      pm[g] = m;
      prod_of_ref[m.ref] = g;
      prims.insert(prims.end(), t.pr.begin(), t.pr.end());
      const int LA = shells[a].L, LB = shells[b].L;
      if (groups.empty() || groups.back().la != LA || groups.back().lb != LB || groups.back().K != m.K)
        groups.push_back(Group{LA, LB, m.K, g, 0});
      groups.back().count++;
    }
    if (!host_only) {
      d_pm.upload(pm, stream);
      d_prims.upload(prims, stream);
    }
    have_pairs = true;
    have_q = have_lists = false;
    Q.clear();  // Q belongs to the previous pair store
  }

  double elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
  }

  void schwarz() {
    if (!have_pairs) throw StateError("schwarz before build_pairs");
    if (host_only) throw CudaError("schwarz needs a CUDA device (host-only context)");
    const int np = static_cast<int>(pm.size());
    d_Q.alloc(np);
    std::vector<int> list;
    CK(cudaEventRecord(ev0, stream));
    for (int c = 0; c < kNumClasses; ++c) {
      const ClassEntry& ce = kClassTable[c];
      if (ce.la != ce.lc || ce.lb != ce.ld) continue;
      list.clear();
      for (const Group& g : groups)
        if (g.la == ce.la && g.lb == ce.lb)
          for (int x = g.first; x < g.first + g.count; ++x) list.push_back(x);
      if (list.empty()) continue;
      DevBuf<int> dl;
      dl.upload(list, stream);
      LaunchArgs a{};
      a.mode = 1;
      a.pair_list = dl.p;
      a.npair_list = static_cast<long long>(list.size());
      a.Qout = d_Q.p;
      a.pm = d_pm.p;
      a.prims = d_prims.p;
      a.boys_tab = d_boys.p;
      a.stream = stream;
      a.block = 128;
      ce.var[variant(c)](a);
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(stream));
    }
    CK(cudaEventRecord(ev1, stream));
    CK(cudaEventSynchronize(ev1));
    last_schwarz_ms = elapsed(ev0, ev1);
    Q.resize(np);
    d_Q.download(Q.data(), np, stream);
    have_q = true;
    have_lists = false;
  }

  void set_q_ref(const double* Qref) {
    if (!have_pairs) throw StateError("set_schwarz before build_pairs");
    Q.resize(pm.size());
    for (size_t r = 0; r < pm.size(); ++r) Q[prod_of_ref[r]] = Qref[r];
    have_q = true;
    have_lists = false;
  }

  // Sort each group by Q descending (ties: reference index), renumber.
  void sort_groups_by_q() {
    std::vector<int> perm(pm.size());
    std::iota(perm.begin(), perm.end(), 0);
    for (const Group& g : groups)
      std::sort(perm.begin() + g.first, perm.begin() + g.first + g.count, [&](int x, int y) {
        if (Q[x] != Q[y]) return Q[x] > Q[y];
        return pm[x].ref < pm[y].ref;
      });
    std::vector<PairMeta> npm(pm.size());
    std::vector<double> nQ(pm.size());
    for (size_t g = 0; g < perm.size(); ++g) {
      npm[g] = pm[perm[g]];
      nQ[g] = Q[perm[g]];
      prod_of_ref[npm[g].ref] = static_cast<int>(g);
    }
    pm.swap(npm);
    Q.swap(nQ);
    // primitive records follow the new pair order: the kets of a warp (Q-
    // consecutive pairs) then read one contiguous block of records, so L2
    // lines and DRAM pages are used whole
    std::vector<PrimRec> nprims;
    nprims.reserve(prims.size());
    for (PairMeta& m : pm) {
      const int off = static_cast<int>(nprims.size());
      nprims.insert(nprims.end(), prims.begin() + m.prim_off, prims.begin() + m.prim_off + m.K);
      m.prim_off = off;
    }
    prims.swap(nprims);
    if (!host_only) {
      d_pm.upload(pm, stream);
      d_prims.upload(prims, stream);
    }
  }

  // Group-transposed copy of the primitive records for ket reads: record j of
  // the pair at rank p of group g sits at base_g + j * count_g + p, so the 32
  // consecutive kets of a warp read 32 consecutive records (coalesced).
  void build_ket_soa() {
    kprims.assign(prims.size(), PrimRec{});
    size_t base = 0;
    for (const Group& g : groups) {
      for (int p = 0; p < g.count; ++p) {
        PairMeta& m = pm[g.first + p];
        m.ksoa = static_cast<int>(base) + p;
        m.kstride = g.count;
        for (int j = 0; j < g.K; ++j) kprims[base + static_cast<size_t>(j) * g.count + p] = prims[m.prim_off + j];
      }
      base += static_cast<size_t>(g.K) * g.count;
    }
    if (!host_only) {
      d_pm.upload(pm, stream);
      d_kprims.upload(kprims, stream);
    }
  }

  // Units of <= kFamMax product pairs with identical primitive records up to
  // U: same oriented sibling shells and the same kept primitive index set,
  // taken in Q-descending order inside each product group. Unit groups are
  // keyed (L_A+L_B, L_A, L_B, K, members) and sorted by unit Q = max member Q.
  void build_units() {
    um.clear();
    ugroups.clear();
    uQ.clear();
    std::vector<UnitMeta> tmp;
    std::vector<double> tq;
    for (const Group& g : groups) {
      std::map<std::pair<int, unsigned long long>, std::vector<int>> buckets;
      std::vector<std::pair<int, unsigned long long>> order;
      for (int x = g.first; x < g.first + g.count; ++x) {
        const int r = pm[x].ref;
        auto key = std::make_pair(fam_sib_ref[r], fam_key_ref[r]);
        auto it = buckets.find(key);
        if (it == buckets.end()) {
          order.push_back(key);
          it = buckets.emplace(key, std::vector<int>{}).first;
        }
        it->second.push_back(x);
      }
      std::vector<UnitMeta> units[kFamMax + 1];
      std::vector<double> uq[kFamMax + 1];
      for (const auto& key : order) {
        const std::vector<int>& v = buckets[key];
        for (size_t s0 = 0; s0 < v.size(); s0 += kFamMax) {
          const int nm = static_cast<int>(std::min<size_t>(kFamMax, v.size() - s0));
          UnitMeta u{};
          u.prim_off = pm[v[s0]].prim_off;
          u.K = pm[v[s0]].K;
          u.nm = nm;
          u.m0 = v[s0];
          u.m1 = nm > 1 ? v[s0 + 1] : v[s0];
          u.ABx = pm[v[s0]].ABx;
          u.ABy = pm[v[s0]].ABy;
          u.ABz = pm[v[s0]].ABz;
          units[nm].push_back(u);
          uq[nm].push_back(std::max(Q.empty() ? 0.0 : Q[u.m0], Q.empty() ? 0.0 : Q[u.m1]));
        }
      }
      for (int nm = 1; nm <= kFamMax; ++nm) {
        if (units[nm].empty()) continue;
        std::vector<int> o(units[nm].size());
        std::iota(o.begin(), o.end(), 0);
        std::stable_sort(o.begin(), o.end(), [&](int a, int b) { return uq[nm][a] > uq[nm][b]; });
        Group ug{g.la, g.lb, g.K, static_cast<int>(um.size()), static_cast<int>(o.size()), nm};
        for (int k : o) {
          um.push_back(units[nm][k]);
          uQ.push_back(uq[nm][k]);
        }
        ugroups.push_back(ug);
      }
    }
    uw.assign(prims.size(), double2{0.0, 0.0});
    for (const UnitMeta& u : um)
      for (int i = 0; i < u.K; ++i) {
        uw[u.prim_off + i].x = prims[pm[u.m0].prim_off + i].U;
        uw[u.prim_off + i].y = u.nm > 1 ? prims[pm[u.m1].prim_off + i].U : 0.0;
      }
    // unit-group-transposed copy for ket reads (as build_ket_soa)
    ukprims.assign(prims.size(), PrimRec{});
    ukw.assign(prims.size(), double2{0.0, 0.0});
    size_t base = 0;
    for (const Group& g : ugroups) {
      for (int p = 0; p < g.count; ++p) {
        UnitMeta& u = um[g.first + p];
        u.ksoa = static_cast<int>(base) + p;
        u.kstride = g.count;
        for (int j = 0; j < g.K; ++j) {
          ukprims[base + static_cast<size_t>(j) * g.count + p] = prims[u.prim_off + j];
          ukw[base + static_cast<size_t>(j) * g.count + p] = uw[u.prim_off + j];
        }
      }
      base += static_cast<size_t>(g.K) * g.count;
    }
    if (!host_only) {
      d_um.upload(um, stream);
      d_uw.upload(uw, stream);
      d_ukprims.upload(ukprims, stream);
      d_ukw.upload(ukw, stream);
      d_Qp.upload(Q.empty() ? std::vector<double>(pm.size(), 0.0) : Q, stream);
    }
  }

  // KetMeta of product pair x (both member slots) / of unit u.
  KetMeta ket_meta_pair(int x) const {
    KetMeta k{};
    for (int s = 0; s < 2; ++s) {
      k.bfa[s] = pm[x].bfa;
      k.bfb[s] = pm[x].bfb;
      k.colc[s] = shell_cpos[pm[x].sha];
      k.cold[s] = shell_cpos[pm[x].shb];
      k.offd[s] = pm[x].sha != pm[x].shb;
      k.m[s] = x;
      k.q[s] = Q.empty() ? 0.0 : Q[x];
    }
    return k;
  }
  void build_ket_meta(bool units) {
    if (host_only) return;
    std::vector<KetMeta> kp(pm.size());
    for (size_t x = 0; x < pm.size(); ++x) kp[x] = ket_meta_pair(static_cast<int>(x));
    d_kmp.upload(kp, stream);
    if (!units) return;
    std::vector<KetMeta> ku(um.size());
    for (size_t u = 0; u < um.size(); ++u) {
      const KetMeta a = ket_meta_pair(um[u].m0), b = ket_meta_pair(um[u].m1);
      ku[u] = a;
      ku[u].bfa[1] = b.bfa[1];
      ku[u].bfb[1] = b.bfb[1];
      ku[u].colc[1] = b.colc[1];
      ku[u].cold[1] = b.cold[1];
      ku[u].offd[1] = b.offd[1];
      ku[u].m[1] = b.m[1];
      ku[u].q[1] = b.q[1];
    }
    d_kmu.upload(ku, stream);
  }

  // Member quartets of unit pair (u, v) that survive (Q_m Q_n >= tau) and
  // are canonical (u == v: members m <= n only).
  int unit_pair_quartets(int u, int v, double t) const {
    const UnitMeta& a = um[u];
    const UnitMeta& b = um[v];
    int c = 0;
    for (int m = 0; m < a.nm; ++m)
      for (int n = 0; n < b.nm; ++n) {
        if (u == v && m > n) continue;
        const int x = m ? a.m1 : a.m0, y = n ? b.m1 : b.m0;
        if (t <= 0.0 || Q[x] * Q[y] >= t) ++c;
      }
    return c;
  }

  void set_screening(double t) {
    if (!have_pairs) throw StateError("set_screening before build_pairs");
    if (t > 0.0 && !have_q) schwarz();
    tau = t;
    if (t > 0.0) sort_groups_by_q();
    build_ket_soa();
    bool any_fam = false;
    for (int c = 0; c < kNumClasses; ++c) any_fam = any_fam || fam_active(c);
    if (any_fam) build_units();
    build_ket_meta(any_fam);
    // enumerate group pairs X >= Y (pair groups, or unit groups for classes
    // served by the shared-primitive kernels), grouped by angular class
    struct GP {
      int X, Y, cls;
      bool fam;
      long long cost;
      int seg = 0;  // unit classes: (nm_x - 1) * 2 + (nm_y - 1)
    };
    std::vector<GP> gps;
    for (int X = 0; X < static_cast<int>(groups.size()); ++X)
      for (int Y = 0; Y <= X; ++Y) {
        const Group& gx = groups[X];
        const Group& gy = groups[Y];
        const int cls = class_index(gx.la, gx.lb, gy.la, gy.lb);
        gps.push_back(GP{X, Y, cls, false, static_cast<long long>(gx.K) * gy.K});
      }
    if (any_fam) {
      // unit group order: (L_A+L_B, L_A, L_B, K) as the pair groups, so the
      // bra/ket roles of a quartet (X >= Y) follow the pair path's rule
      auto gkey = [](const Group& g) { return std::make_tuple(g.la + g.lb, g.la, g.lb, g.K); };
      for (int X = 0; X < static_cast<int>(ugroups.size()); ++X)
        for (int Y = 0; Y < static_cast<int>(ugroups.size()); ++Y) {
          const Group& gx = ugroups[X];
          const Group& gy = ugroups[Y];
          if (gkey(gx) < gkey(gy) || (gkey(gx) == gkey(gy) && X < Y)) continue;
          const int cls = class_index(gx.la, gx.lb, gy.la, gy.lb);
          if (!fam_active(cls)) continue;
          gps.push_back(GP{X, Y, cls, true, static_cast<long long>(gx.K) * gy.K, (gx.nm - 1) * 2 + (gy.nm - 1)});
        }
    }
    std::stable_sort(gps.begin(), gps.end(), [](const GP& a, const GP& b) {
      if (a.cls != b.cls) return a.cls < b.cls;
      if (a.fam != b.fam) return b.fam;
      if (a.seg != b.seg) return a.seg < b.seg;
      return a.cost > b.cost;
    });
    all_items.clear();
    item_q.clear();
    item_p.clear();
    items.clear();
    all_strips.clear();
    strips.clear();
    work.clear();
    cnt.clear();
    quartets = prim_quartets = 0;
    model_flops = 0.0;
    std::vector<long long> bra_tot;  // survivors per bra in the current (class, list, segment)
    for (size_t s = 0; s < gps.size();) {
      const int cls = gps[s].cls;
      const bool fam = gps[s].fam;
      ClassWork cw{};
      cw.cls = cls;
      cw.fam = fam;
      cw.aoff = static_cast<long long>(all_items.size());
      cw.astrip_off = static_cast<long long>(all_strips.size());
      const bool strip_ok = has_strip_variant(cls, fam);
      const std::vector<double>& QQ = fam ? uQ : Q;
      bra_tot.assign(fam ? um.size() : pm.size(), 0);
      for (int sg = 0; sg < 4; ++sg) {
        // the group pairs of this member segment (pair lists: segment 0 only)
        size_t e = s;
        while (e < gps.size() && gps[e].cls == cls && gps[e].fam == fam && gps[e].seg == sg) ++e;
        cw.aseg[sg] = static_cast<long long>(all_items.size()) - cw.aoff;
        cw.asseg[sg] = static_cast<long long>(all_strips.size()) - cw.astrip_off;
        // survivor counts per (group pair, bra): prefix of the Q-descending ket group
        std::vector<int> cfull(e - s);
        for (size_t g = s; g < e; ++g) {
          const Group& gx = fam ? ugroups[gps[g].X] : groups[gps[g].X];
          const Group& gy = fam ? ugroups[gps[g].Y] : groups[gps[g].Y];
          const bool same = gps[g].X == gps[g].Y;
          cfull[g - s] = static_cast<int>(cnt.size());
          for (int r = 0; r < gx.count; ++r) {
            const int x = gx.first + r;
            long long nn = gy.count;
            if (t > 0.0) {
              const double qx = QQ[x];
              int lo = 0, hi = gy.count;
              while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (qx * QQ[gy.first + mid] >= t) lo = mid + 1;
                else hi = mid;
              }
              nn = lo;
            }
            if (same) nn = std::min<long long>(nn, r + 1);
            cnt.push_back(static_cast<int>(nn));
            bra_tot[x] += nn;
          }
          cnt.push_back(0);  // sentinel
        }
        auto eligible = [&](int x) {
          return strip_ok && bra_tot[x] >= kStripMinQuartets && (fam ? um[x].K : pm[x].K) <= kStripBraMax;
        };
        auto emit = [&](int x, int cpos_, int off, int nq, int ygroup_first, const Group& gx, const Group& gy,
                        int cb, int r) {
          all_items.push_back(WorkItem{x, off | (nq << 24), cpos_, ygroup_first});
          int q = nq;
          if (fam) {  // member quartets of these nq unit pairs
            q = 0;
            int rr = r, oo = off;
            for (int l = 0; l < nq; ++l, ++oo) {
              while (oo >= cnt[cb + rr]) {
                oo -= cnt[cb + rr];
                ++rr;
              }
              q += unit_pair_quartets(gx.first + rr, gy.first + oo, t);
            }
          }
          item_q.push_back(static_cast<unsigned char>(q));
          item_p.push_back(static_cast<unsigned>(nq * gx.K * gy.K));
          cw.aquartets += q;
          cw.aprim += static_cast<long long>(nq) * gx.K * gy.K;
        };
        // 1) strips: eligible bras, single-bra items grouped by bra (runs over
        //    the segment's ket groups), cut into strips of <= kStripMaxItems
        if (strip_ok) {
          struct Run {
            int x;
            int g, r;  // group pair (relative to s), bra rank in gx
          };
          std::vector<Run> runs;
          for (size_t g = s; g < e; ++g) {
            const Group& gx = fam ? ugroups[gps[g].X] : groups[gps[g].X];
            for (int r = 0; r < gx.count; ++r)
              if (eligible(gx.first + r) && cnt[cfull[g - s] + r] > 0)
                runs.push_back(Run{gx.first + r, static_cast<int>(g - s), r});
          }
          std::stable_sort(runs.begin(), runs.end(), [](const Run& a, const Run& b) { return a.x < b.x; });
          for (size_t k = 0; k < runs.size();) {
            const int x = runs[k].x;
            Strip st{};
            st.bra = x;
            st.i0 = static_cast<int>(static_cast<long long>(all_items.size()) - cw.aoff);
            for (; k < runs.size() && runs[k].x == x; ++k) {
              const GP& gp = gps[s + runs[k].g];
              const Group& gx = fam ? ugroups[gp.X] : groups[gp.X];
              const Group& gy = fam ? ugroups[gp.Y] : groups[gp.Y];
              const int cb = cfull[runs[k].g];
              const int nn = cnt[cb + runs[k].r];
              for (int o = 0; o < nn; o += 32) {
                if (static_cast<long long>(all_items.size()) - cw.aoff - st.i0 >= kStripMaxItems) {
                  st.i1 = static_cast<int>(static_cast<long long>(all_items.size()) - cw.aoff);
                  push_strip(st, fam);
                  st.i0 = st.i1;
                }
                emit(x, cb + runs[k].r, o, std::min(32, nn - o), gy.first, gx, gy, cb, runs[k].r);
              }
            }
            st.i1 = static_cast<int>(static_cast<long long>(all_items.size()) - cw.aoff);
            if (st.i1 > st.i0) push_strip(st, fam);
          }
        }
        cw.asitem[sg] = static_cast<long long>(all_items.size()) - cw.aoff;
        // 2) the other bras: flat survivor sequence per group pair cut into
        //    warp tasks of 32 (unit) quartets that may span bras; eligible
        //    bras count 0 in this copy of the counts so the walk skips them
        for (size_t g = s; g < e; ++g) {
          const Group& gx = fam ? ugroups[gps[g].X] : groups[gps[g].X];
          const Group& gy = fam ? ugroups[gps[g].Y] : groups[gps[g].Y];
          int cb = cfull[g - s];
          long long total = 0;
          bool any_el = false;
          for (int r = 0; r < gx.count; ++r) any_el = any_el || eligible(gx.first + r);
          if (any_el) {  // counts without the strip bras
            const int cr = static_cast<int>(cnt.size());
            for (int r = 0; r < gx.count; ++r) cnt.push_back(eligible(gx.first + r) ? 0 : cnt[cb + r]);
            cnt.push_back(0);
            cb = cr;
          }
          for (int r = 0; r < gx.count; ++r) total += cnt[cb + r];
          int r = 0;
          long long off = 0;
          for (long long base = 0; base < total; base += 32) {
            while (r < gx.count && off >= cnt[cb + r]) {
              off -= cnt[cb + r];
              ++r;
            }
            emit(gx.first + r, cb + r, static_cast<int>(off), static_cast<int>(std::min<long long>(32, total - base)),
                 gy.first, gx, gy, cb, r);
            off += 32;
          }
        }
        for (size_t g = s; g < e; ++g) {  // reset the per-bra totals of this segment
          const Group& gx = fam ? ugroups[gps[g].X] : groups[gps[g].X];
          for (int r = 0; r < gx.count; ++r) bra_tot[gx.first + r] = 0;
        }
        s = e;
        if (!fam) {  // pair lists have one segment
          for (int k = sg + 1; k < 4; ++k) {
            cw.aseg[k] = static_cast<long long>(all_items.size()) - cw.aoff;
            cw.asseg[k] = static_cast<long long>(all_strips.size()) - cw.astrip_off;
            cw.asitem[k] = cw.aseg[k];
          }
          break;
        }
      }
      cw.an = static_cast<long long>(all_items.size()) - cw.aoff;
      cw.aseg[4] = cw.an;
      cw.asseg[4] = static_cast<long long>(all_strips.size()) - cw.astrip_off;
      if (std::getenv("ERITILE_DEBUG_ITEMS") && cw.an > 0) {  // diagnostics: items spanning > 1 bra
        long long multi = 0, lanes = 0, slanes = 0, sitems = 0;
        for (long long w = cw.aoff; w < cw.aoff + cw.an; ++w) {
          const WorkItem& it = all_items[w];
          if ((it.r0nq & 0xffffff) + (it.r0nq >> 24) > cnt[it.cntp]) ++multi;
          lanes += it.r0nq >> 24;
          bool in_strip = false;
          for (int sg = 0; sg < 4; ++sg)
            if (w - cw.aoff >= cw.aseg[sg] && w - cw.aoff < cw.asitem[sg]) in_strip = true;
          if (in_strip) {
            ++sitems;
            slanes += it.r0nq >> 24;
          }
        }
        std::fprintf(stderr,
                     "class %d fam %d items %lld multi-bra %.3f strips %lld strip items %lld lane fill %.3f "
                     "(strip items %.3f)\n",
                     cls, fam ? 1 : 0, cw.an, static_cast<double>(multi) / cw.an, cw.asseg[4], sitems,
                     lanes / (32.0 * cw.an), sitems ? slanes / (32.0 * sitems) : 0.0);
      }
      if (cw.an > 0) {
        const ClassEntry& ce = kClassTable[cls];
        const double nv = static_cast<double>((ce.la + 1) * (ce.la + 2) / 2 * (ce.lb + 1) * (ce.lb + 2) / 2 *
                                              (ce.lc + 1) * (ce.lc + 2) / 2 * (ce.ld + 1) * (ce.ld + 2) / 2);
        // F_c = Nprim (42 + 3m + 2(P+B+X)) + Nq (2H + 12 n), with
        // P, B, X, H from the plan this kernel executes; Nprim counts the
        // primitive quartets actually evaluated (once per unit pair).
        cw.cost_prim = 42.0 + 3.0 * ce.max_m + 2.0 * (ce.prim_terms + ce.base + ce.contract);
        cw.cost_q = 2.0 * ce.hrr_terms + 12.0 * nv;
        // heaviest strips first within each segment: the strip kernels hand
        // strips out dynamically in this order (greedy LPT over the CTAs)
        for (int sg = 0; sg < 4; ++sg) {
          const long long b = cw.astrip_off + cw.asseg[sg], e = cw.astrip_off + cw.asseg[sg + 1];
          if (e - b < 2) continue;
          std::vector<std::pair<double, Strip>> ws;
          ws.reserve(static_cast<size_t>(e - b));
          for (long long k = b; k < e; ++k) {
            const Strip& st = all_strips[k];
            double wt = 0.0;
            for (long long i = cw.aoff + st.i0; i < cw.aoff + st.i1; ++i)
              wt += cw.cost_prim * item_p[i] + cw.cost_q * item_q[i];
            ws.emplace_back(wt, st);
          }
          std::stable_sort(ws.begin(), ws.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
          for (long long k = b; k < e; ++k) all_strips[k] = ws[k - b].second;
        }
        work.push_back(cw);
      } else {
        all_strips.resize(cw.astrip_off);
      }
    }
    if (!host_only) {
      d_cnt.upload(cnt, stream);
      d_all_items.upload(all_items, stream);
      d_all_strips.upload(all_strips, stream);
      d_sctr.alloc(4 * work.size());
    }
    have_lists = true;
    dealt = false;
    deal();
  }

  // Strip geometry: row blocks = the distinct shells of the bra members.
  long long kStripMinQuartets = 1024;  // bras with fewer survivors stay packed
  long long kStripMaxItems = 1024;     // items per strip (granularity / load balance)
  void push_strip(Strip st, bool fam) {
    int mem[2], nm = 1;
    if (fam) {
      mem[0] = um[st.bra].m0;
      mem[1] = um[st.bra].m1;
      nm = um[st.bra].nm;
    } else {
      mem[0] = st.bra;
    }
    int nb = 0, row = 0;
    int shl[4];
    auto row_of = [&](int sh) {
      for (int k = 0; k < nb; ++k)
        if (shl[k] == sh) {
          int r = 0;
          for (int q = 0; q < k; ++q) r += st.rb_n[q];
          return r;
        }
      shl[nb] = sh;
      st.rb_bf[nb] = bf_off[sh];
      st.rb_n[nb] = shells[sh].nfunc();
      const int r = row;
      row += st.rb_n[nb];
      ++nb;
      return r;
    };
    for (int m = 0; m < nm; ++m) {
      st.rowA[m] = row_of(pm[mem[m]].sha);
      st.rowB[m] = row_of(pm[mem[m]].shb);
    }
    for (int k = nb; k < 4; ++k) {
      st.rb_bf[k] = 0;
      st.rb_n[k] = 0;
    }
    st.nrows = row;
    all_strips.push_back(st);
  }
  bool has_strip_variant(int c, bool fam) const {
    const ClassEntry& ce = kClassTable[c];
    for (int v = 0; v < ce.nvar; ++v)
      if (std::strncmp(ce.var_name[v], fam ? "fstrip" : "strip", fam ? 6 : 5) == 0) return true;
    return false;
  }

  // Quartet-block sharding (quartets are independent,
  // block.hpp:40-42): the active list of every class is cut into chunks of
  // kDealChunk warp tasks (never across a unit member segment), each weighted
  // by its model FLOPs (SURVEY 8d F_c: primitive and contracted quartets of
  // its items), and the chunks are dealt by LPT - heaviest first, each to the
  // least-loaded rank, ties to the lower rank and the lower chunk index. The
  // deal depends only on the lists and the variant table, so every rank
  // computes the same one and the shards are a disjoint cover of the
  // canonical list, PROVIDED all ranks use the same variant table
  // (variant_signature; bench.py broadcasts rank 0's tuned table). A rank's
  // items of a class keep chunk order (Q-sorted locality).
  static constexpr long long kDealChunk = 64;
  void deal() {
    if (!have_lists) return;
    if (nranks == 1) {
      for (ClassWork& cw : work) {
        cw.off = cw.aoff;
        cw.n = cw.an;
        for (int k = 0; k < 5; ++k) cw.seg[k] = cw.aseg[k];
        for (int k = 0; k < 5; ++k) cw.sseg[k] = cw.asseg[k];
        for (int k = 0; k < 4; ++k) cw.sitem[k] = cw.asitem[k];
        cw.strip_off = cw.astrip_off;
        cw.quartets = cw.aquartets;
        cw.prim_quartets = cw.aprim;
        cw.flops = cw.full_flops();
      }
      items.clear();
      strips.clear();
      update_totals();
      dealt = true;
      return;
    }
    // chunks: every strip whole (its K rows are flushed per strip), then the
    // packed items of each segment in runs of kDealChunk
    struct Chunk {
      long long b, e;  // all_items range
      long long strip; // all_strips index, -1 for packed items
      int sg;
      double w;
      int owner;
    };
    std::vector<Chunk> ch;
    std::vector<std::pair<size_t, size_t>> wch(work.size(), {0, 0});  // chunk range per work entry
    for (size_t w = 0; w < work.size(); ++w) {
      const ClassWork& cw = work[w];
      wch[w].first = ch.size();
      auto weight = [&](long long b, long long e) {
        double wt = 0.0;
        for (long long i = b; i < e; ++i) wt += cw.cost_prim * item_p[i] + cw.cost_q * item_q[i];
        return wt;
      };
      if (active(cw)) {
        for (int sg = 0; sg < 4; ++sg) {
          for (long long k = cw.asseg[sg]; k < cw.asseg[sg + 1]; ++k) {
            const Strip& st = all_strips[cw.astrip_off + k];
            const long long b = cw.aoff + st.i0, e = cw.aoff + st.i1;
            ch.push_back(Chunk{b, e, cw.astrip_off + k, sg, weight(b, e), 0});
          }
          const long long s0 = cw.aoff + cw.asitem[sg], s1 = cw.aoff + cw.aseg[sg + 1];
          for (long long b = s0; b < s1; b += kDealChunk) {
            const long long e = std::min(s1, b + kDealChunk);
            ch.push_back(Chunk{b, e, -1, sg, weight(b, e), 0});
          }
        }
      }
      wch[w].second = ch.size();
    }
    std::vector<size_t> ord(ch.size());
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return ch[a].w > ch[b].w; });
    std::vector<double> load(nranks, 0.0);
    for (size_t k : ord) {
      int r = 0;
      for (int q = 1; q < nranks; ++q)
        if (load[q] < load[r]) r = q;
      ch[k].owner = r;
      load[r] += ch[k].w;
    }
    items.clear();
    strips.clear();
    for (size_t w = 0; w < work.size(); ++w) {
      ClassWork& cw = work[w];
      cw.off = static_cast<long long>(items.size());
      cw.strip_off = static_cast<long long>(strips.size());
      cw.quartets = cw.prim_quartets = 0;
      for (int k = 0; k < 5; ++k) cw.seg[k] = cw.sseg[k] = 0;
      for (int k = 0; k < 4; ++k) cw.sitem[k] = 0;
      size_t k = wch[w].first;
      for (int sg = 0; sg < 4; ++sg) {
        cw.seg[sg] = static_cast<long long>(items.size()) - cw.off;
        cw.sseg[sg] = static_cast<long long>(strips.size()) - cw.strip_off;
        bool rest = false;
        for (; k < wch[w].second && ch[k].sg == sg; ++k) {
          const Chunk& c = ch[k];
          if (c.strip < 0 && !rest) {
            cw.sitem[sg] = static_cast<long long>(items.size()) - cw.off;
            rest = true;
          }
          if (c.owner != rank) continue;
          if (c.strip >= 0) {
            Strip st = all_strips[c.strip];
            st.i0 = static_cast<int>(static_cast<long long>(items.size()) - cw.off);
            st.i1 = st.i0 + static_cast<int>(c.e - c.b);
            strips.push_back(st);
          }
          for (long long i = c.b; i < c.e; ++i) {
            items.push_back(all_items[i]);
            cw.quartets += item_q[i];
            cw.prim_quartets += item_p[i];
          }
        }
        if (!rest) cw.sitem[sg] = static_cast<long long>(items.size()) - cw.off;
      }
      cw.n = static_cast<long long>(items.size()) - cw.off;
      cw.seg[4] = cw.n;
      cw.sseg[4] = static_cast<long long>(strips.size()) - cw.strip_off;
      cw.flops = cw.cost_prim * static_cast<double>(cw.prim_quartets) + cw.cost_q * static_cast<double>(cw.quartets);
    }
    if (!host_only) {
      d_items.upload(items, stream);
      d_strips.upload(strips, stream);
    }
    update_totals();
    dealt = true;
  }
  void ensure_dealt() {
    if (have_lists && !dealt) deal();
  }

  void ensure_mats() {
    const size_t NN = static_cast<size_t>(nbf) * nbf;
    d_Ds.alloc(NN);
    d_JK.alloc(2 * NN);
  }

  // Launch errors name the class and kernel variant that raised them.
  void check_launch(const ClassWork& cw) {
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return;
    const ClassEntry& ce = kClassTable[cw.cls];
    throw CudaError("launch of class (" + std::to_string(ce.la) + std::to_string(ce.lb) + std::to_string(ce.lc) +
                    std::to_string(ce.ld) + ") variant " + ce.var_name[variant(cw.cls)] + ": " +
                    cudaGetErrorString(e));
  }

  // Launch every class over D' (pre-scaled, device) into JKacc (zeroed).
  void launch_all(const double* dDs, double* dJK, cudaStream_t st) {
    const size_t NN = static_cast<size_t>(nbf) * nbf;
    CK(cudaMemsetAsync(dJK, 0, sizeof(double) * 2 * NN, st));
    launches_last = 0;  // kernel launches of this build (the memset is not one)
    if (profiling && prof_ev.size() < 2 * work.size()) {
      while (prof_ev.size() < 2 * work.size()) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        prof_ev.push_back(e);
      }
    }
    if (profiling || !concurrent) {  // one stream: per-class events are exact
      for (size_t w = 0; w < work.size(); ++w) {
        const ClassWork& cw = work[w];
        if (!active(cw)) continue;
        if (profiling) CK(cudaEventRecord(prof_ev[2 * w], st));
        LaunchArgs a = class_args(cw, dDs, dJK, st);
        kClassTable[cw.cls].var[variant(cw.cls)](a);
        check_launch(cw);
        launches_last += kernel_launches(cw);
        if (profiling) CK(cudaEventRecord(prof_ev[2 * w + 1], st));
      }
      return;
    }
    // Class launches are independent (commutative FP64 reductions into J/K):
    // heaviest first, dealt over kSide+1 streams so each launch's last wave
    // overlaps the next launch instead of idling SMs. Forked from / joined
    // back to `st` with events.
    if (side[0] == nullptr) {
      for (int k = 0; k < kSide; ++k) {
        CK(cudaStreamCreateWithFlags(&side[k], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&side_ev[k], cudaEventDisableTiming));
      }
      CK(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
    }
    std::vector<int> act = active_work();
    std::stable_sort(act.begin(), act.end(), [&](int a, int b) { return work[a].flops > work[b].flops; });
    CK(cudaEventRecord(fork_ev, st));
    for (int k = 0; k < kSide; ++k) CK(cudaStreamWaitEvent(side[k], fork_ev, 0));
    for (size_t i = 0; i < act.size(); ++i) {
      const ClassWork& cw = work[act[i]];
      cudaStream_t s = (i % (kSide + 1) == 0) ? st : side[i % (kSide + 1) - 1];
      LaunchArgs a = class_args(cw, dDs, dJK, s);
      kClassTable[cw.cls].var[variant(cw.cls)](a);
      check_launch(cw);
      launches_last += kernel_launches(cw);
    }
    for (int k = 0; k < kSide; ++k) {
      CK(cudaEventRecord(side_ev[k], side[k]));
      CK(cudaStreamWaitEvent(st, side_ev[k], 0));
    }
  }

  // Per-class device times of the last launch_all (profiling mode).
  void collect_profile() {
    if (!profiling) return;
    CK(cudaStreamSynchronize(stream));
    for (int w : active_work()) CK(cudaEventSynchronize(prof_ev[2 * w + 1]));
    for (int w : active_work()) work[w].last_ms = elapsed(prof_ev[2 * w], prof_ev[2 * w + 1]);
  }

  void prescale(const double* dD, double* dDs, cudaStream_t st) {
    const size_t NN = static_cast<size_t>(nbf) * nbf;
    const int grid = static_cast<int>(std::min<size_t>((NN + 255) / 256, 148 * 32));
    k_prescale<<<std::max(grid, 1), 256, 0, st>>>(dD, d_scale.p, dDs, nbf);
    CK(cudaGetLastError());
  }

  void finalize(const double* dJK, double* dJ, double* dK, cudaStream_t st) {
    const size_t NN = static_cast<size_t>(nbf) * nbf;
    const int grid = static_cast<int>(std::min<size_t>((NN + 255) / 256, 148 * 32));
    k_finalize<<<std::max(grid, 1), 256, 0, st>>>(dJK, dJK + NN, d_scale.p, dJ, dK, nbf, det ? 1 : 0);
    CK(cudaGetLastError());
  }

  // Per reference pair x: count and splitmix64 sum of y over this rank's
  // canonical quartets (x, y), x <= y (eritile_gpu_pair_survivors).
  long long pair_survivors(long long* count, unsigned long long* ysum) const {
    const size_t np = pm.size();
    std::vector<std::pair<const ClassWork*, long long>> jobs;  // (class list, first local item)
    for (const ClassWork& cw : work)
      if (active(cw))
        for (long long b = 0; b < cw.n; b += 4096) jobs.emplace_back(&cw, b);
    const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::vector<long long>> tc(nt, std::vector<long long>(np, 0));
    std::vector<std::vector<unsigned long long>> th(nt, std::vector<unsigned long long>(np, 0));
    std::atomic<size_t> next{0};
    auto mix = [](unsigned long long z) {
      z += 0x9e3779b97f4a7c15ull;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
      return z ^ (z >> 31);
    };
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        for (size_t j; (j = next.fetch_add(1)) < jobs.size();) {
          const ClassWork& cw = *jobs[j].first;
          const long long e = std::min(cw.n, jobs[j].second + 4096);
          auto add = [&](int px, int py) {
            const int rx = pm[px].ref, ry = pm[py].ref;
            const int lo = std::min(rx, ry), hi = std::max(rx, ry);
            ++tc[t][lo];
            th[t][lo] += mix(static_cast<unsigned long long>(hi));
          };
          for (long long k = jobs[j].second; k < e; ++k) {
            const WorkItem& it = local_item(cw, k);
            const int nq = it.r0nq >> 24;
            int q = it.r0nq & 0xffffff, x = it.bra0, c = it.cntp;
            for (int l = 0; l < nq; ++l, ++q) {
              while (q >= cnt[c]) {
                q -= cnt[c];
                ++x;
                ++c;
              }
              const int y = it.yfirst + q;
              if (!cw.fam) {
                add(x, y);
                continue;
              }
              const UnitMeta& a = um[x];
              const UnitMeta& b = um[y];
              for (int m = 0; m < a.nm; ++m)
                for (int n = 0; n < b.nm; ++n) {
                  if (x == y && m > n) continue;
                  const int px = m ? a.m1 : a.m0, py = n ? b.m1 : b.m0;
                  if (tau > 0.0 && Q[px] * Q[py] < tau) continue;
                  add(px, py);
                }
            }
          }
        }
      });
    for (auto& t : pool) t.join();
    long long total = 0;
    for (size_t x = 0; x < np; ++x) {
      long long cx = 0;
      unsigned long long hx = 0;
      for (unsigned t = 0; t < nt; ++t) {
        cx += tc[t][x];
        hx += th[t][x];
      }
      count[x] = cx;
      ysum[x] = hx;
      total += cx;
    }
    return total;
  }

  void check_ready() {
    if (host_only) throw CudaError("build_jk needs a CUDA device (host-only context)");
    if (!have_lists) throw StateError("build_jk before set_screening");
    ensure_dealt();
  }
  // item k of this rank's share of class list cw
  const WorkItem& local_item(const ClassWork& cw, long long k) const {
    return nranks == 1 ? all_items[cw.aoff + k] : items[cw.off + k];
  }
};

// -------------------------------------------------------------- C ABI
namespace {
int fail(eritile_gpu* c, int code, const std::string& m) {
  if (c) c->err = m;
  return code;
}
template <class F>
int guard(eritile_gpu* c, F&& f) {
  try {
    if (c && !c->host_only) CK(cudaSetDevice(c->device));
    f();
    return ERITILE_OK;
  } catch (const InputError& e) {
    return fail(c, ERITILE_ERR_PARSE, e.what());
  } catch (const CudaError& e) {
    return fail(c, ERITILE_ERR_CUDA, e.what());
  } catch (const StateError& e) {
    return fail(c, ERITILE_ERR_STATE, e.what());
  } catch (const ArgError& e) {
    return fail(c, ERITILE_ERR_ARG, e.what());
  } catch (const std::exception& e) {
    return fail(c, ERITILE_ERR_ARG, e.what());
  }
}
thread_local std::string g_create_err;
}  // namespace

extern "C" {

int eritile_gpu_create(int device, eritile_gpu** out) {
  if (!out) return ERITILE_ERR_ARG;
  *out = nullptr;
  if (device < 0) {  // host-only context: input, pairs, screening lists; no kernels
    auto c = std::make_unique<eritile_gpu>();
    c->device = -1;
    c->host_only = true;
    *out = c.release();
    return ERITILE_OK;
  }
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    g_create_err = "no CUDA device (eritile_gpu has no CPU fallback)";
    return ERITILE_ERR_CUDA;
  }
  if (device < 0 || device >= n) {
    g_create_err = "device index out of range";
    return ERITILE_ERR_ARG;
  }
  auto c = std::make_unique<eritile_gpu>();
  c->device = device;
  int rc = guard(c.get(), [&] {
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    c->d_boys.upload(make_boys_table(), c->stream);
  });
  if (rc != ERITILE_OK) {
    g_create_err = c->err;
    return rc;
  }
  *out = c.release();
  return ERITILE_OK;
}

void eritile_gpu_destroy(eritile_gpu* ctx) { delete ctx; }

const char* eritile_gpu_last_error(const eritile_gpu* ctx) {
  return ctx ? ctx->err.c_str() : g_create_err.c_str();
}

int eritile_gpu_load_molecule(eritile_gpu* ctx, const char* xyz_text, const char* basis_text) {
  if (!ctx || !xyz_text || !basis_text) return ERITILE_ERR_ARG;
  return guard(ctx, [&] {
    auto atoms = read_xyz(xyz_text);
    auto tab = read_basis(basis_text);
    auto sh = attach_basis(atoms, tab);
    ctx->set_molecule(std::move(atoms), std::move(sh));
  });
}

int eritile_gpu_load_shells(eritile_gpu* ctx, int nshell, const int* L, const int* K, const double* center,
                            const int* atom, const double* exps, const double* coefs, int natoms,
                            const int* Z, const double* pos) {
  if (!ctx || nshell <= 0 || !L || !K || !center || !exps || !coefs) return ERITILE_ERR_ARG;
  return guard(ctx, [&] {
    std::vector<ShellData> sh(nshell);
    size_t o = 0;
    for (int s = 0; s < nshell; ++s) {
      if (K[s] < 1 || L[s] < 0) throw ArgError("invalid shell");
      sh[s].L = L[s];
      sh[s].atom = atom ? atom[s] : -1;
      for (int d = 0; d < 3; ++d) sh[s].c[d] = center[3 * s + d];
      sh[s].exps.assign(exps + o, exps + o + K[s]);
      sh[s].coefs.assign(coefs + o, coefs + o + K[s]);
      o += K[s];
    }
    std::vector<Atom> at(natoms > 0 ? natoms : 0);
    for (int a = 0; a < natoms; ++a) {
      at[a].Z = Z[a];
      for (int d = 0; d < 3; ++d) at[a].r[d] = pos[3 * a + d];
    }
    ctx->set_molecule(std::move(at), std::move(sh));
  });
}

int eritile_gpu_nbf(const eritile_gpu* ctx) { return ctx ? ctx->nbf : 0; }
int eritile_gpu_shell_info(const eritile_gpu* ctx, int* L, int* K, int* bf_off) {
  if (!ctx || !L || !K || !bf_off) return ERITILE_ERR_ARG;
  for (size_t s = 0; s < ctx->shells.size(); ++s) {
    L[s] = ctx->shells[s].L;
    K[s] = ctx->shells[s].K();
    bf_off[s] = ctx->bf_off[s];
  }
  return ERITILE_OK;
}
int eritile_gpu_nshells(const eritile_gpu* ctx) { return ctx ? static_cast<int>(ctx->shells.size()) : 0; }
int eritile_gpu_nelectrons(const eritile_gpu* ctx) {
  int n = 0;
  if (ctx)
    for (const Atom& a : ctx->atoms) n += a.Z;
  return n;
}
double eritile_gpu_nuclear_repulsion(const eritile_gpu* ctx) {
  double e = 0.0;
  if (!ctx) return e;
  for (size_t a = 0; a < ctx->atoms.size(); ++a)
    for (size_t b = a + 1; b < ctx->atoms.size(); ++b) {
      double d2 = 0.0;
      for (int k = 0; k < 3; ++k) {
        const double d = ctx->atoms[a].r[k] - ctx->atoms[b].r[k];
        d2 += d * d;
      }
      e += static_cast<double>(ctx->atoms[a].Z) * ctx->atoms[b].Z / std::sqrt(d2);
    }
  return e;
}

int eritile_gpu_build_pairs(eritile_gpu* ctx, double kappa_screen) {
  if (!ctx) return ERITILE_ERR_ARG;
  return guard(ctx, [&] { ctx->build_pairs(kappa_screen); });
}
int eritile_gpu_npairs(const eritile_gpu* ctx) { return ctx ? static_cast<int>(ctx->pm.size()) : 0; }
int eritile_gpu_pair_shells(const eritile_gpu* ctx, int* i, int* j) {
  if (!ctx || !i || !j) return ERITILE_ERR_ARG;
  std::copy(ctx->ref_i.begin(), ctx->ref_i.end(), i);
  std::copy(ctx->ref_j.begin(), ctx->ref_j.end(), j);
  return ERITILE_OK;
}

int eritile_gpu_schwarz(eritile_gpu* ctx, double* Qref) {
  if (!ctx) return ERITILE_ERR_ARG;
  return guard(ctx, [&] {
    if (!ctx->have_q) ctx->schwarz();
    if (Qref)
      for (size_t r = 0; r < ctx->pm.size(); ++r) Qref[r] = ctx->Q[ctx->prod_of_ref[r]];
  });
}
int eritile_gpu_set_schwarz(eritile_gpu* ctx, const double* Q) {
  if (!ctx || !Q) return ERITILE_ERR_ARG;
  return guard(ctx, [&] { ctx->set_q_ref(Q); });
}

int eritile_gpu_set_shard(eritile_gpu* ctx, int rank, int nranks) {
  if (!ctx || nranks < 1 || rank < 0 || rank >= nranks) return fail(ctx, ERITILE_ERR_ARG, "bad shard");
  ctx->rank = rank;
  ctx->nranks = nranks;
  ctx->dealt = false;  // re-dealt before the next build / list export
  return ERITILE_OK;
}

int eritile_gpu_set_screening(eritile_gpu* ctx, double tau) {
  if (!ctx) return ERITILE_ERR_ARG;
  return guard(ctx, [&] { ctx->set_screening(tau); });
}

long long eritile_gpu_num_quartets(const eritile_gpu* ctx) {
  if (!ctx) return -1;
  if (guard(const_cast<eritile_gpu*>(ctx), [&] { const_cast<eritile_gpu*>(ctx)->ensure_dealt(); }) != ERITILE_OK)
    return -1;
  return ctx->quartets;
}

long long eritile_gpu_quartets(const eritile_gpu* ctx, int* xs, int* ys, long long cap) {
  if (!ctx || !ctx->have_lists) return -1;
  if (guard(const_cast<eritile_gpu*>(ctx), [&] { const_cast<eritile_gpu*>(ctx)->ensure_dealt(); }) != ERITILE_OK)
    return -1;
  std::vector<std::pair<int, int>> q;
  q.reserve(static_cast<size_t>(ctx->quartets));
  for (const ClassWork& cw : ctx->work)
    for (long long w = 0; w < (ctx->active(cw) ? cw.n : 0); ++w) {
      const WorkItem& it = ctx->local_item(cw, w);
      const int nq = it.r0nq >> 24;
      for (int l = 0; l < nq; ++l) {
        int qq = (it.r0nq & 0xffffff) + l, x = it.bra0, c = it.cntp;
        while (qq >= ctx->cnt[c]) {
          qq -= ctx->cnt[c];
          ++x;
          ++c;
        }
        const int y = it.yfirst + qq;
        if (!cw.fam) {
          const int rx = ctx->pm[x].ref, ry = ctx->pm[y].ref;
          q.emplace_back(std::min(rx, ry), std::max(rx, ry));
          continue;
        }
        const UnitMeta& a = ctx->um[x];
        const UnitMeta& b = ctx->um[y];
        for (int m = 0; m < a.nm; ++m)
          for (int n = 0; n < b.nm; ++n) {
            if (x == y && m > n) continue;
            const int px = m ? a.m1 : a.m0, py = n ? b.m1 : b.m0;
            if (ctx->tau > 0.0 && ctx->Q[px] * ctx->Q[py] < ctx->tau) continue;
            const int rx = ctx->pm[px].ref, ry = ctx->pm[py].ref;
            q.emplace_back(std::min(rx, ry), std::max(rx, ry));
          }
      }
    }
  std::sort(q.begin(), q.end());
  const long long n = static_cast<long long>(q.size());
  if (xs && ys)
    for (long long k = 0; k < std::min(n, cap); ++k) {
      xs[k] = q[k].first;
      ys[k] = q[k].second;
    }
  return n;
}

int eritile_gpu_build_jk_partial_device(eritile_gpu* ctx, const double* dD, double* dJKacc, void* stream) {
  if (!ctx || !dD || !dJKacc) return ERITILE_ERR_ARG;
  return guard(ctx, [&] {
    ctx->check_ready();
    ctx->ensure_mats();
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    ctx->prescale(dD, ctx->d_Ds.p, st);
    ctx->launch_all(ctx->d_Ds.p, dJKacc, st);
    ctx->launches_last += 1;
  });
}

int eritile_gpu_finalize_device(eritile_gpu* ctx, const double* dJKacc, double* dJ, double* dK, void* stream) {
  if (!ctx || !dJKacc || !dJ || !dK) return ERITILE_ERR_ARG;
  return guard(ctx, [&] {
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    ctx->finalize(dJKacc, dJ, dK, st);
  });
}

int eritile_gpu_build_jk_device(eritile_gpu* ctx, const double* dD, double* dJ, double* dK, void* stream) {
  if (!ctx || !dD || !dJ || !dK) return ERITILE_ERR_ARG;
  return guard(ctx, [&] {
    ctx->check_ready();
    ctx->ensure_mats();
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    CK(cudaEventRecord(ctx->ev0, st));
    ctx->prescale(dD, ctx->d_Ds.p, st);
    ctx->launch_all(ctx->d_Ds.p, ctx->d_JK.p, st);
    ctx->finalize(ctx->d_JK.p, dJ, dK, st);
    ctx->launches_last += 2;
    CK(cudaEventRecord(ctx->ev1, st));
  });
}

int eritile_gpu_build_jk(eritile_gpu* ctx, const double* D, double* J, double* K) {
  if (!ctx || !D || !J || !K) return ERITILE_ERR_ARG;
  return guard(ctx, [&] {
    ctx->check_ready();
    ctx->ensure_mats();
    const size_t NN = static_cast<size_t>(ctx->nbf) * ctx->nbf;
    ctx->d_D.alloc(NN);
    ctx->d_J.alloc(NN);
    ctx->d_K.alloc(NN);
    cudaStream_t st = ctx->stream;
    CK(cudaMemcpyAsync(ctx->d_D.p, D, sizeof(double) * NN, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(ctx->ev0, st));
    ctx->prescale(ctx->d_D.p, ctx->d_Ds.p, st);
    ctx->launch_all(ctx->d_Ds.p, ctx->d_JK.p, st);
    ctx->finalize(ctx->d_JK.p, ctx->d_J.p, ctx->d_K.p, st);
    ctx->launches_last += 2;
    CK(cudaEventRecord(ctx->ev1, st));
    CK(cudaMemcpyAsync(J, ctx->d_J.p, sizeof(double) * NN, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(K, ctx->d_K.p, sizeof(double) * NN, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ctx->last_build_ms = ctx->elapsed(ctx->ev0, ctx->ev1);
  });
}

int eritile_gpu_one_electron(eritile_gpu* ctx, double* S, double* T, double* V) {
  if (!ctx || !S || !T || !V) return ERITILE_ERR_ARG;
  return guard(ctx, [&] {
    if (!ctx->have_mol) throw StateError("one_electron before a molecule was loaded");
    one_electron(ctx->shells, ctx->atoms, ctx->bf_off, ctx->bf_scale, S, T, V);
  });
}

int eritile_gpu_boys(eritile_gpu* ctx, int m_max, const double* T, int n, double* F) {
  if (!ctx || !T || !F || n < 0) return ERITILE_ERR_ARG;
  if (m_max < 0 || m_max > kBoysMmax) return fail(ctx, ERITILE_ERR_DOMAIN, "boys: order out of range");
  for (int i = 0; i < n; ++i)
    if (!(T[i] >= 0.0) || !std::isfinite(T[i]))
      return fail(ctx, ERITILE_ERR_DOMAIN, "boys: argument must be finite and non-negative");
  return guard(ctx, [&] {
    DevBuf<double> dT, dF;
    dT.upload(std::vector<double>(T, T + n), ctx->stream);
    dF.alloc(static_cast<size_t>(n) * (m_max + 1) + 1);
    k_boys<<<(n + 127) / 128 + 1, 128, 0, ctx->stream>>>(m_max, dT.p, n, ctx->d_boys.p, dF.p);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    dF.download(F, static_cast<size_t>(n) * (m_max + 1), ctx->stream);
  });
}

int eritile_gpu_eri_quartet(eritile_gpu* ctx, int x, int y, double* out) {
  if (!ctx || !out) return ERITILE_ERR_ARG;
  return guard(ctx, [&] {
    if (!ctx->have_pairs) throw StateError("eri_quartet before build_pairs");
    const int np = static_cast<int>(ctx->pm.size());
    if (x < 0 || y < 0 || x >= np || y >= np) throw ArgError("eri_quartet: pair index out of range");
    const int px = ctx->prod_of_ref[x], py = ctx->prod_of_ref[y];
    auto key = [&](int p) {
      const PairMeta& m = ctx->pm[p];
      const int LA = ctx->shells[m.sha].L, LB = ctx->shells[m.shb].L;
      return std::make_tuple(LA + LB, LA, LB);
    };
    const bool bk_swap = key(px) < key(py);
    const int pb = bk_swap ? py : px, pk = bk_swap ? px : py;
    const PairMeta& mb = ctx->pm[pb];
    const PairMeta& mk = ctx->pm[pk];
    const int slot_sh[4] = {mb.sha, mb.shb, mk.sha, mk.shb};
    const int L[4] = {ctx->shells[slot_sh[0]].L, ctx->shells[slot_sh[1]].L, ctx->shells[slot_sh[2]].L,
                      ctx->shells[slot_sh[3]].L};
    const int cls = ctx->class_index(L[0], L[1], L[2], L[3]);
    int nslot[4];
    for (int s = 0; s < 4; ++s) nslot[s] = (L[s] + 1) * (L[s] + 2) / 2;
    const int nv = nslot[0] * nslot[1] * nslot[2] * nslot[3];
    DevBuf<int> dq;
    dq.upload(std::vector<int>{pb, pk}, ctx->stream);
    DevBuf<double> dv;
    dv.alloc(nv);
    LaunchArgs a{};
    a.mode = 2;
    a.qpairs = dq.p;
    a.nq = 1;
    a.qout = dv.p;
    a.pm = ctx->d_pm.p;
    a.prims = ctx->d_prims.p;
    a.boys_tab = ctx->d_boys.p;
    a.stream = ctx->stream;
    a.block = 128;
    kClassTable[cls].var[ctx->variant(cls)](a);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    std::vector<double> v(nv);
    dv.download(v.data(), nv, ctx->stream);
    // reference positions (i, j | k, l) -> kernel slots
    const int R[4] = {ctx->ref_i[x], ctx->ref_j[x], ctx->ref_i[y], ctx->ref_j[y]};
    int slot_of[4];
    const int bx = bk_swap ? 2 : 0, by = bk_swap ? 0 : 2;  // kernel slot base of x and y
    slot_of[0] = (slot_sh[bx] == R[0]) ? bx : bx + 1;
    slot_of[1] = (slot_of[0] == bx) ? bx + 1 : bx;
    slot_of[2] = (slot_sh[by] == R[2]) ? by : by + 1;
    slot_of[3] = (slot_of[2] == by) ? by + 1 : by;
    std::vector<std::array<int, 3>> comps[4];
    std::vector<double> sc[4];
    int nr[4];
    for (int r = 0; r < 4; ++r) {
      const int Lr = ctx->shells[R[r]].L;
      cart_components(Lr, comps[r]);
      nr[r] = static_cast<int>(comps[r].size());
      for (auto& c : comps[r]) sc[r].push_back(component_scale(c[0], c[1], c[2]));
    }
    int stride[4] = {nslot[1] * nslot[2] * nslot[3], nslot[2] * nslot[3], nslot[3], 1};
    size_t o = 0;
    int idx[4];
    for (idx[0] = 0; idx[0] < nr[0]; ++idx[0])
      for (idx[1] = 0; idx[1] < nr[1]; ++idx[1])
        for (idx[2] = 0; idx[2] < nr[2]; ++idx[2])
          for (idx[3] = 0; idx[3] < nr[3]; ++idx[3], ++o) {
            int k = 0;
            for (int r = 0; r < 4; ++r) k += idx[r] * stride[slot_of[r]];
            out[o] = v[k] * (sc[0][idx[0]] * sc[1][idx[1]] * sc[2][idx[2]] * sc[3][idx[3]]);
          }
  });
}

int eritile_gpu_set_profiling(eritile_gpu* ctx, int on) {
  if (!ctx) return ERITILE_ERR_ARG;
  ctx->profiling = on != 0;
  return ERITILE_OK;
}

int eritile_gpu_class_profile(eritile_gpu* ctx, int cap, int* cls4, double* ms, double* flops,
                              long long* quartets, long long* prim_quartets) {
  if (!ctx) return ERITILE_ERR_ARG;
  int rc = guard(ctx, [&] {
    ctx->ensure_dealt();
    ctx->collect_profile();
  });
  if (rc != ERITILE_OK) return rc;
  const std::vector<int> act = ctx->active_work();
  const int n = static_cast<int>(act.size());
  for (int k = 0; k < std::min(n, cap); ++k) {
    const ClassWork& cw = ctx->work[act[k]];
    const ClassEntry& ce = kClassTable[cw.cls];
    if (cls4) {
      cls4[4 * k] = ce.la; cls4[4 * k + 1] = ce.lb; cls4[4 * k + 2] = ce.lc; cls4[4 * k + 3] = ce.ld;
    }
    if (ms) ms[k] = cw.last_ms;
    if (flops) flops[k] = cw.flops;
    if (quartets) quartets[k] = cw.quartets;
    if (prim_quartets) prim_quartets[k] = cw.prim_quartets;
  }
  return n;
}

int eritile_gpu_get_stats(const eritile_gpu* ctx, eritile_gpu_stats* out) {
  if (!ctx || !out) return ERITILE_ERR_ARG;
  const int rc = guard(const_cast<eritile_gpu*>(ctx), [&] { const_cast<eritile_gpu*>(ctx)->ensure_dealt(); });
  if (rc != ERITILE_OK) return rc;
  out->nbf = ctx->nbf;
  out->nshells = static_cast<int>(ctx->shells.size());
  out->npairs = static_cast<int>(ctx->pm.size());
  out->nclasses = static_cast<int>(ctx->active_work().size());
  out->quartets = ctx->quartets;
  out->prim_quartets = ctx->prim_quartets;
  out->work_items = 0;
  for (const ClassWork& cw : ctx->work)
    if (ctx->active(cw)) out->work_items += cw.n;
  out->model_flops = ctx->model_flops;
  out->last_build_ms = ctx->last_build_ms;
  out->last_schwarz_ms = ctx->last_schwarz_ms;
  out->gpu_launches_last_build = ctx->launches_last;
  out->job_quartets = out->job_prim_quartets = out->pair_path_prim_quartets = 0;
  out->job_model_flops = out->pair_path_model_flops = 0.0;
  for (const ClassWork& cw : ctx->work) {
    if (ctx->active(cw)) {
      out->job_quartets += cw.aquartets;
      out->job_prim_quartets += cw.aprim;
      out->job_model_flops += cw.full_flops();
    }
    if (!cw.fam) {
      out->pair_path_prim_quartets += cw.aprim;
      out->pair_path_model_flops += cw.full_flops();
    }
  }
  return ERITILE_OK;
}

int eritile_gpu_get_variants(const eritile_gpu* ctx, int* var, int cap) {
  if (!ctx || (cap > 0 && !var)) return ERITILE_ERR_ARG;
  for (int c = 0; c < std::min(cap, kNumClasses); ++c) var[c] = ctx->variant(c);
  return kNumClasses;
}

int eritile_gpu_set_variants(eritile_gpu* ctx, const int* var, int n) {
  if (!ctx || !var || n != kNumClasses) return fail(ctx, ERITILE_ERR_ARG, "set_variants: one entry per class");
  for (int c = 0; c < n; ++c)
    if (var[c] < ctx->var_lo(c) || var[c] >= ctx->var_hi(c))
      return fail(ctx, ERITILE_ERR_ARG, "set_variants: variant not available for class " + std::to_string(c));
  ctx->var_choice.assign(var, var + n);
  ctx->dealt = false;
  return ERITILE_OK;
}

long long eritile_gpu_pair_survivors(const eritile_gpu* ctx, long long* count, unsigned long long* ysum) {
  if (!ctx || !ctx->have_lists || !count || !ysum) return -1;
  eritile_gpu* c = const_cast<eritile_gpu*>(ctx);
  if (guard(c, [&] { c->ensure_dealt(); }) != ERITILE_OK) return -1;
  return c->pair_survivors(count, ysum);
}

int eritile_gpu_tune(eritile_gpu* ctx, const double* D, int reps) {
  if (!ctx || !D || reps < 1) return ERITILE_ERR_ARG;
  return guard(ctx, [&] {
    ctx->check_ready();
    ctx->ensure_mats();
    const size_t NN = static_cast<size_t>(ctx->nbf) * ctx->nbf;
    ctx->d_D.alloc(NN);
    CK(cudaMemcpyAsync(ctx->d_D.p, D, sizeof(double) * NN, cudaMemcpyHostToDevice, ctx->stream));
    ctx->prescale(ctx->d_D.p, ctx->d_Ds.p, ctx->stream);
    ctx->tune(ctx->d_Ds.p, reps);
  });
}

int eritile_gpu_max_variants(void) { return kMaxVariants; }

static int tune_gran_entry(eritile_gpu* ctx, const double* D, int reps, int max_sweeps, int* improved) {
  return guard(ctx, [&] {
    ctx->check_ready();
    ctx->ensure_mats();
    const size_t NN = static_cast<size_t>(ctx->nbf) * ctx->nbf;
    ctx->d_D.alloc(NN);
    CK(cudaMemcpyAsync(ctx->d_D.p, D, sizeof(double) * NN, cudaMemcpyHostToDevice, ctx->stream));
    ctx->prescale(ctx->d_D.p, ctx->d_Ds.p, ctx->stream);
    *improved = ctx->tune_granularity(ctx->d_Ds.p, reps, max_sweeps) ? 1 : 0;
  });
}

int eritile_gpu_tune_granularity(eritile_gpu* ctx, const double* D, int reps, int max_sweeps) {
  if (!ctx || !D || reps < 1 || max_sweeps < 1) return ERITILE_ERR_ARG;
  int improved = 0;
  const int rc = tune_gran_entry(ctx, D, reps, max_sweeps, &improved);
  return rc != 0 ? rc : ctx->alloc.accepted;
}

int eritile_gpu_tune_step(eritile_gpu* ctx, const double* D, int reps) {
  if (!ctx || !D || reps < 1) return ERITILE_ERR_ARG;
  int improved = 0;
  const int rc = tune_gran_entry(ctx, D, reps, 1, &improved);
  return rc != 0 ? rc : improved;
}

int eritile_gpu_get_granularity(const eritile_gpu* ctx, int* g, int cap) {
  if (!ctx) return ERITILE_ERR_ARG;
  if (g)
    for (int c = 0; c < std::min(cap, kNumClasses); ++c) g[c] = ctx->gran(c);
  return kNumClasses;
}

int eritile_gpu_set_granularity(eritile_gpu* ctx, int cls_index, int g) {
  if (!ctx || cls_index < 0 || cls_index >= kNumClasses || g < 1 || g > 4096 || (g & (g - 1)) != 0)
    return ERITILE_ERR_ARG;
  if (ctx->alloc.g.empty()) ctx->alloc.init(kNumClasses);
  ctx->alloc.g[cls_index] = g;
  return 0;
}

int eritile_gpu_granularity_history(const eritile_gpu* ctx, int cls_index, int cap, int* g, double* ms,
                                    double* spread, int* accepted) {
  if (!ctx || cls_index < 0 || cls_index >= kNumClasses) return ERITILE_ERR_ARG;
  if (ctx->alloc.history.empty()) return 0;
  const auto& h = ctx->alloc.history[cls_index];
  for (int k = 0; k < std::min<int>(cap, static_cast<int>(h.size())); ++k) {
    if (g) g[k] = h[k].g;
    if (ms) ms[k] = h[k].median;
    if (spread) spread[k] = h[k].spread;
    if (accepted) accepted[k] = h[k].accepted ? 1 : 0;
  }
  return static_cast<int>(h.size());
}

int eritile_alloc_simulate(int ncls, const int* cap, const double* cost, int stride, int max_sweeps, int* g_out,
                           int* sweeps_out) {
  if (ncls < 1 || !cap || !cost || stride < 1 || max_sweeps < 1 || !g_out) return ERITILE_ERR_ARG;
  AllocState s;
  s.init(ncls);
  for (int c = 0; c < ncls; ++c) {
    s.cap[c] = cap[c];
    long long need = 1;
    int k = 0;
    while (need * 2 <= cap[c]) {
      need *= 2;
      ++k;
    }
    if (k >= stride) return ERITILE_ERR_ARG;  // the table must cover g = 1 .. cap
  }
  auto m = [&](int c, int g) {
    int k = 0;
    while ((1 << k) < g) ++k;
    return AllocMeasure{cost[static_cast<size_t>(c) * stride + k], 0.0};
  };
  alloc_tune(s, m, max_sweeps);
  for (int c = 0; c < ncls; ++c) g_out[c] = s.g[c];
  if (sweeps_out) *sweeps_out = s.sweeps;
  return s.accepted;
}

int eritile_gpu_tune_times(const eritile_gpu* ctx, int cap, int* cls_index, double* ms) {
  if (!ctx) return ERITILE_ERR_ARG;
  if (ctx->tune_ms.size() != static_cast<size_t>(kNumClasses) * kMaxVariants) return 0;
  std::vector<int> cl;
  for (int c = 0; c < kNumClasses; ++c)
    for (int v = 0; v < kMaxVariants; ++v)
      if (ctx->tune_ms[static_cast<size_t>(c) * kMaxVariants + v] > 0.0) {
        cl.push_back(c);
        break;
      }
  const int n = static_cast<int>(cl.size());
  for (int k = 0; k < std::min(n, cap); ++k) {
    if (cls_index) cls_index[k] = cl[k];
    if (ms)
      for (int v = 0; v < kMaxVariants; ++v)
        ms[k * kMaxVariants + v] = ctx->tune_ms[static_cast<size_t>(cl[k]) * kMaxVariants + v];
  }
  return n;
}

int eritile_gpu_set_variant(eritile_gpu* ctx, int cls_index, int var) {
  if (!ctx || cls_index < 0 || cls_index >= kNumClasses) return ERITILE_ERR_ARG;
  if (var < ctx->var_lo(cls_index) || var >= ctx->var_hi(cls_index))
    return fail(ctx, ERITILE_ERR_ARG, "kernel variant not available (families on: fam_* only)");
  if (ctx->var_choice.empty()) ctx->var_choice.assign(kNumClasses, -1);
  ctx->var_choice[cls_index] = var;
  ctx->dealt = false;  // the active lists (pair / unit) may change: re-deal
  return ERITILE_OK;
}

int eritile_gpu_set_strips(eritile_gpu* ctx, long long min_quartets, int max_items) {
  if (!ctx || min_quartets < 1 || max_items < 1) return ERITILE_ERR_ARG;
  ctx->kStripMinQuartets = min_quartets;
  ctx->kStripMaxItems = max_items;
  ctx->have_lists = false;
  return ERITILE_OK;
}

int eritile_gpu_set_mode(eritile_gpu* ctx, int mode) {
  if (!ctx || (mode != ERITILE_MODE_CONCURRENT && mode != ERITILE_MODE_DETERMINISTIC))
    return fail(ctx, ERITILE_ERR_ARG, "set_mode: mode must be concurrent (0) or deterministic (1)");
  ctx->det = mode == ERITILE_MODE_DETERMINISTIC;
  return ERITILE_OK;
}
int eritile_gpu_get_mode(const eritile_gpu* ctx) {
  return ctx ? (ctx->det ? ERITILE_MODE_DETERMINISTIC : ERITILE_MODE_CONCURRENT) : ERITILE_ERR_ARG;
}

int eritile_gpu_pair_nprims(const eritile_gpu* ctx, int* nprim) {
  if (!ctx || !nprim) return ERITILE_ERR_ARG;
  for (size_t r = 0; r < ctx->pm.size(); ++r) nprim[r] = ctx->pm[ctx->prod_of_ref[r]].K;
  return ERITILE_OK;
}

int eritile_gpu_set_concurrent(eritile_gpu* ctx, int on) {
  if (!ctx) return ERITILE_ERR_ARG;
  ctx->concurrent = on != 0;
  return ERITILE_OK;
}

int eritile_gpu_set_families(eritile_gpu* ctx, int on) {
  if (!ctx) return ERITILE_ERR_ARG;
  ctx->families = on != 0;
  ctx->have_lists = false;
  return ERITILE_OK;
}

int eritile_gpu_variant_range(const eritile_gpu* ctx, int cls_index, int* lo, int* hi) {
  if (!ctx || cls_index < 0 || cls_index >= kNumClasses || !lo || !hi) return ERITILE_ERR_ARG;
  *lo = ctx->var_lo(cls_index);
  *hi = ctx->var_hi(cls_index);
  return ERITILE_OK;
}

int eritile_gpu_get_variant(const eritile_gpu* ctx, int cls_index) {
  if (!ctx || cls_index < 0 || cls_index >= kNumClasses) return ERITILE_ERR_ARG;
  return ctx->variant(cls_index);
}

int eritile_gpu_class_nvariants(int i) {
  return (i < 0 || i >= kNumClasses) ? ERITILE_ERR_ARG : kClassTable[i].nvar;
}

const char* eritile_gpu_variant_name(int i, int v) {
  if (i < 0 || i >= kNumClasses || v < 0 || v >= kClassTable[i].nvar) return nullptr;
  return kClassTable[i].var_name[v];
}

int eritile_gpu_num_classes(void) { return kNumClasses; }
int eritile_gpu_class_info(int i, int* o) {
  if (i < 0 || i >= kNumClasses || !o) return ERITILE_ERR_ARG;
  const ClassEntry& c = kClassTable[i];
  const int v[10] = {c.la, c.lb, c.lc, c.ld, c.max_m, c.ops, c.prim_terms, c.base, c.contract, c.hrr_terms};
  std::memcpy(o, v, sizeof v);
  return ERITILE_OK;
}

}  // extern "C"
