// Host-visible types shared by the host library and the generated kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace eritile_b200 {

// One primitive pair of an oriented shell pair (A = first shell, L_A >= L_B).
// Restates PrimPair (block.hpp:16-24) for the device: p, P, PA as in
// build_pairs (block.hpp:76-79); U folds the contraction weight D_ik D_jl
// (block.hpp:82), kappa (block.hpp:81) and the base-case prefactor
// 2 pi^(5/2) / (p q sqrt(p+q)) as U_ab U_cd / sqrt(p+q):
// U = sqrt(2) pi^(5/4) kappa coef / p. PB is never read by a plan and is
// dropped. 80 bytes, 16-byte aligned; the first 48 bytes
// (p, U, P, 1/2p) are what every class reads, PA follows so classes whose
// plan never reads PA (QC) on that side skip two 16-byte loads.
struct alignas(16) PrimRec {
  double p, U, Px, Py, Pz, i2p, PAx, PAy, PAz, pad;
};

// Oriented shell pair (product order). `ref` is the reference pair-store
// index (block.hpp:94-101) used to export quartet lists.
struct alignas(16) PairMeta {
  int prim_off, K, bfa, bfb;
  int sha, shb, ref, kstride;  // kstride: ket-record stride in kprims (group size)
  double ABx, ABy, ABz;
  int ksoa, pad;               // this pair's first ket record in kprims
};

// A warp task: 32 consecutive quartets of the flat survivor sequence of one
// (bra group, ket group) pair. Lane l takes quartet r0 + l counted from bra
// bra0 (whose survivor count is cnt[cntp]); bra x's kets are yfirst ..
// yfirst + cnt[x] - 1. r0nq = r0 | (nq << 24), nq <= 32 active lanes.
struct alignas(16) WorkItem {
  int bra0, r0nq, cntp, yfirst;
};

constexpr int kBoysCols = 10;     // F_{M..M+7}(T_i)/k!, exp(-T_i), pad
constexpr int kBoysRows = 641;    // T_i = i/16, T < 40
constexpr double kBoysTmax = 40.0;
constexpr int kBoysMmax = 16;     // slices M = 0..16 (L <= 4)

// A unit of <= 2 product pairs whose primitive-pair records are identical
// except the contraction weight U (generally contracted sibling shells,
// csrc/jk_family.cuh). Records are those of member m0; uw[prim] holds
// (U of m0, U of m1 or 0) per primitive.
struct alignas(16) UnitMeta {
  int prim_off, K, nm, kstride;  // kstride: ket stride in the unit-group-transposed copy
  int m0, m1, ksoa, pad2;        // member product pair ids; first ket record in ukprims
  double ABx, ABy, ABz, pad3;
};

// A strip (csrc/jk_strip.cuh): the single-bra items [i0, i1) of one bra pair
// (or bra unit) run by one CTA that keeps the bra's K rows (and D rows) in
// shared memory. Row blocks: the distinct shells of the bra members, in
// shared-memory row order (rb_n = 0 unused); rowA/rowB: shared-memory row of
// member m's first A / B component.
constexpr int kStripBraMax = 128;
// Deterministic reduction mode (SPEC.md executor "deterministic" accumulator):
// every J/K contribution is rounded to a multiple of 2^-44 and added as a
// 64-bit integer, so the sums are exact and independent of atomic order
// (bitwise reproducible). Range |Jacc|, |Kacc| < 2^19 (two's complement wrap
// of partial sums is harmless); rounding error <= 2^-45 per contribution.
constexpr double kDetScale = 17592186044416.0;  // 2^44  // strip bras: primitive pairs staged in shared memory

// Digestion metadata of a ket unit (or product pair: member 1 = member 0),
// one 64-byte read per lane and item in the strip kernels instead of the
// dependent PairMeta -> cpos chain after the primitive loop.
struct alignas(16) KetMeta {
  int bfa[2], bfb[2];    // first basis functions of member m's C / D shells
  int colc[2], cold[2];  // compact column (cpos) of member m's C / D shells
  int offd[2];           // 1 if member m's shells differ (sha != shb)
  int m[2];              // product pair id of member m
  double q[2];           // Schwarz Q of member m
};

struct alignas(16) Strip {
  int bra, i0, i1, nrows;
  int rowA[2], rowB[2];
  int rb_bf[4];
  int rb_n[4];
};

struct LaunchArgs {
  int mode;  // 0 = J/K digestion, 1 = Schwarz diagonal, 2 = raw quartets
  const WorkItem* items;
  long long nitems;
  const int* cnt;        // survivor counts per (group pair, bra)
  const int* pair_list;  // Schwarz: product pair ids
  long long npair_list;
  double* Qout;          // Schwarz: per product pair
  const int* qpairs;     // mode 2: (bra, ket) product pair ids
  long long nq;
  double* qout;          // mode 2: NV raw values per quartet, kernel order
  const PairMeta* pm;
  const PrimRec* prims;
  const PrimRec* kprims;  // group-transposed copy of prims (ket reads of the lane kernels)
  const double* D;
  double* J;
  double* K;
  int N;
  const double* boys_tab;  // kBoysMmax+1 slices of kBoysRows*kBoysCols
  cudaStream_t stream;
  int gran;   // Workload Allocator granularity: consecutive work items per warp task (>= 1)
  int grid;   // 0 = auto
  int block;  // threads per CTA
  // family (unit) launches: work items index units
  const UnitMeta* um;
  const double2* uw;     // per primitive: member weights
  const PrimRec* ukprims;  // unit-group-transposed records (ket reads of the unit kernels)
  const double2* ukw;      // ... and their member weights
  const double* Qp;      // Schwarz Q per product pair
  double tau;            // screening threshold (<= 0: none)
  long long seg[5];      // unit launches: item offsets of the (1,1) (1,2) (2,1) (2,2) member segments
  // strip variants: per member segment sg, strips[sseg[sg] .. sseg[sg+1]) own
  // the items [seg[sg], sitem[sg]); items [sitem[sg], seg[sg+1]) are packed
  // multi-bra items for the lane kernels (pair lists: segment 0 only)
  const Strip* strips;
  long long sseg[5];
  long long sitem[4];
  int det;          // deterministic mode: J/K accumulate as int64 fixed point (kDetScale)
  const int* cols;  // compact K/D column list of the class: L_C functions (++ L_D functions if L_D != L_C)
  const int* cpos;  // per shell: first compact column within its own L list
  const KetMeta* kmeta;  // per ket unit (unit kernels) or per product pair
  int ncols, ncolC;
  int* sctr;  // strip variants: 4 zeroed-per-launch strip counters (dynamic strip hand-out); null = static stride
};

using LaunchFn = void (*)(const LaunchArgs&);

// One canonical ERI class and its kernel variants (straight-line lane
// kernels at several residency targets and/or the CTA-cooperative table
// kernel); `def` is the variant used until the allocator tunes the class.
constexpr int kMaxVariants = 32;
struct ClassEntry {
  int la, lb, lc, ld, max_m, ops, prim_terms, base, contract, hrr_terms;
  int nvar;
  LaunchFn var[kMaxVariants];
  const char* var_name[kMaxVariants];
  int def;
  int nfam;     // the last nfam variants are unit ("fam_") kernels
  int fam_def;  // default unit variant (absolute index), -1 if none
};

extern const ClassEntry kClassTable[];
extern const int kNumClasses;
extern const int kMaxL;

}  // namespace eritile_b200
