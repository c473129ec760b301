/* eritile_gpu.h — C ABI of the B200 Fock-build engine (drop-in boundary).
 *
 * The reference (arxiv 2412.13203, proj/include/eritile/) is a header-only
 * C++20 library with no executor; the executor contract it specifies is
 *   eval_block(QuadBlock, ExecutionPlan, D, Accumulator&)
 *   build_g(blocks, plans, D, mode) -> G
 * called once per SCF iteration by scf_iterate. This ABI
 * replaces that contract with plain pointers and sizes; every entry point
 * cites the reference interface it stands in for. The C++ wrapper with the
 * reference's names and exception behaviour is include/eritile/executor.hpp.
 *
 * Conventions: matrices are N x N row-major FP64, caller-owned, N =
 * basis_dimension (molecule.hpp:193-197) in expand_functions order
 * (molecule.hpp:185-191; components x-major, molecule.hpp:176-183). Inputs
 * are copied at call time. Every function returns 0 on success and a
 * negative code on failure; eritile_gpu_last_error() describes it. There is
 * no CPU fallback: without a CUDA device eritile_gpu_create fails.
 */
#ifndef ERITILE_GPU_H
#define ERITILE_GPU_H
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct eritile_gpu eritile_gpu;

enum {
  ERITILE_OK = 0,
  ERITILE_ERR_ARG = -1,     /* std::invalid_argument in the reference */
  ERITILE_ERR_PARSE = -2,   /* eritile::ParseError (molecule.hpp:72-74) */
  ERITILE_ERR_CUDA = -3,    /* device failure / no device */
  ERITILE_ERR_STATE = -4,   /* call order (e.g. build_jk before set_screening) */
  ERITILE_ERR_DOMAIN = -5   /* std::domain_error (boys.hpp:48-50) */
};

/* build_g reduction modes (SPEC.md executor, Accumulator): concurrent FP64
 * atomics (default), or deterministic - contributions are rounded to
 * multiples of 2^-44 and summed as 64-bit integers, exact and independent of
 * scheduling, so results are bitwise reproducible for a given variant table
 * (|J|, |K| accumulators < 2^19). In deterministic mode the partial
 * accumulators of build_jk_partial_device hold int64 values: sum them across
 * ranks as int64. Strip variants run their items on the lane kernels. */
enum { ERITILE_MODE_CONCURRENT = 0, ERITILE_MODE_DETERMINISTIC = 1 };

typedef struct eritile_gpu_stats {
  int nbf, nshells, npairs, nclasses;
  long long quartets;        /* surviving canonical quartets on this rank */
  long long prim_quartets;   /* surviving primitive quartets on this rank */
  long long work_items;      /* warp tasks on this rank */
  double model_flops;        /* SURVEY.md §8d F_c summed over classes (this rank) */
  double last_build_ms;      /* device time of the last build_jk (CUDA events) */
  double last_schwarz_ms;
  int gpu_launches_last_build; /* kernels launched by the last build */
  /* Whole job (all ranks), with the variant table this context uses: */
  long long job_quartets;
  long long job_prim_quartets;      /* primitive quartets the chosen kernels evaluate */
  double job_model_flops;           /* F_c over the executed plans */
  /* The same quartets on the per-pair kernels (no shared-primitive units):
   * the primitive-quartet count of SURVEY 8d's model. */
  long long pair_path_prim_quartets;
  double pair_path_model_flops;
} eritile_gpu_stats;

/* Create a context on CUDA device `device`. Fails if no device.
 * device = -1 creates a host-only context: input parsing, the host Block
 * Constructor and screened-list construction from a supplied Q
 * (eritile_gpu_set_schwarz) work; every integral entry point fails with
 * ERITILE_ERR_CUDA. It exists so the host logic is testable without a GPU;
 * it is not a CPU fallback. */
int eritile_gpu_create(int device, eritile_gpu** out);
void eritile_gpu_destroy(eritile_gpu* ctx);
const char* eritile_gpu_last_error(const eritile_gpu* ctx);

/* parse_xyz (molecule.hpp:105-158) + BasisSetTable::parse (basis_set.hpp:
 * 33-84) + attach_basis (basis_set.hpp:127-155). */
int eritile_gpu_load_molecule(eritile_gpu* ctx, const char* xyz_text, const char* basis_text);
/* Alternative: already-normalised shells (Shell, molecule.hpp:39-50):
 * L[s], K[s], center[3s..], atom[s]; exponents/coefficients concatenated. */
int eritile_gpu_load_shells(eritile_gpu* ctx, int nshell, const int* L, const int* K,
                            const double* center, const int* atom, const double* exps,
                            const double* coefs, int natoms, const int* Z, const double* pos);
int eritile_gpu_nbf(const eritile_gpu* ctx);
/* Shell table after attach_basis: L, contraction degree, first basis
 * function (expand_functions order, molecule.hpp:185-191). */
int eritile_gpu_shell_info(const eritile_gpu* ctx, int* L, int* K, int* bf_off);
int eritile_gpu_nshells(const eritile_gpu* ctx);
int eritile_gpu_nelectrons(const eritile_gpu* ctx);
double eritile_gpu_nuclear_repulsion(const eritile_gpu* ctx);

/* build_pairs (block.hpp:52-103): all S(S+1)/2 pairs, kappa screen
 * |coef|*kappa < kappa_screen drops primitive pairs (0 = off), upload. */
int eritile_gpu_build_pairs(eritile_gpu* ctx, double kappa_screen);
int eritile_gpu_npairs(const eritile_gpu* ctx);
/* Reference pair-store order: shells (i<=j) of pair x, x < npairs. */
int eritile_gpu_pair_shells(const eritile_gpu* ctx, int* i, int* j);
/* Kept primitive pairs of each pair (ShellPair::prims.size(), block.hpp:26-31). */
int eritile_gpu_pair_nprims(const eritile_gpu* ctx, int* nprim);

/* Schwarz diagonal on the GPU; Q per pair in reference pair-store order
 * (Q may be NULL). Not in the reference. */
int eritile_gpu_schwarz(eritile_gpu* ctx, double* Q);
/* Override Q (reference order) — used to share one Q with a checker. */
int eritile_gpu_set_schwarz(eritile_gpu* ctx, const double* Q);

/* Multi-GPU sharding: this context evaluates shard `rank` of
 * `nranks`. Each class's active work list is cut into chunks of 64 warp
 * tasks, weighted by model FLOPs, and dealt by LPT (heaviest chunk to the
 * least-loaded rank). The deal is a function of the screened lists and the
 * variant table only, so ranks that share both get a disjoint cover of the
 * canonical quartet list; give every rank the same table
 * (eritile_gpu_get_variants / eritile_gpu_set_variants). May be called
 * before or after set_screening. */
int eritile_gpu_set_shard(eritile_gpu* ctx, int rank, int nranks);
/* Build the screened quartet work lists: keep (x,y) iff Q_x*Q_y >= tau
 * (tau <= 0: no screening). Blocks are class- and contraction-sorted
 * (Permutation, block.hpp:115-150 / PAPER.md:223-250). */
int eritile_gpu_set_screening(eritile_gpu* ctx, double tau);
long long eritile_gpu_num_quartets(const eritile_gpu* ctx);
/* Export this rank's canonical quartet list as reference pair-store index
 * pairs (x <= y), sorted ascending by (x, y). Returns the count. */
long long eritile_gpu_quartets(const eritile_gpu* ctx, int* xs, int* ys, long long cap);
/* Compact list identity for lists too large to export: per reference pair x
 * (npairs entries), the number of this rank's canonical quartets (x, y),
 * x <= y, and the wrapping 64-bit sum of splitmix64(y) over them. Returns
 * the total count (-1 on error). */
long long eritile_gpu_pair_survivors(const eritile_gpu* ctx, long long* count, unsigned long long* ysum);

/* build_g's J/K half: true Coulomb J and exchange K for a
 * symmetric density D (G = 2J - K for RHF). Host buffers; includes H2D of D
 * and D2H of J, K. Single rank: complete result. */
int eritile_gpu_build_jk(eritile_gpu* ctx, const double* D, double* J, double* K);
/* Device-resident variant for multi-GPU: D, accumulators are device pointers
 * on this context's device; JKacc is 2*N*N doubles (Jacc ‖ Kacc, zeroed by
 * the call) holding this rank's unsymmetrised partial sums, to be summed
 * across ranks (one allreduce) and then passed to eritile_gpu_finalize.
 * stream = cudaStream_t (NULL = context stream). */
int eritile_gpu_build_jk_partial_device(eritile_gpu* ctx, const double* dD, double* dJKacc,
                                        void* stream);
int eritile_gpu_finalize_device(eritile_gpu* ctx, const double* dJKacc, double* dJ, double* dK,
                                void* stream);
int eritile_gpu_build_jk_device(eritile_gpu* ctx, const double* dD, double* dJ, double* dK,
                                void* stream);

/* One-electron S, T, V on the host; N x N. */
int eritile_gpu_one_electron(eritile_gpu* ctx, double* S, double* T, double* V);

/* boys (boys.hpp:46-54) evaluated by the device routine for n arguments. */
int eritile_gpu_boys(eritile_gpu* ctx, int m_max, const double* T, int n, double* F);
/* Scaled integrals of one quartet of reference pairs (x, y) in the reference
 * component order a-major over (i,j,k,l) of pair x=(i,j), y=(k,l). */
int eritile_gpu_eri_quartet(eritile_gpu* ctx, int x, int y, double* out);

int eritile_gpu_get_stats(const eritile_gpu* ctx, eritile_gpu_stats* out);
/* Profiling: with on != 0 every class launch is bracketed by CUDA events on
 * the launch stream. class_profile returns the number of class launches and
 * fills (up to cap) the class (4 ints), last device time (ms), model FLOPs,
 * quartets and primitive quartets of each. */
int eritile_gpu_set_profiling(eritile_gpu* ctx, int on);
int eritile_gpu_class_profile(eritile_gpu* ctx, int cap, int* cls4, double* ms, double* flops,
                              long long* quartets, long long* prim_quartets);
/* Workload Allocator, first stage (kernel variant per class): time every
 * kernel variant of every class on its whole (unsharded) work list on
 * density D (host, N x N), median of `reps` launches each, and keep the
 * fastest per class. The second stage is Algorithm 2 proper
 * (eritile_gpu_tune_granularity below). Variant families
 * (eritile_gpu_variant_name):
 *   "lane_*"   one lane per contracted quartet running the class's
 *              straight-line plan (loop style x CTA shape x register budget);
 *   "fam_*"    the same over shared-primitive units (sibling shells);
 *   "strip_*" / "fstrip_*"  bra-stationary strips (pair / unit lists): K rows
 *              of the bra in shared memory, flushed once per strip; suffixes
 *              _o7 (batched CAS + prefetch), _a (warp-aggregated K updates),
 *              _k2 (two ket primitives per bra record), _p (L1 prefetch),
 *              _s (d-column K updates to global memory), _tNNN CTA size;
 *   "coop" / "coopw"  the CTA- / warp-cooperative level-scheduled plan
 *              (high L).
 * The choice changes atomic summation order only. */
int eritile_gpu_tune(eritile_gpu* ctx, const double* D, int reps);
/* Per class of the last tune: class table index and the median ms of each
 * variant (eritile_gpu_max_variants() slots per class, 0 = not timed). */
int eritile_gpu_tune_times(const eritile_gpu* ctx, int cap, int* cls_index, double* ms);
/* Variant slots per class (the stride of eritile_gpu_tune_times). */
int eritile_gpu_max_variants(void);

/* Workload Allocator, Algorithm 2 (SPEC.md:366-425
 * `tune` / `combine` / `revert` / `measure`): per class, the granularity g
 * = work items (32 contracted quartets each) fused into one warp task is
 * doubled (Combine) and kept only if the class's measured time drops
 * (median of `reps` launches on the class's full work list, warm-up
 * discarded), else reverted; sweeps repeat while any class improved.
 * Cap = min(task count, 4096); the coop table kernels are not tunable
 * (cap 1). Results change only by atomic summation order.
 *   tune_granularity: the loop to convergence (at most max_sweeps sweeps);
 *                     returns the number of accepted combines so far.
 *   tune_step:        one sweep (SCF drivers interleave it with their first
 *                     iterations); returns 1 if a class
 *                     improved, 0 once converged.
 *   get_granularity:  g per class into g[0..cap); returns the class count.
 *   set_granularity:  g must be a power of two in [1, 4096].
 *   granularity_history: every measured (g, median ms, spread, accepted)
 *                     of class cls_index; returns the count.
 * eritile_alloc_simulate runs the same loop against a mock cost table
 * (cost[c * stride + k] = time at g = 2^k; no device needed) and returns
 * the number of accepted combines. */
int eritile_gpu_tune_granularity(eritile_gpu* ctx, const double* D, int reps, int max_sweeps);
int eritile_gpu_tune_step(eritile_gpu* ctx, const double* D, int reps);
int eritile_gpu_get_granularity(const eritile_gpu* ctx, int* g, int cap);
int eritile_gpu_set_granularity(eritile_gpu* ctx, int cls_index, int g);
int eritile_gpu_granularity_history(const eritile_gpu* ctx, int cls_index, int cap, int* g, double* ms,
                                    double* spread, int* accepted);
int eritile_alloc_simulate(int ncls, const int* cap, const double* cost, int stride, int max_sweeps, int* g_out,
                           int* sweeps_out);
int eritile_gpu_set_variant(eritile_gpu* ctx, int cls_index, int var);
/* The whole variant table (one entry per class, eritile_gpu_num_classes):
 * get returns the class count; set validates every entry first. */
int eritile_gpu_get_variants(const eritile_gpu* ctx, int* var, int cap);
int eritile_gpu_set_variants(eritile_gpu* ctx, const int* var, int n);
/* Shared-primitive units (generally contracted sibling shells evaluated once
 * per primitive quartet, csrc/jk_family.cuh): on by default; classes with
 * "fam_" variants then run only those. Takes effect at the next
 * set_screening. Results and quartet lists are unchanged. */
int eritile_gpu_set_families(eritile_gpu* ctx, int on);
/* Strip lists (bra-stationary CTAs, K rows in shared memory): bras with at
 * least min_quartets survivors in a class get single-bra items grouped into
 * strips of at most max_items warp tasks (defaults 1024, 1024); the rest stay
 * packed. Takes effect at the next set_screening; lists and results are
 * unchanged, only the work layout. */
int eritile_gpu_set_strips(eritile_gpu* ctx, long long min_quartets, int max_items);
/* Reduction mode, ERITILE_MODE_* (takes effect at the next build). */
int eritile_gpu_set_mode(eritile_gpu* ctx, int mode);
int eritile_gpu_get_mode(const eritile_gpu* ctx);
/* Class launches of a build on 4 streams (default) or on one stream. */
int eritile_gpu_set_concurrent(eritile_gpu* ctx, int on);
/* Active variant index range [lo, hi) of a class in this context. */
int eritile_gpu_variant_range(const eritile_gpu* ctx, int cls_index, int* lo, int* hi);
int eritile_gpu_get_variant(const eritile_gpu* ctx, int cls_index);
int eritile_gpu_class_nvariants(int cls_index);
const char* eritile_gpu_variant_name(int cls_index, int var);
/* Plan statistics of the generated class kernels, i < num_classes:
 * la lb lc ld max_m ops prim_terms base contract hrr_terms. */
int eritile_gpu_num_classes(void);
int eritile_gpu_class_info(int i, int* out10);

#ifdef __cplusplus
}
#endif
#endif
