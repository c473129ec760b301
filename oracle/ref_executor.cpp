// oracle/_ref driver — TEST INFRASTRUCTURE ONLY (never shipped, never on the
// product path). Compiles the UNMODIFIED reference headers from
// /root/reference/proj/include (block.hpp, boys.hpp, compiler.hpp, dag.hpp,
// molecule.hpp, basis_set.hpp) against oracle/shim/Eigen/Dense and adds the
// executor the reference specifies but does not ship:
//   * plan interpreter: binding + base case SPEC.md:290,316; plan semantics
//     compiler.hpp:131-147,341-365; PrimPair fields block.hpp:16-24;
//   * digestion: shell-level degeneracy with 1/4-weighted K
//     terms, then symmetrisation; true J = J_sym/2, true K = K_sym
//     (SURVEY.md Appendix C);
//   * build_g worker pool over QuadBlocks with private partial matrices
//     merged at the end.
// Schwarz screening is NOT in the reference; the rule used
// here is the one the product uses: Q_x =
// sqrt(max_{mu in i, nu in j} |(mu nu|mu nu)|) over scaled components, keep
// (x,y) iff Q_x*Q_y >= tau.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numbers>
#include <string>
#include <thread>
#include <vector>

#include "eritile/basis_set.hpp"
#include "eritile/block.hpp"
#include "eritile/boys.hpp"
#include "eritile/compiler.hpp"
#include "eritile/molecule.hpp"

using namespace eritile;

namespace {

thread_local std::string g_err;

struct Ctx {
  Molecule mol;
  std::vector<ShellPair> pairs;
  std::vector<PairTile> tiles;
  std::vector<QuadBlock> blocks;
  std::vector<int> bf_off;  // first basis function of each shell
  int nbf = 0;
  std::map<EriClass, ExecutionPlan> plans;
  std::mutex plan_mu;
  std::vector<double> Q;  // Schwarz per pair (pair-store order), lazily
  bool have_q = false;

  const ExecutionPlan& plan(const EriClass& c) {
    std::lock_guard<std::mutex> lk(plan_mu);
    auto it = plans.find(c);
    if (it == plans.end()) it = plans.emplace(c, compile_class(c)).first;
    return it->second;
  }
};

// Component scale per shell component (molecule.hpp:207-213), x-major order
// (molecule.hpp:176-183).
std::vector<double> comp_scales(int L) {
  std::vector<double> s;
  for (const auto& m : shell_components(L)) s.push_back(component_norm_scale(m));
  return s;
}

// Evaluate one shell quartet (bra pair `b`, ket pair `k`) with plan `P`;
// out receives n_i*n_j*n_k*n_l RAW (unscaled) values, a-major.
// Follows SURVEY.md Appendix C exactly (binding list and plan semantics).
void eval_quartet(const ShellPair& b, const ShellPair& k, const ExecutionPlan& P,
                  std::vector<double>& r, std::vector<double>& t,
                  std::vector<double>& F, double* out) {
  t.assign(static_cast<std::size_t>(P.contracted_slot_count), 0.0);
  r.resize(static_cast<std::size_t>(std::max(P.prim_slot_count, 1)));
  F.resize(static_cast<std::size_t>(P.max_m) + 1);
  const double two_pi_25 = 2.0 * std::pow(std::numbers::pi, 2.5);
  for (const PrimPair& a : b.prims) {
    for (const PrimPair& c : k.prims) {
      const double pq = a.p + c.p;
      const double rho = a.p * c.p / pq;
      const Vec3 W = (a.p * a.P + c.p * c.P) / pq;
      const double T = rho * (a.P - c.P).squaredNorm();
      const double pref = two_pi_25 / (a.p * c.p * std::sqrt(pq)) * a.kappa * c.kappa;
      boys_inplace(P.max_m, T, F.data());
      const Vec3 WP = W - a.P, WQ = W - c.P;
      auto coeff = [&](CoeffKind kind, int dir) -> double {
        switch (kind) {
          case CoeffKind::Unit: return 1.0;
          case CoeffKind::PA: return a.PA[dir];
          case CoeffKind::PB: return a.PB[dir];
          case CoeffKind::QC: return c.PA[dir];
          case CoeffKind::QD: return c.PB[dir];
          case CoeffKind::WP: return WP[dir];
          case CoeffKind::WQ: return WQ[dir];
          case CoeffKind::InvTwoP: return a.inv_two_p;
          case CoeffKind::InvTwoQ: return c.inv_two_p;
          case CoeffKind::InvTwoPQ: return 0.5 / pq;
          case CoeffKind::ITP_RP: return a.inv_two_p * rho / a.p;
          case CoeffKind::ITQ_RQ: return c.inv_two_p * rho / c.p;
          case CoeffKind::AB:
          case CoeffKind::CD: return 0.0;  // never in the primitive segment
        }
        return 0.0;
      };
      for (const PlanInstr& ins : P.prim) {
        if (ins.base_m >= 0) {
          r[ins.dst] = pref * F[ins.base_m];
        } else {
          double s = 0.0;
          for (const PlanTerm& tm : ins.terms) s += tm.factor * coeff(tm.kind, tm.dir) * r[tm.src];
          r[ins.dst] = s;
        }
      }
      const double w = a.coef * c.coef;
      for (const auto& [reg, cs] : P.contract) t[cs] += w * r[reg];
    }
  }
  for (const PlanInstr& ins : P.hrr) {
    double s = 0.0;
    for (const PlanTerm& tm : ins.terms) {
      double cf = tm.kind == CoeffKind::Unit ? 1.0
                  : tm.kind == CoeffKind::AB ? b.AB[tm.dir]
                                             : k.AB[tm.dir];
      s += tm.factor * cf * t[tm.src];
    }
    t[ins.dst] = s;
  }
  for (std::size_t n = 0; n < P.targets.size(); ++n) out[n] = t[P.targets[n]];
}

// Component scales per L, built once (no per-quartet allocation).
const std::vector<double>& scales_of(int L) {
  static const std::vector<std::vector<double>> tab = [] {
    std::vector<std::vector<double>> t;
    for (int l = 0; l <= 6; ++l) t.push_back(comp_scales(l));
    return t;
  }();
  return tab.at(static_cast<std::size_t>(L));
}

struct Scratch {
  std::vector<double> r, t, F, v;
};

// Scaled quartet values (Appendix C: "Scale each value by prod component_norm_scale").
void quartet_scaled(Ctx& C, int x, int y, Scratch& S) {
  const ShellPair& b = C.pairs[x];
  const ShellPair& k = C.pairs[y];
  EriClass cls{b.cls.li, b.cls.lj, k.cls.li, k.cls.lj};
  const ExecutionPlan& P = C.plan(cls);
  S.v.resize(P.targets.size());
  eval_quartet(b, k, P, S.r, S.t, S.F, S.v.data());
  const std::vector<double>&si = scales_of(cls.la), &sj = scales_of(cls.lb), &sk = scales_of(cls.lc),
                           &sl = scales_of(cls.ld);
  std::size_t n = 0;
  for (double a : si)
    for (double bb : sj)
      for (double c : sk)
        for (double d : sl) S.v[n++] *= a * bb * c * d;
}

void compute_q(Ctx& C) {
  if (C.have_q) return;
  const int np = static_cast<int>(C.pairs.size());
  C.Q.assign(np, 0.0);
  unsigned nt = std::max(1u, std::thread::hardware_concurrency());
  std::atomic<int> next{0};
  std::vector<std::thread> th;
  for (unsigned w = 0; w < nt; ++w)
    th.emplace_back([&] {
      Scratch S;
      for (int x; (x = next.fetch_add(1)) < np;) {
        quartet_scaled(C, x, x, S);
        const Shell& a = C.mol.shells[C.pairs[x].i];
        const Shell& b = C.mol.shells[C.pairs[x].j];
        const int ni = a.num_functions(), nj = b.num_functions();
        double mx = 0.0;
        for (int m = 0; m < ni; ++m)
          for (int n = 0; n < nj; ++n) {
            // (mn|mn) sits at a-major index ((m*nj+n)*ni+m)*nj+n
            double v = std::fabs(S.v[((std::size_t(m) * nj + n) * ni + m) * nj + n]);
            mx = std::max(mx, v);
          }
        C.Q[x] = std::sqrt(mx);
      }
    });
  for (auto& t : th) t.join();
  C.have_q = true;
}

inline bool keep(const Ctx& C, double tau, int x, int y) {
  return tau <= 0.0 || C.Q[x] * C.Q[y] >= tau;
}

// Digest one canonical quartet (x <= y, pair-store order) into partial J, K.
void digest(const Ctx& C, int x, int y, const double* v, const double* D, double* J,
            double* K) {
  const ShellPair& b = C.pairs[x];
  const ShellPair& k = C.pairs[y];
  const int si = b.i, sj = b.j, sk = k.i, sl = k.j;
  const int oi = C.bf_off[si], oj = C.bf_off[sj], ok = C.bf_off[sk], ol = C.bf_off[sl];
  const int ni = C.mol.shells[si].num_functions(), nj = C.mol.shells[sj].num_functions();
  const int nk = C.mol.shells[sk].num_functions(), nl = C.mol.shells[sl].num_functions();
  const double deg = (si != sj ? 2.0 : 1.0) * (sk != sl ? 2.0 : 1.0) * (x != y ? 2.0 : 1.0);
  const double q = 0.25 * deg;
  const std::size_t N = C.nbf;
  std::size_t n = 0;
  for (int m = 0; m < ni; ++m)
    for (int nn = 0; nn < nj; ++nn)
      for (int l = 0; l < nk; ++l)
        for (int s = 0; s < nl; ++s, ++n) {
          const std::size_t mu = oi + m, nu = oj + nn, la = ok + l, si_ = ol + s;
          const double val = v[n];
          J[mu * N + nu] += D[la * N + si_] * val * deg;
          J[la * N + si_] += D[mu * N + nu] * val * deg;
          K[mu * N + la] += q * D[nu * N + si_] * val;
          K[nu * N + si_] += q * D[mu * N + la] * val;
          K[mu * N + si_] += q * D[nu * N + la] * val;
          K[nu * N + la] += q * D[mu * N + si_] * val;
        }
}

// Enumerate canonical quartets block by block (block.hpp:135-150; diagonal
// blocks iterate y >= x), calling fn(x, y) for survivors.
template <typename Fn>
void for_each_quartet_in_block(const Ctx& C, const QuadBlock& blk, double tau, Fn&& fn) {
  const PairTile& ti = C.tiles[blk.bra_tile];
  const PairTile& tj = C.tiles[blk.ket_tile];
  for (int x = ti.first; x < ti.first + ti.count; ++x) {
    int y0 = blk.bra_tile == blk.ket_tile ? x : tj.first;
    for (int y = y0; y < tj.first + tj.count; ++y)
      if (keep(C, tau, x, y)) fn(x, y);
  }
}

int build_jk_impl(Ctx& C, const double* D, double tau, int nthreads, long long stride,
                  long long offset, double* Jout, double* Kout, long long* nq_out,
                  double* seconds = nullptr) {
  if (tau > 0.0) compute_q(C);
  const std::size_t N = C.nbf, NN = N * N;
  // compile every plan up front (offline step; not part of the build)
  for (const auto& blk : C.blocks) C.plan(blk.cls);
  if (nthreads <= 0) nthreads = std::max(1u, std::thread::hardware_concurrency());
  std::vector<std::vector<double>> Jp(nthreads, std::vector<double>(NN, 0.0));
  std::vector<std::vector<double>> Kp(nthreads, std::vector<double>(NN, 0.0));
  std::vector<long long> nq(nthreads, 0);
  std::atomic<long long> next{0};
  const long long nb = static_cast<long long>(C.blocks.size());
  std::vector<std::thread> th;
  const auto t0 = std::chrono::steady_clock::now();
  for (int w = 0; w < nthreads; ++w)
    th.emplace_back([&, w] {
      Scratch S;
      // only the sampled blocks offset, offset + stride, ... are claimed
      const long long st = stride > 1 ? stride : 1, o0 = stride > 1 ? offset : 0;
      for (long long bi; (bi = o0 + next.fetch_add(1) * st) < nb;) {
        for_each_quartet_in_block(C, C.blocks[bi], tau, [&](int x, int y) {
          quartet_scaled(C, x, y, S);
          digest(C, x, y, S.v.data(), D, Jp[w].data(), Kp[w].data());
          ++nq[w];
        });
      }
    });
  for (auto& t : th) t.join();
  if (seconds)
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::vector<double> J(NN, 0.0), K(NN, 0.0);
  for (int w = 0; w < nthreads; ++w)  // merge in worker order
    for (std::size_t e = 0; e < NN; ++e) {
      J[e] += Jp[w][e];
      K[e] += Kp[w][e];
    }
  for (std::size_t a = 0; a < N; ++a)
    for (std::size_t b = 0; b < N; ++b) {
      Jout[a * N + b] = 0.25 * (J[a * N + b] + J[b * N + a]);
      Kout[a * N + b] = 0.5 * (K[a * N + b] + K[b * N + a]);
    }
  if (nq_out) {
    long long s = 0;
    for (auto v : nq) s += v;
    *nq_out = s;
  }
  return 0;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_create(const char* xyz_text, const char* basis_text, double kappa_screen,
                 int tile_size) {
  try {
    auto C = std::make_unique<Ctx>();
    Molecule geom = parse_xyz(xyz_text);
    C->mol = geom;
    attach_basis(C->mol, BasisSetTable::parse(basis_text));
    C->pairs = build_pairs(C->mol.shells, kappa_screen);
    C->tiles = tile_pairs(C->pairs, tile_size);
    C->blocks = make_blocks(C->tiles);
    int off = 0;
    for (const auto& s : C->mol.shells) {
      C->bf_off.push_back(off);
      off += s.num_functions();
    }
    C->nbf = off;
    return C.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_destroy(void* c) { delete static_cast<Ctx*>(c); }
int ref_nbf(void* c) { return static_cast<Ctx*>(c)->nbf; }
int ref_nshells(void* c) { return static_cast<int>(static_cast<Ctx*>(c)->mol.shells.size()); }
int ref_npairs(void* c) { return static_cast<int>(static_cast<Ctx*>(c)->pairs.size()); }
int ref_ntiles(void* c) { return static_cast<int>(static_cast<Ctx*>(c)->tiles.size()); }
long long ref_nblocks(void* c) { return static_cast<long long>(static_cast<Ctx*>(c)->blocks.size()); }
int ref_nelectrons(void* c) { return static_cast<Ctx*>(c)->mol.electron_count(); }

// Shell table: L, K, atom, first basis function, centre (3), and the folded
// coefficients/exponents (flattened; prim_off gives each shell's start).
void ref_shells(void* cv, int* L, int* K, int* atom, int* bf_off, double* center) {
  Ctx* C = static_cast<Ctx*>(cv);
  for (std::size_t s = 0; s < C->mol.shells.size(); ++s) {
    const Shell& sh = C->mol.shells[s];
    L[s] = sh.total_momentum;
    K[s] = sh.contraction_degree();
    atom[s] = sh.atom;
    bf_off[s] = C->bf_off[s];
    for (int d = 0; d < 3; ++d) center[3 * s + d] = sh.center[d];
  }
}
void ref_shell_prims(void* cv, int s, double* exps, double* coefs) {
  const Shell& sh = static_cast<Ctx*>(cv)->mol.shells[s];
  for (int k = 0; k < sh.contraction_degree(); ++k) {
    exps[k] = sh.exponents[k];
    coefs[k] = sh.coefficients[k];
  }
}
void ref_atoms(void* cv, int* Z, double* pos) {
  Ctx* C = static_cast<Ctx*>(cv);
  for (std::size_t a = 0; a < C->mol.atoms.size(); ++a) {
    Z[a] = C->mol.atoms[a].atomic_number;
    for (int d = 0; d < 3; ++d) pos[3 * a + d] = C->mol.atoms[a].position[d];
  }
}
int ref_natoms(void* c) { return static_cast<int>(static_cast<Ctx*>(c)->mol.atoms.size()); }

// Pair store in reference order (block.hpp:94-101): shells i<=j, prim count,
// and the per-primitive-pair records (p, inv_two_p, P, PA, PB, kappa, coef).
void ref_pairs(void* cv, int* i, int* j, int* nprim) {
  Ctx* C = static_cast<Ctx*>(cv);
  for (std::size_t x = 0; x < C->pairs.size(); ++x) {
    i[x] = C->pairs[x].i;
    j[x] = C->pairs[x].j;
    nprim[x] = static_cast<int>(C->pairs[x].prims.size());
  }
}
void ref_pair_prims(void* cv, int x, double* rec /* nprim x 13 */) {
  const ShellPair& sp = static_cast<Ctx*>(cv)->pairs[x];
  for (std::size_t k = 0; k < sp.prims.size(); ++k) {
    const PrimPair& p = sp.prims[k];
    double* o = rec + 13 * k;
    o[0] = p.p; o[1] = p.inv_two_p;
    for (int d = 0; d < 3; ++d) { o[2 + d] = p.P[d]; o[5 + d] = p.PA[d]; o[8 + d] = p.PB[d]; }
    o[11] = p.kappa; o[12] = p.coef;
  }
}
unsigned long long ref_pair_store_bytes(void* c) {
  return pair_store_bytes(static_cast<Ctx*>(c)->pairs);
}
void ref_tiles(void* cv, int* li, int* lj, int* first, int* count) {
  Ctx* C = static_cast<Ctx*>(cv);
  for (std::size_t t = 0; t < C->tiles.size(); ++t) {
    li[t] = C->tiles[t].cls.li; lj[t] = C->tiles[t].cls.lj;
    first[t] = C->tiles[t].first; count[t] = C->tiles[t].count;
  }
}

int ref_schwarz(void* cv, double* Q) {
  Ctx* C = static_cast<Ctx*>(cv);
  try {
    compute_q(*C);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
  std::memcpy(Q, C->Q.data(), C->Q.size() * sizeof(double));
  return 0;
}

// Use an externally supplied Q (shared-Q identity checks, SURVEY.md §7 open
// decision 1).
void ref_set_schwarz(void* cv, const double* Q) {
  Ctx* C = static_cast<Ctx*>(cv);
  C->Q.assign(Q, Q + C->pairs.size());
  C->have_q = true;
}

// Canonical screened quartets (x <= y, pair-store indices), block order.
// Returns the count; writes at most cap entries.
long long ref_quartets(void* cv, double tau, int* xs, int* ys, long long cap) {
  Ctx* C = static_cast<Ctx*>(cv);
  if (tau > 0.0) compute_q(*C);
  long long n = 0;
  for (const auto& blk : C->blocks)
    for_each_quartet_in_block(*C, blk, tau, [&](int x, int y) {
      if (n < cap) { xs[n] = x; ys[n] = y; }
      ++n;
    });
  return n;
}

// Scaled integrals of one quartet, a-major over (i, j, k, l) components of
// pair x = (i,j) and pair y = (k,l). Returns the value count.
int ref_eri_quartet(void* cv, int x, int y, double* out) {
  Ctx* C = static_cast<Ctx*>(cv);
  try {
    Scratch S;
    quartet_scaled(*C, x, y, S);
    std::memcpy(out, S.v.data(), S.v.size() * sizeof(double));
    return static_cast<int>(S.v.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_build_jk(void* cv, const double* D, double tau, int nthreads, double* J, double* K,
                 long long* nq) {
  try {
    return build_jk_impl(*static_cast<Ctx*>(cv), D, tau, nthreads, 1, 0, J, K, nq);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Bounded CPU-baseline sample: only blocks with index % stride == offset.
int ref_build_jk_sample(void* cv, const double* D, double tau, int nthreads, long long stride,
                        long long offset, double* J, double* K, long long* nq) {
  try {
    return build_jk_impl(*static_cast<Ctx*>(cv), D, tau, nthreads, stride, offset, J, K, nq);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_build_jk_timed(void* cv, const double* D, double tau, int nthreads, long long stride,
                       long long offset, double* J, double* K, long long* nq, double* seconds) {
  try {
    return build_jk_impl(*static_cast<Ctx*>(cv), D, tau, nthreads, stride, offset, J, K, nq, seconds);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Per pair x: canonical survivors (x, y >= x) in block order (block.hpp:
// 135-150) and the wrapping sum of splitmix64(y) over them - list identity at
// sizes too large to export. Returns the total.
long long ref_pair_survivors(void* cv, double tau, long long* count, unsigned long long* ysum) {
  Ctx* C = static_cast<Ctx*>(cv);
  try {
    if (tau > 0.0) compute_q(*C);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
  const std::size_t np = C->pairs.size();
  const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
  std::vector<std::vector<long long>> cn(nt, std::vector<long long>(np, 0));
  std::vector<std::vector<unsigned long long>> hs(nt, std::vector<unsigned long long>(np, 0));
  auto mix = [](unsigned long long z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  };
  std::atomic<long long> next{0};
  const long long nb = static_cast<long long>(C->blocks.size());
  std::vector<std::thread> th;
  for (unsigned w = 0; w < nt; ++w)
    th.emplace_back([&, w] {
      for (long long bi; (bi = next.fetch_add(1)) < nb;)
        for_each_quartet_in_block(*C, C->blocks[bi], tau, [&](int x, int y) {
          ++cn[w][x];
          hs[w][x] += mix(static_cast<unsigned long long>(y));
        });
    });
  for (auto& t : th) t.join();
  long long total = 0;
  for (std::size_t x = 0; x < np; ++x) {
    long long c = 0;
    unsigned long long h = 0;
    for (unsigned w = 0; w < nt; ++w) {
      c += cn[w][x];
      h += hs[w][x];
    }
    count[x] = c;
    ysum[x] = h;
    total += c;
  }
  return total;
}

void ref_boys(int m, double T, double* F) { boys_inplace(m, T, F); }

// Plan statistics of compile_class (compiler.hpp:124-129,303-307) plus the
// Appendix-A sizes: op_count, slot_count, node_count, reuse_count, primT,
// base loads, prim slots, contract entries, hrr terms, contracted slots,
// targets, max_m.
void ref_plan_stats(int la, int lb, int lc, int ld, double lambda, long long* out) {
  CompilerConfig cfg;
  cfg.lambda = lambda;
  ExecutionPlan P = compile_class(EriClass{la, lb, lc, ld}, cfg);
  long long primT = 0, base = 0, hrrT = 0;
  for (const auto& i : P.prim) {
    if (i.base_m >= 0) ++base; else primT += static_cast<long long>(i.terms.size());
  }
  for (const auto& i : P.hrr) hrrT += static_cast<long long>(i.terms.size());
  out[0] = P.stats.op_count; out[1] = P.stats.slot_count; out[2] = P.stats.node_count;
  out[3] = P.stats.reuse_count; out[4] = primT; out[5] = base; out[6] = P.prim_slot_count;
  out[7] = static_cast<long long>(P.contract.size()); out[8] = hrrT;
  out[9] = P.contracted_slot_count; out[10] = static_cast<long long>(P.targets.size());
  out[11] = P.max_m;
}

long long ref_random_plan_ops(int la, int lb, int lc, int ld, unsigned long long seed) {
  return compile_random_class(EriClass{la, lb, lc, ld}, seed).stats.op_count;
}

// emit_source (compiler.hpp:319-367) into buf; returns required length.
long long ref_emit_source(int la, int lb, int lc, int ld, char* buf, long long cap) {
  std::string s = emit_source(compile_class(EriClass{la, lb, lc, ld}));
  if (buf && cap > 0) {
    long long n = std::min<long long>(cap - 1, static_cast<long long>(s.size()));
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return static_cast<long long>(s.size());
}

}  // extern "C"
