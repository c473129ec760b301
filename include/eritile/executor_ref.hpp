// eritile/executor_ref.hpp — the SPEC executor over the reference's own types.
//
// The reference library (proj/include/eritile, arxiv 2412.13203) ships the
// block constructor and plan compiler but not the executor its SPEC defines:
//   build_g(blocks, plans, D, mode) -> G
//   Accumulator modes concurrent | deterministic
// This header is that executor for a caller that already holds the
// reference's objects — Molecule after attach_basis (basis_set.hpp:127-155),
// std::vector<ShellPair> from build_pairs (block.hpp:52-103), PairTile from
// tile_pairs (block.hpp:115-131), QuadBlock from make_blocks (block.hpp:
// 135-150) and the ExecutionPlan per EriClass from compile_class
// (compiler.hpp:193-307) — and runs the Fock build on the B200 engine
// through the C ABI (eritile_gpu.h). It is a drop-in for the SCF driver's
// call: same arguments, G = 2J - K back, reference
// exception kinds on error.
//
// Include it after putting the reference's include directory on the path
// (it includes "eritile/block.hpp", "eritile/compiler.hpp",
// "eritile/molecule.hpp"); link liberitile_b200.so.
//
// What is checked, and why:
//  * the GPU pair store is rebuilt from the same shells with the same kappa
//    screen and must equal `pairs` (shell pairs in order, kept primitive
//    counts) - std::invalid_argument otherwise;
//  * `blocks` must be the complete canonical block list of `tiles` (any
//    order): the GPU engine evaluates the canonical quartet set x <= y
//    (Schwarz-screened when tau > 0) in its own class/contraction order
//    (Permutation), not an arbitrary block subset;
//  * every block class needs a plan whose class matches (SPEC.md:331
//    "class mismatch -> error", :339 "missing plan -> error"). The kernels
//    are generated offline from compile_class plans of the same classes
//    (tests/test_compiler.py checks the plans equal the reference's).
#pragma once

#include <algorithm>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "eritile/block.hpp"
#include "eritile/compiler.hpp"
#include "eritile/molecule.hpp"
#include "eritile_gpu.h"

namespace eritile {
namespace gpu {

// SPEC.md Accumulator reduction modes.
enum class ReduceMode { concurrent, deterministic };

class Executor {
 public:
  // `pairs` must come from build_pairs(mol.shells, screen_threshold).
  // tau > 0 adds Schwarz screening (Q_x Q_y >= tau; not in the reference,
  // SURVEY.md 8a-3), tau = 0 evaluates every canonical quartet as the
  // reference's build_g does.
  Executor(const Molecule& mol, const std::vector<ShellPair>& pairs, double screen_threshold = 0.0,
           double tau = 0.0, int device = 0)
      : tau_(tau) {
    if (eritile_gpu_create(device, &ctx_) != ERITILE_OK)
      throw std::runtime_error(std::string("eritile_gpu_create: ") + eritile_gpu_last_error(nullptr));
    const int S = static_cast<int>(mol.shells.size());
    std::vector<int> L(S), K(S), atom(S);
    std::vector<double> centre(3 * static_cast<size_t>(S)), ex, co;
    for (int s = 0; s < S; ++s) {
      const Shell& sh = mol.shells[s];
      L[s] = sh.total_momentum;
      K[s] = sh.contraction_degree();
      atom[s] = sh.atom;
      for (int d = 0; d < 3; ++d) centre[3 * s + d] = sh.center[d];
      ex.insert(ex.end(), sh.exponents.begin(), sh.exponents.end());
      co.insert(co.end(), sh.coefficients.begin(), sh.coefficients.end());
    }
    const int A = static_cast<int>(mol.atoms.size());
    std::vector<int> Z(A);
    std::vector<double> pos(3 * static_cast<size_t>(A));
    for (int a = 0; a < A; ++a) {
      Z[a] = mol.atoms[a].atomic_number;
      for (int d = 0; d < 3; ++d) pos[3 * a + d] = mol.atoms[a].position[d];
    }
    check(eritile_gpu_load_shells(ctx_, S, L.data(), K.data(), centre.data(), atom.data(), ex.data(), co.data(), A,
                                  Z.data(), pos.data()));
    check(eritile_gpu_build_pairs(ctx_, screen_threshold));
    const int np = eritile_gpu_npairs(ctx_);
    if (np != static_cast<int>(pairs.size()))
      throw std::invalid_argument("executor: pair store differs from build_pairs(shells, screen_threshold) (" +
                                  std::to_string(np) + " vs " + std::to_string(pairs.size()) + " pairs)");
    std::vector<int> pi(np), pj(np), npr(np);
    check(eritile_gpu_pair_shells(ctx_, pi.data(), pj.data()));
    check(eritile_gpu_pair_nprims(ctx_, npr.data()));
    for (int x = 0; x < np; ++x)
      if (pi[x] != pairs[x].i || pj[x] != pairs[x].j || npr[x] != static_cast<int>(pairs[x].prims.size()))
        throw std::invalid_argument("executor: pair " + std::to_string(x) +
                                    " differs from the reference pair store (order or kept primitives)");
    check(eritile_gpu_set_screening(ctx_, tau_));
    nbf_ = eritile_gpu_nbf(ctx_);
  }
  ~Executor() { eritile_gpu_destroy(ctx_); }
  Executor(const Executor&) = delete;
  Executor& operator=(const Executor&) = delete;

  // True J and K (SURVEY.md Appendix C convention).
  std::pair<std::vector<double>, std::vector<double>> build_jk(const std::vector<PairTile>& tiles,
                                                               const std::vector<QuadBlock>& blocks,
                                                               const std::map<EriClass, ExecutionPlan>& plans,
                                                               const std::vector<double>& D, ReduceMode mode) {
    validate(tiles, blocks, plans);
    const size_t NN = static_cast<size_t>(nbf_) * nbf_;
    if (D.size() != NN) throw std::invalid_argument("build_g: density must be N x N (row-major)");
    check(eritile_gpu_set_mode(ctx_, mode == ReduceMode::deterministic ? ERITILE_MODE_DETERMINISTIC
                                                                        : ERITILE_MODE_CONCURRENT));
    std::vector<double> J(NN), K(NN);
    check(eritile_gpu_build_jk(ctx_, D.data(), J.data(), K.data()));
    return {std::move(J), std::move(K)};
  }

  // G = 2J - K for restricted HF.
  std::vector<double> build_g(const std::vector<PairTile>& tiles, const std::vector<QuadBlock>& blocks,
                              const std::map<EriClass, ExecutionPlan>& plans, const std::vector<double>& D,
                              ReduceMode mode) {
    auto jk = build_jk(tiles, blocks, plans, D, mode);
    std::vector<double> G(jk.first.size());
    for (size_t e = 0; e < G.size(); ++e) G[e] = 2.0 * jk.first[e] - jk.second[e];
    return G;
  }

  int nbf() const { return nbf_; }
  eritile_gpu* handle() { return ctx_; }

 private:
  void validate(const std::vector<PairTile>& tiles, const std::vector<QuadBlock>& blocks,
                const std::map<EriClass, ExecutionPlan>& plans) const {
    // tiles: consecutive same-class runs covering the pair store (block.hpp:115-131)
    int next = 0;
    for (const PairTile& t : tiles) {
      if (t.first != next || t.count <= 0) throw std::invalid_argument("build_g: tiles do not cover the pair store");
      next += t.count;
    }
    if (next != eritile_gpu_npairs(ctx_)) throw std::invalid_argument("build_g: tiles do not cover the pair store");
    // blocks: exactly the tile pairs ti <= tj (block.hpp:135-150), each once
    const long long nt = static_cast<long long>(tiles.size());
    if (static_cast<long long>(blocks.size()) != nt * (nt + 1) / 2)
      throw std::invalid_argument("build_g: the GPU executor evaluates the complete canonical block list; got " +
                                  std::to_string(blocks.size()) + " of " + std::to_string(nt * (nt + 1) / 2));
    std::set<std::pair<int, int>> seen;
    for (const QuadBlock& b : blocks) {
      if (b.bra_tile < 0 || b.ket_tile < b.bra_tile || b.ket_tile >= nt || !seen.emplace(b.bra_tile, b.ket_tile).second)
        throw std::invalid_argument("build_g: blocks are not the canonical tile pairs");
      const PairTile& ti = tiles[b.bra_tile];
      const PairTile& tj = tiles[b.ket_tile];
      const EriClass c{ti.cls.li, ti.cls.lj, tj.cls.li, tj.cls.lj};
      if (!(b.cls == c)) throw std::invalid_argument("build_g: block class does not match its tiles");
      const auto it = plans.find(c);
      if (it == plans.end()) throw std::invalid_argument("build_g: missing plan for class " + to_string(c));
      const ExecutionPlan& P = it->second;
      const size_t nv = static_cast<size_t>((c.la + 1) * (c.la + 2) / 2) * ((c.lb + 1) * (c.lb + 2) / 2) *
                        ((c.lc + 1) * (c.lc + 2) / 2) * ((c.ld + 1) * (c.ld + 2) / 2);
      if (!(P.cls == c) || P.targets.size() != nv || P.max_m != c.la + c.lb + c.lc + c.ld)
        throw std::invalid_argument("build_g: plan class mismatch for " + to_string(c));
    }
  }
  void check(int rc) const {
    if (rc == ERITILE_OK) return;
    const std::string m = eritile_gpu_last_error(ctx_);
    switch (rc) {
      case ERITILE_ERR_PARSE: throw ParseError(m);
      case ERITILE_ERR_ARG: throw std::invalid_argument(m);
      case ERITILE_ERR_DOMAIN: throw std::domain_error(m);
      default: throw std::runtime_error(m);
    }
  }
  eritile_gpu* ctx_ = nullptr;
  double tau_ = 0.0;
  int nbf_ = 0;
};

// Free-function form of SPEC.md:334 for a one-off build (an SCF driver
// keeps an Executor across iterations instead: pairs and lists are built
// once per geometry).
inline std::vector<double> build_g(const Molecule& mol, const std::vector<ShellPair>& pairs,
                                   const std::vector<PairTile>& tiles, const std::vector<QuadBlock>& blocks,
                                   const std::map<EriClass, ExecutionPlan>& plans, const std::vector<double>& D,
                                   ReduceMode mode, double screen_threshold = 0.0, int device = 0) {
  Executor ex(mol, pairs, screen_threshold, 0.0, device);
  return ex.build_g(tiles, blocks, plans, D, mode);
}

}  // namespace gpu
}  // namespace eritile
