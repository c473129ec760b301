// eritile/executor.hpp — C++ face of the B200 Fock-build engine.
//
// The reference library (proj/include/eritile, arxiv 2412.13203) specifies an
// executor it does not ship:
//   eval_block(QuadBlock, ExecutionPlan, D, Accumulator&)
//   build_g(blocks, plans, D, mode) -> G
// with exceptions for errors (ParseError molecule.hpp:72-74,
// std::invalid_argument block.hpp:55,118, std::domain_error boys.hpp:48-50).
// This header keeps that calling convention for an SCF driver — build_g(D)
// returns G = 2J - K, build_jk(D) the true J and K — over the C ABI in
// eritile_gpu.h (no torch types, plain pointers). Header-only; link
// liberitile_b200.so. Matrices are row-major N x N std::vector<double>.
#pragma once

#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../eritile_gpu.h"

namespace eritile {

// Same role as eritile::ParseError (molecule.hpp:72-74).
struct GpuParseError : std::runtime_error {
  explicit GpuParseError(const std::string& w) : std::runtime_error(w) {}
};

class GpuExecutor {
 public:
  explicit GpuExecutor(int device = 0) {
    if (eritile_gpu_create(device, &ctx_) != ERITILE_OK)
      throw std::runtime_error(std::string("eritile_gpu_create: ") + eritile_gpu_last_error(nullptr));
  }
  ~GpuExecutor() { eritile_gpu_destroy(ctx_); }
  GpuExecutor(const GpuExecutor&) = delete;
  GpuExecutor& operator=(const GpuExecutor&) = delete;

  // parse_xyz + BasisSetTable::parse + attach_basis
  void load_molecule(const std::string& xyz, const std::string& basis) {
    check(eritile_gpu_load_molecule(ctx_, xyz.c_str(), basis.c_str()));
  }
  // build_pairs (block.hpp:52): screen_threshold is the kappa screen.
  void build_pairs(double screen_threshold = 0.0) { check(eritile_gpu_build_pairs(ctx_, screen_threshold)); }
  std::vector<double> schwarz() {
    std::vector<double> q(static_cast<size_t>(eritile_gpu_npairs(ctx_)));
    check(eritile_gpu_schwarz(ctx_, q.data()));
    return q;
  }
  void set_shard(int rank, int nranks) { check(eritile_gpu_set_shard(ctx_, rank, nranks)); }
  // Workload Allocator: fastest kernel variant per class on D.
  void tune(const std::vector<double>& D, int reps = 2) { check(eritile_gpu_tune(ctx_, D.data(), reps)); }
  void set_screening(double tau) { check(eritile_gpu_set_screening(ctx_, tau)); }
  int nbf() const { return eritile_gpu_nbf(ctx_); }

  // True J and K for a symmetric density.
  std::pair<std::vector<double>, std::vector<double>> build_jk(const std::vector<double>& D) {
    const size_t NN = static_cast<size_t>(nbf()) * nbf();
    if (D.size() != NN) throw std::invalid_argument("build_jk: density must be N x N");
    std::vector<double> J(NN), K(NN);
    check(eritile_gpu_build_jk(ctx_, D.data(), J.data(), K.data()));
    return {std::move(J), std::move(K)};
  }
  // G = 2J - K (closed-shell RHF).
  std::vector<double> build_g(const std::vector<double>& D) {
    auto jk = build_jk(D);
    std::vector<double> G(jk.first.size());
    for (size_t e = 0; e < G.size(); ++e) G[e] = 2.0 * jk.first[e] - jk.second[e];
    return G;
  }
  eritile_gpu* handle() { return ctx_; }

 private:
  void check(int rc) const {
    if (rc == ERITILE_OK) return;
    const std::string m = eritile_gpu_last_error(ctx_);
    switch (rc) {
      case ERITILE_ERR_PARSE: throw GpuParseError(m);
      case ERITILE_ERR_ARG: throw std::invalid_argument(m);
      case ERITILE_ERR_DOMAIN: throw std::domain_error(m);
      default: throw std::runtime_error(m);
    }
  }
  eritile_gpu* ctx_ = nullptr;
};

// Free-function spelling of the SPEC executor entry points.
inline std::pair<std::vector<double>, std::vector<double>> build_jk(GpuExecutor& ex, const std::vector<double>& D) {
  return ex.build_jk(D);
}
inline std::vector<double> build_g(GpuExecutor& ex, const std::vector<double>& D) { return ex.build_g(D); }

}  // namespace eritile
