// Drop-in boundary check (TEST INFRASTRUCTURE ONLY; built by oracle/Makefile
// "driver" into oracle/_ref/ref_driver because it needs the reference
// headers). An SCF-driver-like caller holding the reference's own objects -
// Molecule/attach_basis, build_pairs, tile_pairs, make_blocks and a
// compile_class plan per class (the UNMODIFIED /root/reference/proj/include
// headers + oracle/shim) - calls the GPU executor of
// include/eritile/executor_ref.hpp exactly as SPEC.md:334-343 specifies
// build_g, in both reduction modes.
//
//   ref_driver <xyz file> <basis file> <kappa screen> <out.bin>
// out.bin: int64 N, then D, G(concurrent), G(deterministic, run 1),
// G(deterministic, run 2), each N*N doubles row-major. Prints "errors ok"
// when the error paths raise the reference's exception kinds.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>

#include "eritile/basis_set.hpp"
#include "eritile/block.hpp"
#include "eritile/compiler.hpp"
#include "eritile/molecule.hpp"
#include "eritile/executor_ref.hpp"

static std::string slurp(const char* path) {
  std::ifstream f(path);
  std::stringstream s;
  s << f.rdbuf();
  return s.str();
}

int main(int argc, char** argv) {
  if (argc != 5) {
    std::fprintf(stderr, "usage: ref_driver xyz basis kappa out.bin\n");
    return 2;
  }
  using namespace eritile;
  Molecule mol = parse_xyz(slurp(argv[1]));
  attach_basis(mol, BasisSetTable::parse(slurp(argv[2])));
  const double kappa = std::atof(argv[3]);
  const std::vector<ShellPair> pairs = build_pairs(mol.shells, kappa);
  const std::vector<PairTile> tiles = tile_pairs(pairs, 32);
  const std::vector<QuadBlock> blocks = make_blocks(tiles);
  std::map<EriClass, ExecutionPlan> plans;
  for (const QuadBlock& b : blocks)
    if (!plans.count(b.cls)) plans.emplace(b.cls, compile_class(b.cls));

  gpu::Executor ex(mol, pairs, kappa);
  const int N = ex.nbf();
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd(0.0, 1.0);
  std::vector<double> D(static_cast<size_t>(N) * N);
  for (int a = 0; a < N; ++a)
    for (int b = 0; b <= a; ++b) D[static_cast<size_t>(a) * N + b] = D[static_cast<size_t>(b) * N + a] = nd(rng) / std::sqrt(N);

  std::vector<double> Gc = ex.build_g(tiles, blocks, plans, D, gpu::ReduceMode::concurrent);
  std::vector<double> Gd1 = ex.build_g(tiles, blocks, plans, D, gpu::ReduceMode::deterministic);
  std::vector<double> Gd2 = ex.build_g(tiles, blocks, plans, D, gpu::ReduceMode::deterministic);

  std::ofstream out(argv[4], std::ios::binary);
  const long long n64 = N;
  out.write(reinterpret_cast<const char*>(&n64), sizeof n64);
  for (const std::vector<double>* v : {&D, &Gc, &Gd1, &Gd2}) out.write(reinterpret_cast<const char*>(v->data()), 8 * v->size());

  // error paths (SPEC.md:331,339 and the block-list contract of executor_ref.hpp)
  int ok = 0;
  try {
    std::vector<QuadBlock> sub(blocks.begin(), blocks.end() - 1);
    ex.build_g(tiles, sub, plans, D, gpu::ReduceMode::concurrent);
  } catch (const std::invalid_argument&) {
    ++ok;
  }
  try {
    auto p2 = plans;
    p2.erase(p2.begin());
    ex.build_g(tiles, blocks, p2, D, gpu::ReduceMode::concurrent);
  } catch (const std::invalid_argument&) {
    ++ok;
  }
  try {
    std::vector<double> bad(3, 0.0);
    ex.build_g(tiles, blocks, plans, bad, gpu::ReduceMode::concurrent);
  } catch (const std::invalid_argument&) {
    ++ok;
  }
  try {
    std::vector<ShellPair> p3(pairs.begin(), pairs.end() - 1);
    gpu::Executor bad(mol, p3, kappa);
  } catch (const std::invalid_argument&) {
    ++ok;
  }
  if (ok == 4) std::cout << "errors ok" << std::endl;
  std::cout << "N " << N << " pairs " << pairs.size() << " blocks " << blocks.size() << " classes " << plans.size()
            << std::endl;
  return 0;
}
