// Product input layer types (host). See molecule.cpp.
#pragma once
#include <array>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace eritile_b200 {

constexpr double kAngstromToBohr = 1.8897259886;  // molecule.hpp:16
constexpr int kMaxShellL = 4;  // parser + one-electron bound; ERI classes: kMaxL (registry)

struct InputError : std::runtime_error {
  explicit InputError(const std::string& m) : std::runtime_error(m) {}
};

struct Atom {
  int Z = 0;
  double r[3] = {0, 0, 0};  // Bohr
};

struct BasisRecord {
  int L = 0;
  std::vector<double> exps, coefs;
};
using BasisTable = std::map<int, std::vector<BasisRecord>>;

// Contracted Cartesian shell with normalisation folded into coefs
// (Shell, molecule.hpp:39-50).
struct ShellData {
  double c[3] = {0, 0, 0};
  int L = 0, atom = -1;
  std::vector<double> exps, coefs;
  int K() const { return static_cast<int>(exps.size()); }
  int nfunc() const { return (L + 1) * (L + 2) / 2; }
};

int element_z(const std::string& sym);
std::vector<Atom> read_xyz(const std::string& text);
BasisTable read_basis(const std::string& text);
std::vector<ShellData> attach_basis(const std::vector<Atom>& atoms, const BasisTable& tab);
double odd_double_factorial(int n);
void cart_components(int L, std::vector<std::array<int, 3>>& out);
double component_scale(int ax, int ay, int az);

}  // namespace eritile_b200
