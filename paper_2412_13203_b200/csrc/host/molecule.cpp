// Product input layer: XYZ geometry, basis-table text, normalisation.
// Restates the reference's input semantics (molecule.hpp:105-158 parse_xyz,
// basis_set.hpp:33-84 BasisSetTable::parse, basis_set.hpp:112-155
// attach_basis) so that shells and coefficients are bit-identical to the
// reference's for the same text (checked by tests/test_abi.py and
// tests/test_oracle_pins.py against the oracle and oracle/_ref).
#include "molecule.h"

#include <cctype>
#include <cmath>
#include <cstdlib>
#include <map>
#include <sstream>

namespace eritile_b200 {

namespace {
const char* kElements[36] = {"H",  "He", "Li", "Be", "B",  "C",  "N",  "O",  "F",
                             "Ne", "Na", "Mg", "Al", "Si", "P",  "S",  "Cl", "Ar",
                             "K",  "Ca", "Sc", "Ti", "V",  "Cr", "Mn", "Fe", "Co",
                             "Ni", "Cu", "Zn", "Ga", "Ge", "As", "Se", "Br", "Kr"};

std::string strip(const std::string& s) {
  size_t b = 0, e = s.size();
  while (b < e && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
  while (e > b && std::isspace(static_cast<unsigned char>(s[e - 1]))) --e;
  return s.substr(b, e - b);
}

double number(const std::string& tok, int line_no) {
  char* end = nullptr;
  double v = std::strtod(tok.c_str(), &end);
  if (tok.empty() || *end != 0)
    throw InputError("line " + std::to_string(line_no) + ": malformed number '" + tok + "'");
  if (!std::isfinite(v))
    throw InputError("line " + std::to_string(line_no) + ": non-finite value '" + tok + "'");
  return v;
}
}  // namespace

int element_z(const std::string& sym) {
  if (sym.empty()) return 0;
  std::string s = sym;
  s[0] = static_cast<char>(std::toupper(static_cast<unsigned char>(s[0])));
  for (size_t i = 1; i < s.size(); ++i) s[i] = static_cast<char>(std::tolower(static_cast<unsigned char>(s[i])));
  for (int z = 0; z < 36; ++z)
    if (s == kElements[z]) return z + 1;
  return 0;
}

std::vector<Atom> read_xyz(const std::string& text) {
  std::istringstream in(text);
  std::string line;
  int line_no = 0;
  if (!std::getline(in, line)) throw InputError("empty XYZ input");
  ++line_no;
  long declared = 0;
  {
    std::string t = strip(line);
    char* end = nullptr;
    declared = std::strtol(t.c_str(), &end, 10);
    if (t.empty() || end == t.c_str()) throw InputError("line 1: expected atom count, got '" + t + "'");
  }
  if (declared < 0) throw InputError("line 1: negative atom count");
  if (!std::getline(in, line)) throw InputError("unexpected end of file");
  ++line_no;
  std::vector<Atom> atoms;
  while (std::getline(in, line)) {
    ++line_no;
    std::string t = strip(line);
    if (t.empty()) continue;
    std::istringstream ls(t);
    std::string sym, xs, ys, zs;
    if (!(ls >> sym >> xs >> ys >> zs))
      throw InputError("line " + std::to_string(line_no) + ": expected 'symbol x y z', got '" + t + "'");
    int z = element_z(sym);
    if (!z) throw InputError("line " + std::to_string(line_no) + ": unknown element symbol '" + sym + "'");
    Atom a;
    a.Z = z;
    // Angstrom -> Bohr, element-wise product (molecule.hpp:147-151)
    a.r[0] = number(xs, line_no) * kAngstromToBohr;
    a.r[1] = number(ys, line_no) * kAngstromToBohr;
    a.r[2] = number(zs, line_no) * kAngstromToBohr;
    atoms.push_back(a);
  }
  if (static_cast<long>(atoms.size()) != declared)
    throw InputError("declared " + std::to_string(declared) + " atoms, found " + std::to_string(atoms.size()));
  return atoms;
}

BasisTable read_basis(const std::string& text) {
  BasisTable tab;
  std::istringstream in(text);
  std::string line;
  int line_no = 0, current = 0;
  auto fail = [&](const std::string& m) {
    throw InputError("basis table line " + std::to_string(line_no) + ": " + m);
  };
  while (std::getline(in, line)) {
    ++line_no;
    std::string t = strip(line);
    if (t.empty() || t[0] == '#') continue;
    std::istringstream ls(t);
    std::string head;
    ls >> head;
    if (head == "element") {
      std::string sym;
      if (!(ls >> sym)) fail("missing element symbol");
      current = element_z(sym);
      if (!current) fail("unknown element symbol '" + sym + "'");
      tab[current];
      continue;
    }
    if (!current) fail("shell block before any 'element' record");
    std::istringstream hs(t);
    int L = 0, K = 0;
    if (!(hs >> L >> K) || L < 0 || K < 1) fail("expected shell header 'L K', got '" + t + "'");
    if (L > kMaxShellL) fail("angular momentum above the compiled maximum");
    BasisRecord rec;
    rec.L = L;
    for (int k = 0; k < K; ++k) {
      if (!std::getline(in, line)) fail("unexpected end of shell block");
      ++line_no;
      std::istringstream rs(strip(line));
      std::string es, cs;
      if (!(rs >> es >> cs)) fail("expected 'exponent coefficient'");
      double e = number(es, line_no), c = number(cs, line_no);
      if (e <= 0.0) fail("exponent must be positive");
      rec.exps.push_back(e);
      rec.coefs.push_back(c);
    }
    tab[current].push_back(rec);
  }
  return tab;
}

double odd_double_factorial(int n) {
  double v = 1.0;
  for (int k = 2 * n - 1; k > 1; k -= 2) v *= k;
  return v;
}

// Self-overlap of two primitives with momentum (L,0,0) on one centre
// (basis_set.hpp:112-116); evaluation order kept for bit-identity.
static double prim_overlap(double a, double b, int L) {
  const double p = a + b;
  return std::pow(M_PI / p, 1.5) * odd_double_factorial(L) / std::pow(2.0 * p, L);
}

std::vector<ShellData> attach_basis(const std::vector<Atom>& atoms, const BasisTable& tab) {
  std::vector<ShellData> out;
  for (int ai = 0; ai < static_cast<int>(atoms.size()); ++ai) {
    auto it = tab.find(atoms[ai].Z);
    if (it == tab.end() || it->second.empty())
      throw InputError("basis table has no element '" + std::string(kElements[atoms[ai].Z - 1]) + "'");
    for (const BasisRecord& rec : it->second) {
      ShellData sh;
      for (int d = 0; d < 3; ++d) sh.c[d] = atoms[ai].r[d];
      sh.L = rec.L;
      sh.atom = ai;
      sh.exps = rec.exps;
      sh.coefs = rec.coefs;
      const int K = static_cast<int>(sh.exps.size());
      for (int k = 0; k < K; ++k) sh.coefs[k] *= 1.0 / std::sqrt(prim_overlap(sh.exps[k], sh.exps[k], sh.L));
      double self = 0.0;
      for (int k = 0; k < K; ++k)
        for (int l = 0; l < K; ++l) self += sh.coefs[k] * sh.coefs[l] * prim_overlap(sh.exps[k], sh.exps[l], sh.L);
      const double scale = 1.0 / std::sqrt(self);
      for (double& c : sh.coefs) c *= scale;
      out.push_back(std::move(sh));
    }
  }
  return out;
}

void cart_components(int L, std::vector<std::array<int, 3>>& out) {
  out.clear();
  for (int ax = L; ax >= 0; --ax)
    for (int ay = L - ax; ay >= 0; --ay) out.push_back({ax, ay, L - ax - ay});
}

double component_scale(int ax, int ay, int az) {
  const int L = ax + ay + az;
  if (L <= 1) return 1.0;
  return std::sqrt(odd_double_factorial(L) /
                   (odd_double_factorial(ax) * odd_double_factorial(ay) * odd_double_factorial(az)));
}

}  // namespace eritile_b200
