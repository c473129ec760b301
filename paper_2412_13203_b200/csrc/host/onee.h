// One-electron integrals S, T, V for the SCF harness.
#pragma once
#include <vector>

#include "molecule.h"

namespace eritile_b200 {
void one_electron(const std::vector<ShellData>& shells, const std::vector<Atom>& atoms,
                  const std::vector<int>& bf_off, const std::vector<double>& bf_scale, double* S,
                  double* T, double* V);
void host_boys(int m_max, double T, double* F);
}  // namespace eritile_b200
