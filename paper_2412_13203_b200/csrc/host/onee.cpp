// One-electron integrals by Obara-Saika recurrences (host, multithreaded).
// Overlap/kinetic: 1-D OS overlap recursion and the kinetic relation
// T = -1/2 <a|d2/dx2|b>. Nuclear attraction: OS vertical recursion on the
// bra with auxiliary index m from [0|0]^(m) = 2 pi/p kappa F_m(p|PC|^2),
// then horizontal transfer to the ket. (The oracle uses McMurchie-Davidson,
// an independent route, for the same matrices.)
#include "onee.h"

#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

namespace eritile_b200 {

// Boys F_0..F_m(T): series at m_max + downward recursion for moderate T,
// closed form + upward recursion for large T (same split as boys.hpp:27-43).
void host_boys(int m_max, double T, double* F) {
  const double e = std::exp(-T);
  if (T < 35.0 || 2 * m_max + 1 >= T) {
    double term = 1.0 / (2 * m_max + 1), sum = term;
    for (int k = 0; k < 10000 && term > 1e-17 * sum; ++k) {
      term *= 2.0 * T / (2 * m_max + 2 * k + 3);
      sum += term;
    }
    F[m_max] = e * sum;
    for (int m = m_max; m > 0; --m) F[m - 1] = (2.0 * T * F[m] + e) / (2 * m - 1);
  } else {
    F[0] = 0.5 * std::sqrt(M_PI / T) * std::erf(std::sqrt(T));
    for (int m = 0; m < m_max; ++m) F[m + 1] = ((2 * m + 1) * F[m] - e) / (2.0 * T);
  }
}

namespace {
constexpr int LM = 2 * kMaxShellL + 3;

// 1-D overlap table s[i][j] for i <= la, j <= lb (without the sqrt(pi/p)
// and exp prefactors), OS: s[i+1][j] = PA s[i][j] + (i s[i-1][j] + j s[i][j-1])/(2p)
void overlap1d(int la, int lb, double PA, double PB, double p, double s[LM][LM]) {
  const double h = 0.5 / p;
  for (int i = 0; i <= la; ++i)
    for (int j = 0; j <= lb; ++j) {
      double v;
      if (i == 0 && j == 0) v = 1.0;
      else if (i > 0) {
        v = PA * s[i - 1][j];
        if (i > 1) v += h * (i - 1) * s[i - 2][j];
        if (j > 0) v += h * j * s[i - 1][j - 1];
      } else {
        v = PB * s[i][j - 1];
        if (j > 1) v += h * (j - 1) * s[i][j - 2];
      }
      s[i][j] = v;
    }
}

struct Idx3 {
  int n;
  int idx[LM][LM][LM];
  int mom[400][3];
};

void build_idx(int L, Idx3& t) {
  t.n = 0;
  for (int l = 0; l <= L; ++l)
    for (int ax = l; ax >= 0; --ax)
      for (int ay = l - ax; ay >= 0; --ay) {
        t.idx[ax][ay][l - ax - ay] = t.n;
        t.mom[t.n][0] = ax;
        t.mom[t.n][1] = ay;
        t.mom[t.n][2] = l - ax - ay;
        ++t.n;
      }
}
}  // namespace

void one_electron(const std::vector<ShellData>& shells, const std::vector<Atom>& atoms,
                  const std::vector<int>& bf_off, const std::vector<double>& bf_scale, double* S,
                  double* T, double* V) {
  const int ns = static_cast<int>(shells.size());
  const size_t N = static_cast<size_t>(bf_off.back());
  std::memset(S, 0, sizeof(double) * N * N);
  std::memset(T, 0, sizeof(double) * N * N);
  std::memset(V, 0, sizeof(double) * N * N);
  static Idx3 idx;
  static bool init = false;
  if (!init) {
    build_idx(2 * kMaxShellL, idx);
    init = true;
  }
  unsigned nt = std::max(1u, std::thread::hardware_concurrency());
  std::vector<std::thread> th;
  for (unsigned w = 0; w < nt; ++w)
    th.emplace_back([&, w] {
      std::vector<std::array<int, 3>> ca, cb;
      const int nab = idx.n;
      std::vector<double> vr;
      for (int s1 = static_cast<int>(w); s1 < ns; s1 += static_cast<int>(nt)) {
        const ShellData& A = shells[s1];
        cart_components(A.L, ca);
        for (int s2 = 0; s2 < ns; ++s2) {
          const ShellData& B = shells[s2];
          cart_components(B.L, cb);
          const int Lt = A.L + B.L;
          double AB[3];
          for (int d = 0; d < 3; ++d) AB[d] = A.c[d] - B.c[d];
          const double ab2 = AB[0] * AB[0] + AB[1] * AB[1] + AB[2] * AB[2];
          for (int k = 0; k < A.K(); ++k)
            for (int l = 0; l < B.K(); ++l) {
              const double a = A.exps[k], b = B.exps[l], p = a + b, mu = a * b / p;
              const double w8 = A.coefs[k] * B.coefs[l];
              double P[3], PA[3], PB[3];
              for (int d = 0; d < 3; ++d) {
                P[d] = (a * A.c[d] + b * B.c[d]) / p;
                PA[d] = P[d] - A.c[d];
                PB[d] = P[d] - B.c[d];
              }
              const double kap = std::exp(-mu * ab2);
              const double pre = std::pow(M_PI / p, 1.5) * kap * w8;
              double s1d[3][LM][LM];
              for (int d = 0; d < 3; ++d) overlap1d(A.L, B.L + 2, PA[d], PB[d], p, s1d[d]);
              for (size_t ia = 0; ia < ca.size(); ++ia)
                for (size_t ib = 0; ib < cb.size(); ++ib) {
                  double sv[3], tv[3];
                  for (int d = 0; d < 3; ++d) {
                    const int i = ca[ia][d], j = cb[ib][d];
                    sv[d] = s1d[d][i][j];
                    double t = 4.0 * b * b * s1d[d][i][j + 2] - 2.0 * b * (2 * j + 1) * s1d[d][i][j];
                    if (j >= 2) t += static_cast<double>(j * (j - 1)) * s1d[d][i][j - 2];
                    tv[d] = t;
                  }
                  const size_t mu_ = bf_off[s1] + ia, nu = bf_off[s2] + ib;
                  S[mu_ * N + nu] += pre * sv[0] * sv[1] * sv[2];
                  T[mu_ * N + nu] += -0.5 * pre * (tv[0] * sv[1] * sv[2] + sv[0] * tv[1] * sv[2] + sv[0] * sv[1] * tv[2]);
                }
              // nuclear attraction: OS VRR on e up to Lt, then HRR to (a|b)
              const int ne = (Lt + 1) * (Lt + 2) * (Lt + 3) / 6;
              vr.assign(static_cast<size_t>(ne) * (Lt + 1), 0.0);
              for (const Atom& at : atoms) {
                double PC[3];
                for (int d = 0; d < 3; ++d) PC[d] = P[d] - at.r[d];
                const double U = p * (PC[0] * PC[0] + PC[1] * PC[1] + PC[2] * PC[2]);
                double F[2 * kMaxShellL + 1];
                host_boys(Lt, U, F);
                const double base = 2.0 * M_PI / p * kap * w8 * -static_cast<double>(at.Z);
                auto R = [&](int e, int m) -> double& { return vr[static_cast<size_t>(e) * (Lt + 1) + m]; };
                for (int m = 0; m <= Lt; ++m) R(0, m) = base * F[m];
                for (int e = 1; e < ne; ++e) {
                  const int* em = idx.mom[e];
                  const int et = em[0] + em[1] + em[2];
                  const int i = em[0] ? 0 : (em[1] ? 1 : 2);
                  int q[3] = {em[0], em[1], em[2]};
                  q[i] -= 1;
                  const int e1 = idx.idx[q[0]][q[1]][q[2]];
                  int e2 = -1;
                  if (q[i] > 0) {
                    int r2[3] = {q[0], q[1], q[2]};
                    r2[i] -= 1;
                    e2 = idx.idx[r2[0]][r2[1]][r2[2]];
                  }
                  for (int m = 0; m <= Lt - et; ++m) {
                    double v = PA[i] * R(e1, m) - PC[i] * R(e1, m + 1);
                    if (e2 >= 0) v += q[i] * (0.5 / p) * (R(e2, m) - R(e2, m + 1));
                    R(e, m) = v;
                  }
                }
                // HRR (a|b+1_i) = (a+1_i|b) + AB_i (a|b) over m = 0 values
                for (size_t ia = 0; ia < ca.size(); ++ia)
                  for (size_t ib = 0; ib < cb.size(); ++ib) {
                    // expand b by binomial transfer: (a|b) = sum over splits
                    // of b along each axis: prod_d sum_k C(b_d,k) AB_d^(b_d-k) (a_d+k ...)
                    double acc = 0.0;
                    const int bx = cb[ib][0], by = cb[ib][1], bz = cb[ib][2];
                    for (int kx = 0; kx <= bx; ++kx)
                      for (int ky = 0; ky <= by; ++ky)
                        for (int kz = 0; kz <= bz; ++kz) {
                          const double c = std::tgamma(bx + 1.0) / (std::tgamma(kx + 1.0) * std::tgamma(bx - kx + 1.0)) *
                                           std::tgamma(by + 1.0) / (std::tgamma(ky + 1.0) * std::tgamma(by - ky + 1.0)) *
                                           std::tgamma(bz + 1.0) / (std::tgamma(kz + 1.0) * std::tgamma(bz - kz + 1.0)) *
                                           std::pow(AB[0], bx - kx) * std::pow(AB[1], by - ky) * std::pow(AB[2], bz - kz);
                          const int e = idx.idx[ca[ia][0] + kx][ca[ia][1] + ky][ca[ia][2] + kz];
                          acc += c * R(e, 0);
                        }
                    const size_t mu_ = bf_off[s1] + ia, nu = bf_off[s2] + ib;
                    V[mu_ * N + nu] += acc;
                  }
              }
            }
        }
      }
    });
  for (auto& t : th) t.join();
  for (size_t a = 0; a < N; ++a)
    for (size_t b = 0; b < N; ++b) {
      const double f = bf_scale[a] * bf_scale[b];
      S[a * N + b] *= f;
      T[a * N + b] *= f;
      V[a * N + b] *= f;
    }
}

}  // namespace eritile_b200
