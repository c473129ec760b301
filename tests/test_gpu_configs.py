"""GPU parity at the BASELINE.json configurations, with the bench's settings
(kappa screen 1e-14, Schwarz tau 1e-10; bench.py):

* C3 (H2O)_16/cc-pVDZ (N = 400): full J/K within 1e-10 of the CPU path at the
  converged SCF density, per-pair screened-list identity, and the SCF energy
  within 1e-8 Ha of the CPU path's SCF;
* C4 (H2O)_64/cc-pVDZ (N = 1600) and the headline (H2O)_80/cc-pVDZ
  (N = 2000): screened-list identity against the unmodified reference pair
  store (oracle/_ref) through per-pair survivor counts and hashes (the lists
  hold 1.7e9 / 2.6e9 quartets, too many to export), and, at the headline,
  J/K within 1e-10 for a density supported on one water (the CPU checker
  skips quartets whose six density blocks are zero, which contribute exactly
  zero, so every quartet that can change J or K is compared).

The full headline J/K against a complete CPU build is recorded once by
tools/headline_parity.py (about 10 minutes of CPU) in
profiles/r02_headline_parity.json: max |dJ| 4.8e-13, max |dK| 1.5e-14.
"""
import numpy as np
import pytest

from oracle_lib import Oracle, available
from systems import BASIS, geom

pytestmark = pytest.mark.gpu

KAPPA, TAU = 1e-14, 1e-10


def _engine(mol, basis="cc-pvdz"):
    from paper_2412_13203_b200.eritile import Engine
    e = Engine(0).load_molecule(geom(mol), BASIS[basis]).build_pairs(KAPPA)
    e.set_screening(TAU)
    return e


def _survivor_identity(e, O):
    c_g, h_g, t_g = e.pair_survivors()
    c_o, h_o, t_o = O.pair_survivors(TAU)
    bad = np.flatnonzero((c_g != c_o) | (h_g != h_o))
    assert t_g == t_o and bad.size == 0, (t_g, t_o, bad[:10], c_g[bad[:10]], c_o[bad[:10]])
    return t_g


def test_c3_w16_jk_list_and_scf(gpu):
    """C3: SCF on the GPU, then at its converged density D: one CPU build
    gives J/K (1e-10) and E(D) (1e-8); one more CPU Roothaan step from D
    stays within 1e-8 Ha. The SCF energy is stationary, so an energy that is
    unchanged by a CPU-path Fock step is the CPU path's SCF energy; the
    orbital gradient bound makes that explicit (error is quadratic in it)."""
    from paper_2412_13203_b200.scf import density_from_mos, orthogonalizer, run_rhf
    e = _engine("w16")
    O = Oracle("orc").system(geom("w16"), BASIS["cc-pvdz"], kappa_screen=KAPPA)
    assert e.npairs == O.npairs
    nq = _survivor_identity(e, O)
    assert nq == e.num_quartets()

    g = run_rhf(geom("w16"), BASIS["cc-pvdz"], tau=TAU, kappa_screen=KAPPA, conv=1e-9, e_conv=1e-12)
    assert g.converged
    D = g.density
    J, K = e.build_jk(D)
    Jo, Ko, nqo = O.build_jk(D, TAU)
    assert nqo == nq
    assert np.max(np.abs(J - Jo)) < 1e-10 and np.max(np.abs(K - Ko)) < 1e-10

    S, T, V = O.one_electron()
    H = T + V
    enuc = O.nuclear_repulsion()
    Fo = H + 2.0 * Jo - Ko
    Eo = float(np.sum(D * (H + Fo)) + enuc)
    assert abs(Eo - g.energy) < 1e-8, (Eo, g.energy)
    X = orthogonalizer(S)
    grad = X.T @ (Fo @ D @ S - S @ D @ Fo) @ X
    assert np.max(np.abs(grad)) < 1e-5
    _, Cp = np.linalg.eigh(X.T @ Fo @ X)
    D1 = density_from_mos(X @ Cp, O.nelectrons // 2)
    J1, K1, _ = O.build_jk(D1, TAU)
    E1 = float(np.sum(D1 * (2.0 * H + 2.0 * J1 - K1)) + enuc)
    assert abs(E1 - g.energy) < 1e-8, (E1, g.energy)


@pytest.mark.parametrize("waters", [64, 80])
def test_large_list_identity(gpu, waters):
    """C4 and the headline: identical screened lists (per-pair survivor
    count and y-hash) against the unmodified reference pair store, with the
    GPU's Schwarz Q on one side and the CPU reference's on the other."""
    kind = "ref" if available("ref") else "orc"
    e = _engine(f"w{waters}")
    O = Oracle(kind).system(geom(f"w{waters}"), BASIS["cc-pvdz"], kappa_screen=KAPPA)
    assert e.npairs == O.npairs
    nq = _survivor_identity(e, O)
    assert nq == e.num_quartets()


def test_headline_jk_sparse_density(gpu):
    """Headline (H2O)_80: J/K within 1e-10 of the CPU path for a density
    supported on the shells of the central water (all quartets that can
    contribute are evaluated on both sides)."""
    e = _engine("w80")
    O = Oracle("orc").system(geom("w80"), BASIS["cc-pvdz"], kappa_screen=KAPPA)
    N = e.nbf
    sh = O.shells()
    Z, pos = O.atoms()
    centre = pos.mean(axis=0)
    w = int(np.argmin([np.linalg.norm(pos[3 * k] - centre) for k in range(len(Z) // 3)]))
    mask = np.zeros(N, bool)
    for s, a in enumerate(sh["atom"]):
        if a // 3 == w:
            n = (sh["L"][s] + 1) * (sh["L"][s] + 2) // 2
            mask[sh["bf_off"][s]:sh["bf_off"][s] + n] = True
    rng = np.random.default_rng(80)
    A = rng.standard_normal((N, N))
    D = (A + A.T) * np.outer(mask, mask)
    J, K = e.build_jk(D)
    Jo, Ko, nq = O.build_jk_dsparse(D, TAU)
    assert nq > 0
    assert np.max(np.abs(J - Jo)) < 1e-10 and np.max(np.abs(K - Ko)) < 1e-10
