"""Config 5 (BASELINE.json configs[4]: alanine oligomer / taxol-sized, cc-pVTZ,
f shells, the high-L Deconstruction path) on an idealised H-(Ala)_n-OH strand
(geometry.alanine_chain; taxol coordinates are not available
offline). Bench settings: kappa screen 1e-14, Schwarz tau 1e-10.

* (Ala)_1 / cc-pVTZ (N = 315, L <= 3 on C/N/O): screened-list identity
  against the unmodified reference pair store, full J/K within 1e-10 of the
  CPU reference at the GPU SCF's converged density, and E(D) within 1e-8 Ha.
* (Ala)_2 / cc-pVTZ (N = 565): list identity, and J/K within 1e-10 for a
  density supported on the second residue (the CPU checker skips quartets
  whose six density blocks vanish: every quartet that can change J or K is
  compared).
"""
import numpy as np
import pytest

from oracle_lib import Oracle, available
from systems import BASIS, geom

pytestmark = pytest.mark.gpu

KAPPA, TAU = 1e-14, 1e-10


def _engine(mol):
    from paper_2412_13203_b200.eritile import Engine
    e = Engine(0).load_molecule(geom(mol), BASIS["cc-pvtz"]).build_pairs(KAPPA)
    e.set_screening(TAU)
    return e


def _survivor_identity(e, O):
    c_g, h_g, t_g = e.pair_survivors()
    c_o, h_o, t_o = O.pair_survivors(TAU)
    bad = np.flatnonzero((c_g != c_o) | (h_g != h_o))
    assert t_g == t_o and bad.size == 0, (t_g, t_o, bad[:10])
    return t_g


def test_ala1_cctz_list_jk_energy(gpu):
    from paper_2412_13203_b200.scf import run_rhf
    kind = "ref" if available("ref") else "orc"
    e = _engine("ala1")
    O = Oracle(kind).system(geom("ala1"), BASIS["cc-pvtz"], kappa_screen=KAPPA)
    assert e.npairs == O.npairs and e.nbf == O.nbf == 315
    nq = _survivor_identity(e, O)
    assert nq == e.num_quartets()
    g = run_rhf(geom("ala1"), BASIS["cc-pvtz"], tau=TAU, kappa_screen=KAPPA, conv=1e-8, e_conv=1e-11)
    assert g.converged
    D = g.density
    J, K = e.build_jk(D)
    Jo, Ko, nqo = O.build_jk(D, TAU)
    assert nqo == nq
    assert np.max(np.abs(J - Jo)) < 1e-10 and np.max(np.abs(K - Ko)) < 1e-10
    O1 = Oracle("orc").system(geom("ala1"), BASIS["cc-pvtz"], kappa_screen=KAPPA)
    S, T, V = O1.one_electron()
    H = T + V
    Eo = float(np.sum(D * (2.0 * H + 2.0 * Jo - Ko)) + O1.nuclear_repulsion())
    assert abs(Eo - g.energy) < 1e-8, (Eo, g.energy)


def test_ala2_cctz_list_and_residue_density_jk(gpu):
    e = _engine("ala2")
    kind = "ref" if available("ref") else "orc"
    Oref = Oracle(kind).system(geom("ala2"), BASIS["cc-pvtz"], kappa_screen=KAPPA)
    assert e.npairs == Oref.npairs
    assert _survivor_identity(e, Oref) == e.num_quartets()
    O = Oracle("orc").system(geom("ala2"), BASIS["cc-pvtz"], kappa_screen=KAPPA)
    N = e.nbf
    sh = O.shells()
    # residue 2 = atoms 11 .. 22 of H-(Ala)_2-OH (residue 1 carries the NH2 cap, residue 2 the OH)
    mask = np.zeros(N, bool)
    for s, a in enumerate(sh["atom"]):
        if a >= 11:
            n = (sh["L"][s] + 1) * (sh["L"][s] + 2) // 2
            mask[sh["bf_off"][s]:sh["bf_off"][s] + n] = True
    rng = np.random.default_rng(2)
    A = rng.standard_normal((N, N))
    D = (A + A.T) * np.outer(mask, mask)
    J, K = e.build_jk(D)
    Jo, Ko, nq = O.build_jk_dsparse(D, TAU)
    assert nq > 0
    assert np.max(np.abs(J - Jo)) < 1e-10 and np.max(np.abs(K - Ko)) < 1e-10
