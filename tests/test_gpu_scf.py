"""SCF energy parity (north star: total SCF energy within 1e-8 Ha of the CPU
reference path on the same molecule and basis)."""
import pytest

from oracle_lib import Oracle
from systems import BASIS, geom

pytestmark = pytest.mark.gpu


def _oracle_scf(mol, basis, tau):
    from paper_2412_13203_b200.scf import rhf
    S_ = Oracle("orc").system(geom(mol), BASIS[basis])
    S, T, V = S_.one_electron()
    return rhf(lambda D: S_.build_jk(D, tau)[:2], S, T + V, S_.nuclear_repulsion(), S_.nelectrons // 2,
               conv=1e-9, e_conv=1e-12)


@pytest.mark.parametrize("mol,basis,tau", [("water", "sto-3g", 0.0), ("water", "cc-pvdz", 1e-12),
                                           ("benzene", "6-31g*", 1e-12), ("w4", "cc-pvdz", 1e-10),
                                           ("water", "cc-pvtz", 1e-12)])
def test_scf_energy_vs_oracle(gpu, mol, basis, tau):
    from paper_2412_13203_b200.scf import run_rhf
    g = run_rhf(geom(mol), BASIS[basis], tau=tau, conv=1e-9, e_conv=1e-12)
    o = _oracle_scf(mol, basis, tau)
    assert g.converged and o.converged
    assert abs(g.energy - o.energy) < 1e-8, (g.energy, o.energy)
    if (mol, basis) == ("water", "sto-3g"):
        assert abs(g.energy - (-74.9630231287)) < 1e-8


@pytest.mark.parametrize("mol,basis,tau", [("water", "cc-pvdz", 1e-12), ("w4", "cc-pvdz", 1e-10)])
def test_device_resident_scf_matches_host_scf(gpu, mol, basis, tau):
    """the post-Fock step on the GPU (cuSOLVER eigh, DGEMM
    density, device DIIS) reaches the same energy as the host driver."""
    from paper_2412_13203_b200.scf import run_rhf
    h = run_rhf(geom(mol), BASIS[basis], tau=tau, conv=1e-9, e_conv=1e-12)
    d = run_rhf(geom(mol), BASIS[basis], tau=tau, conv=1e-9, e_conv=1e-12, device_resident=True)
    assert h.converged and d.converged
    assert abs(h.energy - d.energy) < 1e-8, (h.energy, d.energy)
