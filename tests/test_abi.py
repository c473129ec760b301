"""C ABI boundary (include/eritile_gpu.h) without a GPU: symbol exports,
error behaviour, and the host Block Constructor in a host-only context."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import Oracle
from systems import BASIS, geom

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    txt = (ROOT / "include" / "eritile_gpu.h").read_text()
    return sorted(set(re.findall(r"\b(eritile_gpu_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2412_13203_b200 import _native
    lib = _native.load()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s


def test_cpp_wrapper_header_declares_reference_names():
    txt = (ROOT / "include" / "eritile" / "executor.hpp").read_text()
    for name in ("build_jk", "build_g", "GpuExecutor"):
        assert name in txt


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2412_13203_b200.eritile import Engine
    with pytest.raises(RuntimeError, match="no CUDA device"):
        Engine(0)


def test_class_table():
    from paper_2412_13203_b200.eritile import class_table
    from paper_2412_13203_b200.eritile import variant_names
    t = class_table()
    assert len(t) == 55  # canonical classes for L <= 3 (La>=Lb, Lc>=Ld, bra key >= ket key)
    assert t[0][:4] == (0, 0, 0, 0)
    assert {r[:4] for r in t} >= {(3, 3, 3, 3), (2, 2, 2, 2), (3, 0, 1, 0)}
    for i, r in enumerate(t):  # every class has >= 1 kernel; coop for the big plans
        names = variant_names(i)
        assert names and len(set(names)) == len(names)
        if r[5] > 21000:  # table kernels only
            assert set(names) <= {"coop", "coopw"} and "coop" in names
        elif r[5] > 4000:  # + one straight-line J/K lane kernel (255 registers)
            assert set(names) <= {"coop", "coopw", "lane_plm1"} and "coop" in names and "lane_plm1" in names


@pytest.mark.parametrize("mol,basis", [("water", "sto-3g"), ("benzene", "6-31g*"), ("w8", "cc-pvdz")])
def test_host_block_constructor_matches_reference_order(mol, basis):
    from paper_2412_13203_b200.eritile import Engine
    e = Engine(-1).load_molecule(geom(mol), BASIS[basis]).build_pairs(0.0)
    O = Oracle("orc").system(geom(mol), BASIS[basis])
    i, j = e.pair_shells()
    oi, oj, _ = O.pairs()
    assert np.array_equal(i, oi) and np.array_equal(j, oj)
    assert e.nbf == O.nbf and e.nelectrons == O.nelectrons
    assert abs(e.nuclear_repulsion() - O.nuclear_repulsion()) < 1e-10


@pytest.mark.parametrize("tau", [0.0, 1e-10, 1e-12])
def test_screened_lists_identical_with_shared_q(tau):
    from paper_2412_13203_b200.eritile import Engine
    xyz, bas = geom("w8"), BASIS["cc-pvdz"]
    O = Oracle("orc").system(xyz, bas)
    Q = O.schwarz()
    e = Engine(-1).load_molecule(xyz, bas).build_pairs(0.0)
    e.set_schwarz(Q)
    e.set_screening(tau)
    xs, ys = e.quartets()
    ox, oy = O.quartets(tau)
    o = np.lexsort((oy, ox))
    assert np.array_equal(xs, ox[o]) and np.array_equal(ys, oy[o])
    assert e.num_quartets() == len(ox)


def test_kappa_screen_pairs_match():
    from paper_2412_13203_b200.eritile import Engine
    xyz, bas = geom("w8"), BASIS["cc-pvdz"]
    e = Engine(-1).load_molecule(xyz, bas).build_pairs(1e-14)
    O = Oracle("orc").system(xyz, bas, kappa_screen=1e-14)
    i, j = e.pair_shells()
    oi, oj, _ = O.pairs()
    assert np.array_equal(i, oi) and np.array_equal(j, oj)


def test_one_electron_vs_oracle():
    from paper_2412_13203_b200.eritile import Engine
    for mol, basis in [("water", "cc-pvdz"), ("benzene", "6-31g*")]:
        e = Engine(-1).load_molecule(geom(mol), BASIS[basis])
        O = Oracle("orc").system(geom(mol), BASIS[basis])
        for a, b in zip(e.one_electron(), O.one_electron()):
            assert np.max(np.abs(a - b)) < 1e-11


def test_errors_map_to_reference_exceptions():
    from paper_2412_13203_b200.eritile import Engine, ParseError
    e = Engine(-1)
    with pytest.raises(ParseError):
        e.load_molecule("2\n\nH 0 0 0\n", BASIS["sto-3g"])
    with pytest.raises(ParseError):
        e.load_molecule("1\n\nHe 0 0 0\n", BASIS["sto-3g"])
    with pytest.raises(RuntimeError):
        e.build_pairs(0.0)  # no molecule loaded (state error)
    e.load_molecule(geom("water"), BASIS["sto-3g"]).build_pairs(0.0)
    with pytest.raises(RuntimeError):
        e.schwarz()  # host-only: needs a device


def test_cpp_wrapper_compiles_and_runs_host_only(tmp_path):
    import subprocess
    src = tmp_path / "t.cpp"
    src.write_text(r'''
#include <cstdio>
#include "eritile/executor.hpp"
int main() {
  eritile::GpuExecutor ex(-1);  // host-only context
  ex.load_molecule("3\nw\nO 0 0 0.1173\nH 0 0.7572 -0.4692\nH 0 -0.7572 -0.4692\n",
                   "element H\n0 3\n3.42525091 0.15432897\n0.62391373 0.53532814\n0.16885540 0.44463454\n"
                   "element O\n0 3\n130.7093200 0.15432897\n23.8088610 0.53532814\n6.4436083 0.44463454\n"
                   "0 3\n5.0331513 -0.09996723\n1.1695961 0.39951283\n0.3803890 0.70011547\n"
                   "1 3\n5.0331513 0.15591627\n1.1695961 0.60768372\n0.3803890 0.39195739\n");
  ex.build_pairs(0.0);
  try { ex.build_jk(std::vector<double>(49, 0.0)); return 3; } catch (const std::runtime_error&) {}
  try { ex.load_molecule("2\n\nH 0 0 0\n", "element H\n0 1\n1.0 1.0\n"); return 4; }
  catch (const eritile::GpuParseError&) {}
  std::printf("%d\n", ex.nbf());
  return ex.nbf() == 7 ? 0 : 2;
}
''')
    lib = ROOT / "paper_2412_13203_b200" / "_lib"
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++17", "-I", str(ROOT / "include"), str(src), "-L", str(lib),
                    "-leritile_b200", "-Wl,-rpath," + str(lib), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("tau,kappa", [(1e-10, 0.0), (1e-10, 1e-14), (0.0, 1e-14)])
def test_family_units_keep_the_quartet_list(tau, kappa):
    """Shared-primitive units (generally contracted sibling shells) change
    only how many primitive quartets are evaluated: the canonical screened
    quartet list and its count are identical with units on and off."""
    from paper_2412_13203_b200.eritile import Engine
    xyz, bas = geom("w8"), BASIS["cc-pvdz"]
    O = Oracle("orc").system(xyz, bas, kappa_screen=kappa)
    Q = O.schwarz()
    out = {}
    for fam in (False, True):
        e = Engine(-1).load_molecule(xyz, bas).build_pairs(kappa)
        e.set_families(fam)
        e.set_schwarz(Q)
        e.set_screening(tau)
        if fam:  # run every class that has unit kernels on them
            from paper_2412_13203_b200.eritile import class_table, variant_names
            for i in range(len(class_table())):
                names = variant_names(i)
                if any(n.startswith("fam_") for n in names):
                    e.set_variant(i, next(k for k, n in enumerate(names) if n.startswith("fam_")))
        xs, ys = e.quartets()
        out[fam] = (xs, ys, e.num_quartets(), e.stats()["prim_quartets"])
    assert np.array_equal(out[True][0], out[False][0]) and np.array_equal(out[True][1], out[False][1])
    assert out[True][2] == out[False][2] == len(out[True][0])
    assert out[True][3] < 0.8 * out[False][3]  # O 1s/2s share their nine exponents


def test_host_edge_cases_lists():
    """Host Block Constructor edge cases: all quartets screened away, a single
    shell (one pair, one quartet), and the reference's empty-pair drop under
    the kappa screen (block.hpp:86-87)."""
    from paper_2412_13203_b200.eritile import Engine
    xyz, bas = geom("water"), BASIS["cc-pvdz"]
    O = Oracle("orc").system(xyz, bas)
    e = Engine(-1).load_molecule(xyz, bas).build_pairs(0.0)
    e.set_schwarz(O.schwarz())
    e.set_screening(1e6)
    assert e.num_quartets() == 0 and len(e.quartets()[0]) == 0
    h = "1\nH atom\nH 0.0 0.0 0.0\n"
    e = Engine(-1).load_molecule(h, BASIS["sto-3g"]).build_pairs(0.0)
    e.set_screening(0.0)
    xs, ys = e.quartets()
    assert (e.npairs, e.num_quartets(), xs.tolist(), ys.tolist()) == (1, 1, [0], [0])
    far = "2\nfar apart\nH 0 0 0\nH 0 0 40.0\n"
    e = Engine(-1).load_molecule(far, BASIS["sto-3g"]).build_pairs(1e-14)
    o = Oracle("orc").system(far, BASIS["sto-3g"], kappa_screen=1e-14)
    assert e.npairs == o.npairs == 2  # the inter-atomic pair has no primitive left
