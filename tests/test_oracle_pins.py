"""Pin the CPU oracle restatement (oracle/eri_oracle.c) to the reference.

Golden fixtures in tests/golden/ were produced by the unmodified reference
headers (oracle/_ref, tests/golden/make_golden.py). The oracle must reproduce
them: pair store bit-for-bit (block.hpp:52-103), Boys (boys.hpp:23-44) to
1e-15, every water/STO-3G integral to 1e-14, J/K to 1e-12, and the screened
quartet lists exactly. Plus the SPEC's own examples.
"""
import hashlib
import json
import math
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import Oracle, available
from systems import BASIS, geom

G = Path(__file__).resolve().parent / "golden"


def load(name):
    return json.loads((G / name).read_text())


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def orc():
    return Oracle("orc")


def test_boys_spec_examples(orc):
    assert orc.boys(0, 0.0)[0] == 1.0
    assert np.allclose(orc.boys(3, 0.0), [1, 1 / 3, 1 / 5, 1 / 7], rtol=0, atol=1e-16)
    assert abs(orc.boys(0, 1.0)[0] - 0.7468241328) < 1e-10


def test_boys_vs_reference_grid(orc):
    g = load("reference_plans_boys.json")["boys"]
    for T, ref in zip(g["T"], g["F16"]):
        F = orc.boys(16, T)
        assert np.allclose(F, ref, rtol=1e-15, atol=0), T


def test_boys_vs_quadrature(orc):
    from scipy.integrate import quad
    for T in [0.0, 1e-6, 0.5, 1.0, 5.0, 20.0, 50.0, 200.0]:
        F = orc.boys(16, T)
        for m in range(17):
            q, _ = quad(lambda t: t ** (2 * m) * math.exp(-T * t * t), 0.0, 1.0, epsabs=1e-15, epsrel=1e-14,
                        limit=200)
            assert abs(F[m] - q) < 1e-13, (T, m)
        # downward consistency F_m = (2T F_{m+1} + e^-T)/(2m+1)
        for m in range(16):
            assert abs(F[m] - (2 * T * F[m + 1] + math.exp(-T)) / (2 * m + 1)) < 1e-12


def test_water_sto3g_pair_store_bitwise(orc):
    w = load("water_sto3g.json")
    S = orc.system(geom("water"), BASIS["sto-3g"])
    assert (S.nbf, S.npairs, S.ntiles, S.nblocks) == (w["nbf"], w["npairs"], w["ntiles"], w["nblocks"])
    i, j, k = S.pairs()
    assert i.tolist() == w["pair_i"] and j.tolist() == w["pair_j"] and k.tolist() == w["pair_nprim"]
    for x in range(S.npairs):
        assert S.pair_prims(x, int(k[x])).ravel().tolist() == w["prims"][x]  # bit-identical


def test_water_sto3g_integrals_and_jk(orc):
    w = load("water_sto3g.json")
    S = orc.system(geom("water"), BASIS["sto-3g"])
    for key, ref in w["eri"].items():
        x, y = map(int, key.split(","))
        assert np.allclose(S.eri(x, y), ref, rtol=1e-14, atol=1e-15), key
    assert np.allclose(S.schwarz(), w["Q"], rtol=1e-14, atol=0)
    rng = np.random.default_rng(w["D_seed"])
    A = rng.standard_normal((S.nbf, S.nbf))
    D = (A + A.T) / np.sqrt(S.nbf)
    J, K, nq = S.build_jk(D, 0.0, 1)
    assert nq == w["nquartets"] == 120
    assert np.max(np.abs(J.ravel() - w["J"])) < 1e-13 and np.max(np.abs(K.ravel() - w["K"])) < 1e-13
    # textbook (O1s O1s|O1s O1s)
    assert abs(S.eri(0, 0)[0] - 4.7850654047) < 1e-9


def test_benzene_lists_identical(orc):
    b = load("benzene_631gs.json")
    S = orc.system(geom("benzene"), BASIS["6-31g*"])
    assert (S.nbf, S.npairs, S.ntiles, S.nblocks) == (b["nbf"], b["npairs"], b["ntiles"], b["nblocks"])
    Q = S.schwarz()
    assert np.allclose(Q, b["Q"], rtol=1e-13, atol=1e-300)
    for tau, ref in b["lists"].items():
        xs, ys = S.quartets(float(tau))
        o = np.lexsort((ys, xs))
        assert len(xs) == ref["n"]
        assert sha(np.stack([xs[o], ys[o]])) == ref["sha256_sorted_xy"]


def test_w4_ccpvdz_jk(orc):
    c = load("w4_ccpvdz.json")
    S = orc.system(geom("w4"), BASIS["cc-pvdz"])
    rng = np.random.default_rng(c["D_seed"])
    A = rng.standard_normal((S.nbf, S.nbf))
    D = (A + A.T) / np.sqrt(S.nbf)
    J, K, nq = S.build_jk(D, c["tau"], 0)
    assert nq == c["nquartets"]
    assert np.max(np.abs(J.ravel() - c["J"])) < 1e-12 and np.max(np.abs(K.ravel() - c["K"])) < 1e-12
    xs, ys = S.quartets(c["tau"])
    o = np.lexsort((ys, xs))
    assert sha(np.stack([xs[o], ys[o]])) == c["sha256_sorted_xy"]


def test_shell_normalisation(orc):
    for b in ("sto-3g", "6-31g*", "cc-pvdz", "cc-pvtz"):
        S = orc.system(geom("water"), BASIS[b])
        Sm, _, _ = S.one_electron()
        assert np.allclose(np.diag(Sm), 1.0, atol=1e-10), b


def test_parse_errors(orc):
    with pytest.raises(ValueError):
        orc.system("2\n\nH 0 0 0\n", BASIS["sto-3g"])  # declared 2, found 1 (SPEC.md input)
    with pytest.raises(ValueError):
        orc.system("1\n\nXx 0 0 0\n", BASIS["sto-3g"])
    with pytest.raises(ValueError):
        orc.system("1\n\nHe 0 0 0\n", BASIS["sto-3g"])  # element missing from the table


@pytest.mark.skipif(not available("ref"), reason="reference headers not built here")
def test_ref_library_matches_golden():
    R = Oracle("ref")
    w = load("water_sto3g.json")
    S = R.system(geom("water"), BASIS["sto-3g"])
    for key, ref in list(w["eri"].items())[:40]:
        x, y = map(int, key.split(","))
        assert S.eri(x, y).tolist() == ref
