"""GPU parity: the sm_100a path through the C ABI against the CPU oracle.

Bars (BASELINE.json north_star): J/K within 1e-10 absolute, identical
screened-quartet lists (bit-exact reference pair-store indexing), SCF energy
within 1e-8 Ha (tests/test_gpu_scf.py).
"""
import numpy as np
import pytest

from oracle_lib import Oracle
from systems import BASIS, geom

pytestmark = pytest.mark.gpu


def _engine(xyz, basis, tau):
    from paper_2412_13203_b200.eritile import Engine
    e = Engine(0).load_molecule(xyz, basis).build_pairs(0.0)
    e.set_screening(tau)
    return e


def _rand_density(n, seed=0):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    return (A + A.T) / np.sqrt(n)


def test_boys_device_vs_reference(gpu):
    from paper_2412_13203_b200.eritile import Engine
    e = Engine(0)
    o = Oracle("orc")
    Ts = np.array([0.0, 1e-6, 1e-3, 0.5, 1.0, 2.03125, 5.0, 12.7, 20.0, 33.3, 35.999, 36.0, 39.99,
                   40.0, 40.01, 50.0, 79.9, 80.1, 200.0, 1e4])
    for m in range(0, 17):
        F = e.boys(m, Ts)
        for t, row in zip(Ts, F):
            ref = o.boys(m, float(t))
            assert np.allclose(row, ref, rtol=2e-14, atol=1e-300), (m, t, row, ref)


def test_boys_device_uniform_warps(gpu):
    """Warps whose lanes all sit below T = 40, all above, or straddle it give
    the reference values (boys.hpp:23-44) from the straight-line Boys form."""
    from paper_2412_13203_b200.eritile import Engine
    e = Engine(0)
    o = Oracle("orc")
    rng = np.random.default_rng(4)
    for Ts in (rng.uniform(0.0, 39.99, 64), rng.uniform(40.0, 120.0, 64), np.linspace(0.0, 80.0, 64)):
        for m in range(0, 17):
            F = e.boys(m, Ts)
            for t, row in zip(Ts, F):
                assert np.allclose(row, o.boys(m, float(t)), rtol=2e-14, atol=1e-300), (m, t)


@pytest.mark.parametrize("mol,basis", [("water", "sto-3g"), ("water", "cc-pvdz"), ("benzene", "6-31g*")])
def test_eri_quartets_all_classes(gpu, mol, basis):
    xyz, bas = geom(mol), BASIS[basis]
    e = _engine(xyz, bas, 0.0)
    O = Oracle("orc").system(xyz, bas)
    n = O.npairs
    rng = np.random.default_rng(1)
    pairs = [(x, y) for x in range(n) for y in range(x, n)]
    if len(pairs) > 3000:
        idx = rng.choice(len(pairs), 3000, replace=False)
        pairs = [pairs[i] for i in idx]
    worst = 0.0
    for x, y in pairs:
        g = e.eri_quartet(x, y)
        r = O.eri(x, y)
        worst = max(worst, float(np.max(np.abs(g - r) / (1.0 + np.abs(r)))))
        assert np.allclose(g, r, rtol=1e-12, atol=1e-14), (x, y, np.max(np.abs(g - r)))
    assert worst < 1e-12


@pytest.mark.parametrize("mol,basis", [("water", "cc-pvdz"), ("benzene", "6-31g*"), ("w8", "cc-pvdz")])
def test_schwarz_and_quartet_lists(gpu, mol, basis):
    xyz, bas = geom(mol), BASIS[basis]
    e = _engine(xyz, bas, 0.0)
    O = Oracle("orc").system(xyz, bas)
    Qg = e.schwarz()
    Qo = O.schwarz()
    # Q of near-zero-overlap pairs carries horizontal-recurrence cancellation;
    # the list identity below is the strict bar.
    rel = np.abs(Qg - Qo) / np.maximum(np.abs(Qo), 1e-300)
    assert np.max(np.abs(Qg - Qo)) < 1e-12 and np.median(rel) < 1e-14, (rel.max(), np.argmax(rel))
    for tau in (1e-10, 1e-12):
        e.set_screening(tau)
        xs, ys = e.quartets()
        ox, oy = O.quartets(tau)
        order = np.lexsort((oy, ox))
        assert len(xs) == len(ox)
        assert np.array_equal(xs, ox[order]) and np.array_equal(ys, oy[order])


def test_quartet_list_shared_q_identity(gpu):
    """With one shared Q the lists must be identical by construction."""
    xyz, bas = geom("w4"), BASIS["cc-pvdz"]
    e = _engine(xyz, bas, 0.0)
    O = Oracle("orc").system(xyz, bas)
    Q = O.schwarz()
    e.set_schwarz(Q)
    e.set_screening(1e-10)
    xs, ys = e.quartets()
    ox, oy = O.quartets(1e-10)
    order = np.lexsort((oy, ox))
    assert np.array_equal(xs, ox[order]) and np.array_equal(ys, oy[order])


@pytest.mark.parametrize("mol,basis,tau", [("water", "sto-3g", 0.0), ("water", "cc-pvdz", 0.0),
                                           ("benzene", "6-31g*", 1e-12), ("w4", "cc-pvdz", 1e-10),
                                           ("w8", "cc-pvdz", 1e-10)])
def test_jk_vs_oracle(gpu, mol, basis, tau):
    xyz, bas = geom(mol), BASIS[basis]
    e = _engine(xyz, bas, tau)
    O = Oracle("orc").system(xyz, bas)
    D = _rand_density(e.nbf)
    J, K = e.build_jk(D)
    Jo, Ko, nq = O.build_jk(D, tau)
    assert nq == e.num_quartets()
    assert np.max(np.abs(J - Jo)) < 1e-10
    assert np.max(np.abs(K - Ko)) < 1e-10
    assert np.allclose(J, J.T, atol=1e-14) and np.allclose(K, K.T, atol=1e-14)


def test_jk_zero_and_linearity(gpu):
    xyz, bas = geom("w4"), BASIS["cc-pvdz"]
    e = _engine(xyz, bas, 1e-10)
    N = e.nbf
    J0, K0 = e.build_jk(np.zeros((N, N)))
    assert not J0.any() and not K0.any()
    D1, D2 = _rand_density(N, 1), _rand_density(N, 2)
    J1, K1 = e.build_jk(D1)
    J2, K2 = e.build_jk(D2)
    J3, K3 = e.build_jk(0.7 * D1 - 1.3 * D2)
    assert np.max(np.abs(J3 - (0.7 * J1 - 1.3 * J2))) < 1e-9
    assert np.max(np.abs(K3 - (0.7 * K1 - 1.3 * K2))) < 1e-9


def test_dense_reference_loop_water(gpu):
    """J/K against a dense O(N^4) einsum over the oracle's full ERI tensor."""
    xyz, bas = geom("water"), BASIS["sto-3g"]
    O = Oracle("orc").system(xyz, bas)
    N = O.nbf
    sh = O.shells()
    i, j, _ = O.pairs()
    nc = lambda l: (l + 1) * (l + 2) // 2
    G = np.zeros((N, N, N, N))
    for x in range(O.npairs):
        for y in range(O.npairs):
            v = O.eri(x, y)
            a, b, c, d = i[x], j[x], i[y], j[y]
            la, lb, lc, ld = (sh["L"][s] for s in (a, b, c, d))
            v = v.reshape(nc(la), nc(lb), nc(lc), nc(ld))
            oa, ob, oc, od = (sh["bf_off"][s] for s in (a, b, c, d))
            blk = G[oa:oa + nc(la), ob:ob + nc(lb), oc:oc + nc(lc), od:od + nc(ld)]
            blk[...] = v
            G[ob:ob + nc(lb), oa:oa + nc(la), oc:oc + nc(lc), od:od + nc(ld)] = v.transpose(1, 0, 2, 3)
            G[oa:oa + nc(la), ob:ob + nc(lb), od:od + nc(ld), oc:oc + nc(lc)] = v.transpose(0, 1, 3, 2)
            G[ob:ob + nc(lb), oa:oa + nc(la), od:od + nc(ld), oc:oc + nc(lc)] = v.transpose(1, 0, 3, 2)
    D = _rand_density(N, 5)
    Jd = np.einsum("mnls,ls->mn", G, D)
    Kd = np.einsum("mlns,ls->mn", G, D)
    e = _engine(xyz, bas, 0.0)
    J, K = e.build_jk(D)
    assert np.max(np.abs(J - Jd)) < 1e-10 and np.max(np.abs(K - Kd)) < 1e-10


def _force_variant(e, k):
    """Set every class to its k-th active kernel variant (clamped)."""
    from paper_2412_13203_b200.eritile import class_table
    for i in range(len(class_table())):
        lo, hi = e.variant_range(i)
        e.set_variant(i, lo + min(k, hi - lo - 1))


@pytest.mark.parametrize("k", list(range(16)))
def test_every_kernel_variant_eri_and_jk(gpu, k):
    """Every kernel variant (lane / unit / strip / coop families) of every class gives the
    oracle's integrals and J/K (benzene 6-31G* covers all L<=2 classes that
    occur with d shells; water cc-pVDZ the s/p/d mixes)."""
    for mol, basis, tau in [("benzene", "6-31g*", 1e-12), ("water", "cc-pvdz", 0.0)]:
        xyz, bas = geom(mol), BASIS[basis]
        e = _engine(xyz, bas, tau)
        _force_variant(e, k)
        O = Oracle("orc").system(xyz, bas)
        rng = np.random.default_rng(7 + k)
        n = O.npairs
        for _ in range(300):
            x, y = sorted(rng.integers(0, n, 2))
            g, r = e.eri_quartet(int(x), int(y)), O.eri(int(x), int(y))
            assert np.allclose(g, r, rtol=1e-12, atol=1e-14), (mol, k, x, y)
        D = _rand_density(e.nbf, 3)
        J, K = e.build_jk(D)
        Jo, Ko, nq = O.build_jk(D, tau)
        assert nq == e.num_quartets()
        assert np.max(np.abs(J - Jo)) < 1e-10 and np.max(np.abs(K - Ko)) < 1e-10, (mol, k)


def test_tuned_build_matches_oracle(gpu):
    """The Workload Allocator only picks variants: results stay within 1e-10."""
    xyz, bas = geom("w4"), BASIS["cc-pvdz"]
    e = _engine(xyz, bas, 1e-10)
    D = _rand_density(e.nbf, 4)
    e.tune(D, reps=1)
    J, K = e.build_jk(D)
    Jo, Ko, _ = Oracle("orc").system(xyz, bas).build_jk(D, 1e-10)
    assert np.max(np.abs(J - Jo)) < 1e-10 and np.max(np.abs(K - Ko)) < 1e-10


@pytest.mark.parametrize("kappa", [1e-14, 1e-12])
def test_kappa_screen_parity(gpu, kappa):
    """The reference's primitive-pair screen (block.hpp:83-89)
    applied on both sides: identical lists, J/K within 1e-10; and within 1e-10
    of the unscreened build as well."""
    xyz, bas = geom("w4"), BASIS["cc-pvdz"]
    e = Engine_k(xyz, bas, kappa, 1e-10)
    O = Oracle("orc").system(xyz, bas, kappa_screen=kappa)
    assert e.npairs == O.npairs
    xs, ys = e.quartets()
    ox, oy = O.quartets(1e-10)
    order = np.lexsort((oy, ox))
    assert np.array_equal(xs, ox[order]) and np.array_equal(ys, oy[order])
    D = _rand_density(e.nbf, 6)
    J, K = e.build_jk(D)
    Jo, Ko, _ = O.build_jk(D, 1e-10)
    assert np.max(np.abs(J - Jo)) < 1e-10 and np.max(np.abs(K - Ko)) < 1e-10
    if kappa > 1e-14:
        return
    J0, K0 = _engine(xyz, bas, 1e-10).build_jk(D)
    assert np.max(np.abs(J - J0)) < 1e-10 and np.max(np.abs(K - K0)) < 1e-10


def Engine_k(xyz, bas, kappa, tau):
    from paper_2412_13203_b200.eritile import Engine
    e = Engine(0).load_molecule(xyz, bas).build_pairs(kappa)
    e.set_screening(tau)
    return e


@pytest.mark.parametrize("k", [0, 1])
def test_f_shells_cc_pvtz(gpu, k):
    """L=3 (f) classes: water/cc-pVTZ integrals and J/K vs the oracle, for the
    default and the alternative kernel variant of every class."""
    xyz, bas = geom("water"), BASIS["cc-pvtz"]
    e = _engine(xyz, bas, 1e-12)
    if k:
        _force_variant(e, 9)
    O = Oracle("orc").system(xyz, bas)
    rng = np.random.default_rng(11)
    n = O.npairs
    for _ in range(400):
        x, y = sorted(rng.integers(0, n, 2))
        g, r = e.eri_quartet(int(x), int(y)), O.eri(int(x), int(y))
        assert np.allclose(g, r, rtol=1e-12, atol=1e-13), (x, y, np.max(np.abs(g - r)))
    D = _rand_density(e.nbf, 12)
    J, K = e.build_jk(D)
    Jo, Ko, nq = O.build_jk(D, 1e-12)
    assert nq == e.num_quartets()
    assert np.max(np.abs(J - Jo)) < 1e-10 and np.max(np.abs(K - Ko)) < 1e-10


@pytest.mark.parametrize("mol,basis,tau,kappa", [("w4", "cc-pvdz", 1e-10, 0.0), ("w8", "cc-pvdz", 1e-10, 1e-14),
                                                 ("benzene", "6-31g*", 1e-12, 0.0)])
def test_family_units_jk_match_pairs_and_oracle(gpu, mol, basis, tau, kappa):
    """Shared-primitive unit kernels give the oracle's J/K (1e-10) and the
    pair kernels' J/K, with identical quartet lists."""
    from paper_2412_13203_b200.eritile import Engine
    xyz, bas = geom(mol), BASIS[basis]
    D = _rand_density(Engine_k(xyz, bas, kappa, tau).nbf, 9)
    res = {}
    for fam in (False, True):
        e = Engine(0).load_molecule(xyz, bas).build_pairs(kappa)
        e.set_families(fam)
        e.set_screening(tau)
        if fam:  # unit kernels for every class that has them
            from paper_2412_13203_b200.eritile import class_table, variant_names
            for i in range(len(class_table())):
                names = variant_names(i)
                if any(n.startswith("fam_") for n in names):
                    e.set_variant(i, next(k for k, n in enumerate(names) if n.startswith("fam_")))
        res[fam] = (e.build_jk(D), e.quartets(), e.stats()["prim_quartets"])
    (Jf, Kf), (xf, yf), pf = res[True]
    (Jp, Kp), (xp, yp), pp = res[False]
    assert np.array_equal(xf, xp) and np.array_equal(yf, yp)
    if mol.startswith("w"):
        assert pf < pp  # O 1s/2s primitive quartets evaluated once
    assert np.max(np.abs(Jf - Jp)) < 1e-11 and np.max(np.abs(Kf - Kp)) < 1e-11
    Jo, Ko, nq = Oracle("orc").system(xyz, bas, kappa_screen=kappa).build_jk(D, tau)
    assert nq == len(xf)
    assert np.max(np.abs(Jf - Jo)) < 1e-10 and np.max(np.abs(Kf - Ko)) < 1e-10


def test_edge_cases_empty_and_tiny(gpu):
    """Edge cases: every quartet screened out (J = K = 0, no launches of class
    kernels), a single-shell system, and H2 (two identical s shells)."""
    xyz, bas = geom("water"), BASIS["cc-pvdz"]
    e = _engine(xyz, bas, 1e6)
    assert e.num_quartets() == 0 and len(e.quartets()[0]) == 0
    J, K = e.build_jk(_rand_density(e.nbf))
    assert not J.any() and not K.any()
    h = "1\nH atom\nH 0.0 0.0 0.0\n"
    for x, b in [(h, BASIS["sto-3g"]), (geom("h2"), BASIS["sto-3g"]), (geom("h2"), BASIS["cc-pvdz"])]:
        e = _engine(x, b, 0.0)
        O = Oracle("orc").system(x, b)
        D = _rand_density(e.nbf, 2)
        J, K = e.build_jk(D)
        Jo, Ko, nq = O.build_jk(D, 0.0)
        assert nq == e.num_quartets()
        assert np.max(np.abs(J - Jo)) < 1e-12 and np.max(np.abs(K - Ko)) < 1e-12


def test_concurrent_and_serial_launches_agree(gpu):
    """Class launches on 4 streams (default) and on one stream give the same
    J/K up to FP64 atomic summation order."""
    xyz, bas = geom("w4"), BASIS["cc-pvdz"]
    e = _engine(xyz, bas, 1e-10)
    D = _rand_density(e.nbf, 21)
    J1, K1 = e.build_jk(D)
    e.set_concurrent(False)
    J2, K2 = e.build_jk(D)
    assert np.max(np.abs(J1 - J2)) < 1e-12 and np.max(np.abs(K1 - K2)) < 1e-12


def test_ss_closed_form_and_bra_ket_symmetry(gpu):
    """(ss|ss) of unit-exponent Gaussians is pi^(5/2)/4 before
    normalisation, i.e. 2/sqrt(pi) for normalised functions; and the
    bra<->ket permutation identity on 200 random quartets (all L<=2 classes
    of benzene/6-31G*)."""
    import math
    from paper_2412_13203_b200.eritile import Engine
    basis = "element H\n0 1\n1.0 1.0\n"
    e = Engine(0).load_molecule("1\nunit s\nH 0 0 0\n", basis).build_pairs(0.0)
    v = e.eri_quartet(0, 0)
    assert abs(v[0] - 2.0 / math.sqrt(math.pi)) < 1e-14
    assert abs(v[0] * (math.pi / 2.0) ** 3 - math.pi ** 2.5 / 4.0) < 1e-13
    xyz, bas = geom("benzene"), BASIS["6-31g*"]
    e = _engine(xyz, bas, 0.0)
    L, _, _ = e.shell_info()
    i, j = e.pair_shells()
    nc = lambda l: (l + 1) * (l + 2) // 2
    rng = np.random.default_rng(5)
    for _ in range(200):
        x, y = (int(t) for t in rng.integers(0, e.npairs, 2))
        a = e.eri_quartet(x, y).reshape(nc(L[i[x]]) * nc(L[j[x]]), nc(L[i[y]]) * nc(L[j[y]]))
        b = e.eri_quartet(y, x).reshape(nc(L[i[y]]) * nc(L[j[y]]), nc(L[i[x]]) * nc(L[j[x]]))
        assert np.allclose(a, b.T, rtol=1e-12, atol=1e-14), (x, y)


@pytest.mark.parametrize("mol,basis,kappa,smin,smax", [("water", "cc-pvdz", 0.0, 1, 3), ("benzene", "6-31g*", 0.0, 1, 1000),
                                                       ("w4", "cc-pvdz", 1e-14, 1, 5), ("w8", "cc-pvdz", 1e-14, 64, 256)])
def test_strip_kernels_vs_oracle(gpu, mol, basis, kappa, smin, smax):
    """Bra-stationary strip kernels (K rows in shared memory, csrc/jk_strip.cuh)
    on pair and unit lists: J/K within 1e-10 of the oracle, lists unchanged.
    Small strip thresholds put (nearly) every bra into strips; short strips
    (smax) exercise the per-strip flush many times per bra."""
    from paper_2412_13203_b200.eritile import Engine, class_table, variant_names
    xyz, bas = geom(mol), BASIS[basis]
    tau = 1e-10
    O = Oracle("orc").system(xyz, bas, kappa_screen=kappa)
    D = _rand_density(O.nbf, 31)
    Jo, Ko, nq = O.build_jk(D, tau)
    ox, oy = O.quartets(tau)
    order = np.lexsort((oy, ox))
    ncls = len(class_table())
    for fam in (False, True):
        e = Engine(0).load_molecule(xyz, bas).build_pairs(kappa)
        e.set_families(fam).set_strips(smin, smax)
        e.set_screening(tau)
        xs, ys = e.quartets()
        assert np.array_equal(xs, ox[order]) and np.array_equal(ys, oy[order])
        assert nq == e.num_quartets()
        # every strip variant (loop styles, batched / aggregated / split K
        # updates, prefetch options), each on every class that has it
        want = "fstrip" if fam else "strip"
        vnames = sorted({n for i in range(ncls) for n in variant_names(i) if n.startswith(want)})
        assert vnames
        for vn in vnames:
            for i in range(ncls):
                if vn in variant_names(i):
                    e.set_variant(i, vn)
            J, K = e.build_jk(D)
            dj, dk = np.max(np.abs(J - Jo)), np.max(np.abs(K - Ko))
            assert dj < 1e-10 and dk < 1e-10, (fam, vn, dj, dk)
