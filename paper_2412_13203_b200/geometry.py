"""Deterministic benchmark geometries.

``water_cluster(n)`` builds the (H2O)_n lattice: side k = ceil(n^(1/3)),
spacing 3.1 Å, site w at 3.1*(w mod k, floor(w/k) mod k, floor(w/k^2)),
O at the site and the two H at (±0.9572 sin 52.26°, 0, 0.9572 cos 52.26°)
rotated by a uniform random quaternion from std::mt19937_64(2412) with
std::uniform_real_distribution<double>(0,1) (libstdc++ generate_canonical:
one 64-bit draw divided by 2^64). Atom order O, H, H per water.
"""
from __future__ import annotations

import math

_MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the 64-bit Mersenne Twister of the C++ standard)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _MASK64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & _MASK64
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK64

    def uniform01(self) -> float:
        r = float(self()) / 18446744073709551616.0
        return r if r < 1.0 else math.nextafter(1.0, 0.0)


def _rotation(u1: float, u2: float, u3: float):
    a = math.sqrt(1.0 - u1)
    b = math.sqrt(u1)
    q0 = a * math.sin(2 * math.pi * u2)
    q1 = a * math.cos(2 * math.pi * u2)
    q2 = b * math.sin(2 * math.pi * u3)
    q3 = b * math.cos(2 * math.pi * u3)
    # q = (w=q0, x=q1, y=q2, z=q3) -> standard rotation matrix
    w, x, y, z = q0, q1, q2, q3
    return [
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ]


def water_cluster_atoms(n: int, seed: int = 2412, spacing: float = 3.1):
    k = 1
    while k * k * k < n:
        k += 1
    rng = MT19937_64(seed)
    half = math.radians(52.26)
    hx, hz = 0.9572 * math.sin(half), 0.9572 * math.cos(half)
    atoms = []
    for w in range(n):
        site = (spacing * (w % k), spacing * ((w // k) % k), spacing * (w // (k * k)))
        u1, u2, u3 = rng.uniform01(), rng.uniform01(), rng.uniform01()
        R = _rotation(u1, u2, u3)
        atoms.append(("O", site))
        for sgn in (1.0, -1.0):
            v = (sgn * hx, 0.0, hz)
            r = tuple(site[i] + sum(R[i][j] * v[j] for j in range(3)) for i in range(3))
            atoms.append(("H", r))
    return atoms


def to_xyz(atoms, comment: str = "") -> str:
    lines = [str(len(atoms)), comment]
    for sym, (x, y, z) in atoms:
        lines.append(f"{sym} {x:.12f} {y:.12f} {z:.12f}")
    return "\n".join(lines) + "\n"


def water_cluster(n: int, seed: int = 2412) -> str:
    return to_xyz(water_cluster_atoms(n, seed), f"(H2O)_{n} lattice, spacing 3.1 A, mt19937_64({seed})")


# ---- (Ala)_n: idealised extended polyalanine ----
#
# Taxol coordinates are not available offline, so the config-5 workload (an
# f-shell, N-containing, peptide-like L mix at cc-pVTZ) is an idealised
# H-(Ala)_n-OH strand built from standard peptide internal coordinates
# (Engh & Huber bond lengths / angles; planar trans peptides, omega = 180;
# extended beta strand phi = -139, psi = +135 degrees by default) with the
# natural extension reference frame (NeRF). Deterministic, no randomness.

def _sub(a, b):
    return (a[0] - b[0], a[1] - b[1], a[2] - b[2])


def _add(a, b):
    return (a[0] + b[0], a[1] + b[1], a[2] + b[2])


def _scale(a, s):
    return (a[0] * s, a[1] * s, a[2] * s)


def _norm(a):
    n = math.sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2])
    return (a[0] / n, a[1] / n, a[2] / n)


def _cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def _place(a, b, c, bond: float, angle_deg: float, dihedral_deg: float):
    """NeRF: the atom d bonded to c with |cd| = bond, angle(b, c, d) and
    dihedral(a, b, c, d) given in degrees."""
    th, ph = math.radians(angle_deg), math.radians(dihedral_deg)
    bc = _norm(_sub(c, b))
    n = _norm(_cross(_sub(b, a), bc))
    m = _cross(n, bc)
    d2 = (-bond * math.cos(th), bond * math.sin(th) * math.cos(ph), bond * math.sin(th) * math.sin(ph))
    return _add(c, _add(_scale(bc, d2[0]), _add(_scale(m, d2[1]), _scale(n, d2[2]))))


def alanine_chain_atoms(n: int, phi: float = -139.0, psi: float = 135.0, omega: float = 180.0):
    if n < 1:
        raise ValueError("alanine_chain: n >= 1")
    # backbone N, CA, C of every residue, then one virtual N for the C-terminus
    bb = [(0.0, 0.0, 0.0), (1.458, 0.0, 0.0)]
    bb.append(_place((0.0, 1.0, 0.0), bb[0], bb[1], 1.525, 111.2, -60.0))
    for i in range(1, n + 1):
        N = _place(bb[-3], bb[-2], bb[-1], 1.329, 116.2, psi)      # C(i-1)-N(i), dihedral N-CA-C-N = psi
        if i == n:
            bb.append(N)
            break
        CA = _place(bb[-2], bb[-1], N, 1.458, 121.7, omega)        # omega: CA-C-N-CA
        C = _place(bb[-1], N, CA, 1.525, 111.2, phi)               # phi: C-N-CA-C
        bb += [N, CA, C]
    atoms = []
    for i in range(n):
        N, CA, C = bb[3 * i], bb[3 * i + 1], bb[3 * i + 2]
        Nn = bb[3 * i + 3]  # next residue's N (the C-terminal OXT position for the last one)
        Cp = bb[3 * i - 1] if i > 0 else None
        atoms.append(("N", N))
        if Cp is None:  # N-terminal NH2
            atoms.append(("H", _place(C, CA, N, 1.01, 109.5, 120.0)))
            atoms.append(("H", _place(C, CA, N, 1.01, 109.5, -120.0)))
        else:  # amide H in the peptide plane, bisecting the external angle at N
            u = _norm(_add(_norm(_sub(N, Cp)), _norm(_sub(N, CA))))
            atoms.append(("H", _add(N, _scale(u, 1.01))))
        atoms.append(("C", CA))
        # HA and CB: the two remaining tetrahedral positions at CA (L configuration)
        bis = _norm(_add(_norm(_sub(CA, N)), _norm(_sub(CA, C))))
        nrm = _norm(_cross(_sub(N, CA), _sub(C, CA)))
        h = math.radians(54.75)
        cb = _add(CA, _scale(_add(_scale(bis, math.cos(h)), _scale(nrm, math.sin(h))), 1.530))
        ha = _add(CA, _scale(_add(_scale(bis, math.cos(h)), _scale(nrm, -math.sin(h))), 1.090))
        atoms.append(("H", ha))
        atoms.append(("C", cb))
        for dih in (60.0, 180.0, 300.0):
            atoms.append(("H", _place(N, CA, cb, 1.090, 109.5, dih)))
        atoms.append(("C", C))
        u = _norm(_add(_norm(_sub(C, CA)), _norm(_sub(C, Nn))))
        atoms.append(("O", _add(C, _scale(u, 1.231))))
        if i == n - 1:  # C-terminal OH at the virtual next-N position
            oxt = _add(C, _scale(_norm(_sub(Nn, C)), 1.340))
            atoms.append(("O", oxt))
            atoms.append(("H", _place(CA, C, oxt, 0.970, 106.0, 180.0)))
    return atoms


def alanine_chain(n: int, **kw) -> str:
    """H-(Ala)_n-OH extended strand (10 n + 2 atoms), XYZ in Angstrom."""
    return to_xyz(alanine_chain_atoms(n, **kw), f"H-(Ala)_{n}-OH extended strand (idealised internal coordinates)")
