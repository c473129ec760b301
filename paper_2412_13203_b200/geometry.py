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
