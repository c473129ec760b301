"""Shared test systems (fixtures) for the parity tests."""
from paper_2412_13203_b200.eritile import read_fixture
from paper_2412_13203_b200.geometry import alanine_chain, water_cluster

BASIS = {b: read_fixture("basis", f) for b, f in
         [("sto-3g", "sto-3g.txt"), ("6-31g*", "6-31gs.txt"), ("cc-pvdz", "cc-pvdz.txt"),
          ("cc-pvtz", "cc-pvtz.txt")]}


def geom(name: str) -> str:
    if name.startswith("w") and name[1:].isdigit():
        return water_cluster(int(name[1:]))
    if name.startswith("ala") and name[3:].isdigit():
        return alanine_chain(int(name[3:]))
    return read_fixture("geom", name + ".xyz")
