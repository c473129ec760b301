from paper_2412_13203_b200.geometry import MT19937_64, water_cluster


def test_mt19937_64_known_answer():
    # C++ standard [rand.predef]: the 10000th output of a default-constructed
    # std::mt19937_64 (seed 5489) is 9981545732273789042
    g = MT19937_64(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042


def test_water_cluster_sizes():
    for n, atoms in [(1, 3), (16, 48), (80, 240)]:
        lines = water_cluster(n).splitlines()
        assert int(lines[0]) == atoms and len(lines) == atoms + 2
    assert water_cluster(16) == water_cluster(16)
