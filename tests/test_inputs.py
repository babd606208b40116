"""The seeded input generator (kpm_inputs): pinned to the published splitmix64
test vector and to the statistical contract of Eq (14)."""
import numpy as np

import kpm_inputs as ki


def test_mix64_matches_published_splitmix64_vector():
    # splitmix64 seeded with 0: first output = mix64(0 + golden gamma) = 0xE220A8397B1DCDAF
    assert ki.mix64_int(ki.GOLDEN) == 0xE220A8397B1DCDAF
    assert int(ki.mix64(np.array([ki.GOLDEN], dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF
    z = np.arange(1000, dtype=np.uint64) * np.uint64(0x1234567)
    assert all(int(v) == ki.mix64_int(int(u)) for u, v in zip(z, ki.mix64(z)))


def test_rademacher_is_pm1_mean0_var1_and_partition_independent():
    r = ki.rademacher(7, 16, 4096)
    assert set(np.unique(r)) == {-1.0, 1.0}
    assert abs(r.mean()) < 5 * (1 / np.sqrt(r.size))           # <<xi>> = 0   (Eq 14)
    # <<xi_r,i xi_r',i'>> = delta delta: off-diagonal correlations are O(1/sqrt(D))
    C = r @ r.T / r.shape[1]
    assert np.allclose(np.diag(C), 1.0)
    assert np.abs(C - np.eye(16)).max() < 6 / np.sqrt(4096)
    # global counters: a sub-block drawn with offsets equals the slice of the full block
    sub = ki.rademacher(7, 4, 1000, r_offset=5, D_total=4096, i_offset=300)
    assert np.array_equal(sub, r[5:9, 300:1300])


def test_anderson_onsite_uniform_in_range():
    e = ki.anderson_onsite(103, 1 << 16, 2.0)
    assert e.min() >= -1.0 and e.max() < 1.0
    assert abs(e.mean()) < 0.02 and abs(e.var() - 4.0 / 12) < 0.01
    assert np.array_equal(e, ki.anderson_onsite(103, 1 << 16, 2.0))


def test_configs_match_baseline_json():
    import json, os
    bj = json.load(open(os.path.join(os.path.dirname(__file__), "..", "BASELINE.json")))
    assert len(bj["configs"]) == 5
    c = ki.CONFIGS
    assert (c["c1"]["L"][0], c["c1"]["N"], c["c1"]["R"]) == (1024, 128, 8)
    assert (ki.num_sites(c["c2"]["L"]), c["c2"]["N"], c["c2"]["R"]) == (262144, 1024, 64)
    assert (ki.num_sites(c["c3"]["L"]), c["c3"]["N"], c["c3"]["R"]) == (2097152, 2048, 128)
    assert (ki.num_sites(c["c4"]["L"]), c["c4"]["N"], c["c4"]["R"]) == (1048576, 4096, 256)
    assert (ki.num_sites(c["c5"]["L"]), c["c5"]["N"], c["c5"]["R"]) == (134217728, 1024, 32)


def test_lattice_csr_input_equals_oracle_matrix():
    """kpm_inputs.lattice_csr (the CSR fed to kpm_create_csr in bench.py) is the same H the
    oracle builds (oracle O1, itself pinned in test_oracle_pins.py)."""
    import oracle
    cases = [dict(ndim=2, L=(16, 8, 1), t=-1.0, onsite=None, flux=0.125),
             dict(ndim=3, L=(5, 4, 3), t=-1.3, onsite=ki.anderson_onsite(1, 60, 2.0), flux=0.0),
             dict(ndim=1, L=(7, 1, 1), t=-1.0, onsite=None, flux=0.0),
             dict(ndim=2, L=(2, 6, 1), t=-0.5, onsite=ki.anderson_onsite(2, 12, 1.0), flux=0.5)]
    for lat in cases:
        rp, col, val = ki.lattice_csr(lat)
        D = rp.size - 1
        Hd = np.zeros((D, D), dtype=complex)
        for i in range(D):
            for k in range(rp[i], rp[i + 1]):
                Hd[i, col[k]] += val[k]
        assert np.array_equal(Hd, oracle.lattice_csr(lat).dense())
