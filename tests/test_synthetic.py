"""The seeded input generator (synthetic/) — determinism, sharding and the config recipe."""
import numpy as np
import pytest

import synthetic


def test_deterministic_and_shard_equal_full():
    cfg = synthetic.CONFIGS[1]
    a = synthetic.generate(cfg)
    b = synthetic.generate(cfg, tasks=[2, 3])
    np.testing.assert_array_equal(a["phi"][2:], b["phi"])
    np.testing.assert_array_equal(a["y"][2:], b["y"])
    np.testing.assert_array_equal(a["z"][2:], b["z"])
    c = synthetic.generate(cfg)
    np.testing.assert_array_equal(a["phi"], c["phi"])


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_recipe_shapes_and_supports(cid):
    cfg = synthetic.CONFIGS[cid]
    d = synthetic.generate(cfg, tasks=[0, cfg.T - 1])
    assert d["phi"].shape == (2, cfg.N, cfg.D) and d["phi"].dtype == np.float32
    assert d["y"].shape == (2, cfg.N) and d["y"].dtype == np.float32
    lab = synthetic.labels(cfg)
    assert np.bincount(lab).tolist() == sorted(cfg.cluster_sizes, reverse=False) or \
        sorted(np.bincount(lab).tolist()) == sorted(cfg.cluster_sizes)
    for i, t in enumerate(d["tasks"]):
        sup = synthetic.supports(cfg)[lab[t]]
        assert set(np.nonzero(d["z"][i])[0]) <= set(sup.tolist())
    # Φ entries ~ N(0, 1/N)
    v = d["phi"].astype(np.float64).var()
    assert abs(v * cfg.N - 1.0) < 0.05


def test_c2_overlap_is_twenty_percent():
    cfg = synthetic.CONFIGS[2]
    s = [set(x.tolist()) for x in synthetic.supports(cfg)]
    for i in range(4):
        assert len(s[i]) == 30
        for j in range(i + 1, 4):
            assert len(s[i] & s[j]) == 6


def test_shard_partition():
    for T in (1, 5, 16, 64, 256):
        for world in (1, 2, 3, 4, 8):
            blocks = [synthetic.shard(T, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == T
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            sizes = [e - b for b, e in blocks]
            assert max(sizes) - min(sizes) <= 1
