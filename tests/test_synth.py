"""The shared seeded input generator (synth/): determinism, subset
regeneration, stored-dtype exactness and value domains (reading Z9, Z12)."""
import numpy as np

import synth


def test_deterministic_and_subset_regeneration():
    rc = synth.Recipe(seed=1234)
    a = synth.tokens(rc, np.arange(6), np.arange(5), 2, 4, 16, layer=3)
    b = synth.tokens(rc, [4], [2, 3], 2, 4, 16, layer=3)
    for name in a:
        assert np.array_equal(a[name][4:5, 2:4], b[name]), name
    c = synth.tokens(rc, np.arange(6), np.arange(5), 2, 4, 16, layer=4)
    assert not np.array_equal(a["k"], c["k"])
    s_all = synth.state0(rc, np.arange(4), 3, 8, 8)
    s_one = synth.state0(rc, [2], 3, 8, 8)
    assert np.array_equal(s_all[2:3], s_one)


def test_domains_and_rounding():
    rc = synth.Recipe(seed=7, in_dtype="bf16", dist="stress")
    t = synth.tokens(rc, np.arange(8), np.arange(16), 4, 8, 128)
    for name in ("q", "k", "v"):
        x = t[name]
        assert x.dtype == np.float32
        assert np.array_equal(synth.round_bf16(x), x)          # bf16-exact
    n = np.linalg.norm(t["k"].astype(np.float64), axis=-1)
    assert np.all(np.abs(n - 1.0) < 1e-2)
    assert np.all((t["alpha"] > 0.9) & (t["alpha"] <= 1.0))
    assert np.all((t["beta"] > 0.0) & (t["beta"] < 1.0))
    rq = synth.Recipe(seed=7, in_dtype="f32", dist="qwen")
    tq = synth.tokens(rq, [0], np.arange(4), 2, 2, 128)
    nq = np.linalg.norm(tq["q"].astype(np.float64), axis=-1)
    np.testing.assert_allclose(nq, 1 / np.sqrt(128), rtol=1e-6)


def test_round_bf16_rne():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -2.5, 0.0], dtype=np.float32)
    r = synth.round_bf16(x)
    # 1 + 2^-8 is a tie between 1 and 1 + 2^-7 -> even (1.0); 1 + 3*2^-9 rounds up
    assert r[0] == 1.0 and r[1] == 1.0 and r[2] == np.float32(1.0 + 2 ** -7)
    assert r[3] == -2.5 and r[4] == 0.0


def test_state0_scale_and_acceptance():
    rc = synth.Recipe(seed=99)
    s = synth.state0(rc, np.arange(4), 4, 128, 128)
    assert abs(s.std() - np.sqrt(1 / 512)) < 2e-3
    acc = synth.n_accepted(rc, np.arange(4096), 4, round_idx=0)
    assert acc.min() >= 0 and acc.max() <= 4
    # P(n_acc = 4) = 0.7^4
    assert abs(np.mean(acc == 4) - 0.7 ** 4) < 0.03
    assert abs(np.mean(acc == 0) - 0.3) < 0.03
    acc2 = synth.n_accepted(rc, np.arange(4096), 4, round_idx=0)
    assert np.array_equal(acc, acc2)
