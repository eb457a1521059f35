"""Pin the CPU oracle (oracle/oracle.c) against golden vectors dumped from the
compiled reference (tests/golden/make_golden.py) and against the known-answer
tests of the reference's own unit tests (proj/tests/*.cpp).  CPU only."""
import os

import numpy as np
import pytest

from oracle import lib as O

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


# ------------------------------------------------------------------ golden vectors
@pytest.mark.parametrize("seed", [0, 12345, 99, 0xFFFFFFFF])
def test_lcg_golden(seed):
    st, got = seed, []
    for _ in range(8):
        v, st = O.lcg_next(st)
        got.append(v)
    np.testing.assert_array_equal(np.array(got, np.uint32), G[f"lcg_{seed}"])
    assert O.lcg_jump(seed, 8) == G[f"lcg_{seed}"][-1]


@pytest.mark.parametrize("i", range(6))
def test_quantize_golden(i):
    x, clip = G[f"q{i}_x"], float(G[f"q{i}_meta"][0])
    seed, st_after = (int(v) for v in G[f"q{i}_seed"])
    np.testing.assert_array_equal(O.quantize(x, clip)[0], G[f"q{i}_nearest"])
    q, st = O.quantize(x, clip, True, seed)
    np.testing.assert_array_equal(q, G[f"q{i}_stoch"])
    assert st == st_after


def test_quantize_ties_and_partitioned_golden():
    np.testing.assert_array_equal(O.quantize(G["qties_x"], 1.27)[0], G["qties_nearest"])
    x = G["qpart_x"]
    np.testing.assert_array_equal(O.quantize_partitioned(x, float(np.abs(x).max()), 900, 8), G["qpart_q"])


@pytest.mark.parametrize("i", range(16))
def test_conv_golden(i):
    n, c, h, w, k, kh, kw, s, p, dw = (int(v) for v in G[f"conv{i}_g"])
    g = O.geom(n, c, h, w, k, kh, kw, s, p, bool(dw), floor_mode=False)
    sa, sw, sg = O.quant_scale(1.27), O.quant_scale(12.7), O.quant_scale(0.5)
    _, z = O.conv_fwd(G[f"conv{i}_qa"], G[f"conv{i}_qw"], g, sa, sw)
    np.testing.assert_array_equal(z, G[f"conv{i}_z"])
    _, ga = O.conv_dgrad(G[f"conv{i}_qg"], G[f"conv{i}_qw"], g, sg, sw)
    np.testing.assert_array_equal(ga, G[f"conv{i}_ga"])
    _, gw = O.conv_wgrad(G[f"conv{i}_qg"], G[f"conv{i}_qa"], g, sg, sa)
    np.testing.assert_array_equal(gw, G[f"conv{i}_gw"])


@pytest.mark.parametrize("i", range(5))
def test_search_golden(i):
    g = G[f"search{i}_g"]
    grid, rounds = (int(v) for v in G[f"search{i}_cfg"])
    c, d = O.search_clip(g, grid, rounds)
    assert np.float32(c) == np.float32(G[f"search{i}_res"][0])
    assert d == G[f"search{i}_res"][1]
    for cc, dd in zip((1e-3, 5e-3, 2e-2), G[f"search{i}_dcs"]):
        assert O.measure_dc(g, cc) == dd


def test_maybe_update_golden():
    st = O.ClipState(0.0, 0.0, -1, 3)
    g1, g2 = G["maybe_g1"], G["maybe_g2"]
    for it, g in enumerate([g1, g2, g2, g1, np.zeros(512, np.float32), g2, g1]):
        O.maybe_update(st, g, it)
        exp = G["maybe_seq"][it]
        assert np.float32(st.clip) == np.float32(exp[0]) and st.last_dc == exp[1] and st.iter_of_last_update == exp[2]


def test_phi_golden():
    for row, d in zip(G["phi"], np.linspace(0.0, 2.0, 41)):
        for f, form in enumerate(("exp", "linear", "quadratic")):
            assert O.scale_factor(d, 20.0, 0.1, form) == row[f]


@pytest.mark.parametrize("li", range(2))
def test_layer_step_golden(li):
    n, c, h, w, k, kh, kw, s, p, dw = (int(v) for v in G[f"layer{li}_g"])
    g = O.geom(n, c, h, w, k, kh, kw, s, p, floor_mode=False)
    W, X, GO = G[f"layer{li}_W"], G[f"layer{li}_X"], G[f"layer{li}_GO"]
    stats = G[f"layer{li}_stats"]
    cw, ca = max(O.max_abs(W), 1e-12), max(O.max_abs(X), 1e-12)
    assert np.float32(cw) == np.float32(stats[0]) and np.float32(ca) == np.float32(stats[1])
    qw, _ = O.quantize(W, cw)
    qa, _ = O.quantize(X, ca)
    _, z = O.conv_fwd(qa, qw, g, O.quant_scale(ca), O.quant_scale(cw))
    np.testing.assert_array_equal(z, G[f"layer{li}_z"])
    st = O.new_clip_state(100)
    seed, st_after = (int(v) for v in G[f"layer{li}_stream"])
    qg, sg, stream, ss = O.quantize_gradient(st, GO, 0, seed)
    assert stream == st_after
    assert np.float32(st.clip) == np.float32(stats[2])
    assert (ss["dc"], ss["lr_scale"], ss["eps_norm"], ss["ghat_sqnorm"]) == tuple(stats[3:7])
    _, ga = O.conv_dgrad(qg, qw, g, sg, O.quant_scale(cw))
    _, gw = O.conv_wgrad(qg, qa, g, sg, O.quant_scale(ca))
    np.testing.assert_array_equal(ga, G[f"layer{li}_ga"])
    np.testing.assert_array_equal(gw, G[f"layer{li}_gw"])


# ------------------------------------------------------------------ reference KATs
def test_lcg_kat():  # test_quantize.cpp:11-24
    v, st = O.lcg_next(0)
    assert v == 1013904223
    v2, _ = O.lcg_next(st)
    assert v2 == (1664525 * 1013904223 + 1013904223) % 2**32


def test_lcg_no_repeat_prefix():  # test_quantize.cpp:26-31 (2^16 prefix here; jump-consistency below)
    st, seen = 99, set()
    for _ in range(1 << 16):
        v, st = O.lcg_next(st)
        assert v not in seen
        seen.add(v)
    assert O.lcg_jump(99, 1 << 16) == st


def test_quantize_basics():  # test_quantize.cpp:33-45
    assert O.quant_scale(127.0) == 1.0
    assert (O.quantize(np.zeros(3, np.float32), 127.0)[0] == 0).all()
    assert O.quantize(np.array([200.0], np.float32), 127.0)[0][0] == 127
    assert O.quantize(np.array([-200.0], np.float32), 127.0)[0][0] == -127


def test_stochastic_rates():  # test_quantize.cpp:47-61
    n = 100_000
    q, _ = O.quantize(np.full(n, 3.4, np.float32), 127.0, True, 2024)
    assert set(np.unique(q)) <= {3, 4}
    assert abs(q.mean() - 3.4) < 3 * np.sqrt(0.24) / np.sqrt(n)


def test_quantize_errors():  # test_quantize.cpp:63-73
    with pytest.raises(ArithmeticError):
        O.quantize(np.array([np.nan], np.float32), 1.0)
    with pytest.raises(ValueError):
        O.quant_scale(0.0)
    with pytest.raises(ValueError):
        O.quant_scale(-1.0)


def test_dequantize_kat():  # test_quantize.cpp:75-83
    out = O.dequantize(np.array([127, 0], np.int8), O.quant_scale(1.27))
    assert out[0] == pytest.approx(1.27, rel=1e-6) and out[1] == 0.0


def test_nearest_roundtrip_half_step():  # test_quantize.cpp:85-95
    c = np.float32(0.8)
    s = O.quant_scale(float(c))
    x = (-c + 2.0 * c * np.arange(10001, dtype=np.float32) / np.float32(10000)).astype(np.float32)
    back = O.dequantize(O.quantize(x, float(c))[0], s)
    assert (np.abs(back - x) <= s * 0.5 * (1 + 1e-5)).all()


def test_stochastic_unbiased():  # test_quantize.cpp:97-110
    n = 100_000
    for x in (-0.83, -0.31, 0.0, 0.204, 0.77):
        q, _ = O.quantize(np.full(n, x, np.float32), 1.0, True, 7)
        mean = O.dequantize(q, O.quant_scale(1.0)).astype(np.float64).mean()
        assert abs(mean - np.float32(x)) < 4 * O.quant_scale(1.0) / np.sqrt(12 * n)


def test_one_draw_per_element():  # test_quantize.cpp:112-126
    x = O.gaussian((257,), 5)
    clip = O.max_abs(x)
    a, s1 = O.quantize(x, clip, True, 31337)
    b, s2 = O.quantize(x, clip, True, 31337)
    assert (a == b).all() and s1 == s2 == O.lcg_jump(31337, 257)


def test_idempotence_and_symmetry():  # test_quantize.cpp:128-141
    x = O.gaussian((512,), 11, 0.3)
    q1, _ = O.quantize(x, 0.7)
    q2, _ = O.quantize(O.dequantize(q1, O.quant_scale(0.7)), 0.7)
    assert (q1 == q2).all()
    assert (O.quantize(-x, 0.7)[0] == -q1).all()


def test_gemm_kats():  # test_kernels.cpp:79-118
    assert O.gemm_i8(np.array([[1, 2], [3, 4]], np.int8), np.array([[5, 6], [7, 8]], np.int8)).tolist() == [[19, 22], [43, 50]]
    assert O.gemm_i8(np.full((1, 4), 127, np.int8), np.full((4, 1), 127, np.int8))[0, 0] == 64516
    rng = np.random.default_rng(17)
    for _ in range(25):
        m, k, n = (int(v) for v in 1 + rng.integers(0, 16, 3))
        a = rng.integers(-127, 128, (m, k)).astype(np.int8)
        b = rng.integers(-127, 128, (k, n)).astype(np.int8)
        np.testing.assert_array_equal(O.gemm_i8(a, b), a.astype(np.int64) @ b.astype(np.int64))


def test_im2col_layouts():  # test_kernels.cpp:144-161
    x = np.arange(1, 10, dtype=np.int8).reshape(1, 1, 3, 3)
    col = O.im2col_i8(x, O.geom(1, 1, 3, 3, 1, 2, 2, floor_mode=False))
    assert col[:, 0].tolist() == [1, 2, 4, 5]
    col2 = O.im2col_i8(x, O.geom(1, 1, 3, 3, 1, 3, 3, floor_mode=False))
    assert col2[:, 0].tolist() == list(range(1, 10))


def test_conv_1x1_matrix_calculus():  # test_kernels.cpp:271-300
    rng = np.random.default_rng(99)
    g = O.geom(1, 3, 2, 2, 4, 1, 1, floor_mode=False)
    xa = rng.integers(-127, 128, (1, 3, 2, 2)).astype(np.int8)
    xw = rng.integers(-127, 128, (4, 3, 1, 1)).astype(np.int8)
    xg = rng.integers(-127, 128, (1, 4, 2, 2)).astype(np.int8)
    s = O.quant_scale(1.27)
    wacc, _ = O.conv_wgrad(xg, xa, g, s, s)
    dacc, _ = O.conv_dgrad(xg, xw, g, s, s)
    A, Wm, Gm = xa.reshape(3, 4).astype(np.int64), xw.reshape(4, 3).astype(np.int64), xg.reshape(4, 4).astype(np.int64)
    np.testing.assert_array_equal(wacc.reshape(4, 3), Gm @ A.T)
    np.testing.assert_array_equal(dacc.reshape(3, 4), Wm.T @ Gm)


def test_geometry_validation():  # conv.cpp:11-18 + EXT floor mode
    with pytest.raises(ValueError):
        O.out_hw(O.geom(1, 1, 4, 4, 1, 3, 3, stride=2, pad=0, floor_mode=False))
    assert O.out_hw(O.geom(1, 1, 4, 4, 1, 3, 3, stride=2, pad=0, floor_mode=True)) == (1, 1)
    with pytest.raises(ValueError):
        O.out_hw(O.geom(1, 2, 4, 4, 3, 3, 3, depthwise=True))


def test_cosine_kats():  # test_clip.cpp:38-52
    g = np.array([0.5, -1.0, 2.0], np.float32)
    assert abs(O.cosine_distance(g, g)) < 1e-12
    a, b, c, z = (np.array(v, np.float32) for v in ([1, 0], [0, 1], [1, 1], [0, 0]))
    assert O.cosine_distance(a, b) == pytest.approx(1.0)
    assert O.cosine_distance(c, a) == pytest.approx(1 - 1 / np.sqrt(2), rel=1e-9)
    assert O.cosine_distance(z, z) == 0.0 and O.cosine_distance(a, z) == 1.0 and O.cosine_distance(z, a) == 1.0


def test_search_kats():  # test_clip.cpp:61-129
    g = (np.arange(-127, 128) * np.float32(0.01)).astype(np.float32)
    c, dc = O.search_clip(g)
    assert c == O.max_abs(g) and abs(dc) < 1e-12
    rng = np.random.default_rng(5)
    g = np.where(rng.random(1000) < 0.5, -0.01, 0.01).astype(np.float32)
    g[999] = 10.0
    c, dc = O.search_clip(g, 512, 0)
    assert c < 10.0 and dc < O.measure_dc(g, 10.0)
    for seed in range(10, 18):
        g = O.gradient_like((1024,), seed, 0.01, 0.02)
        c, dc = O.search_clip(g)
        assert dc <= O.measure_dc(g, O.max_abs(g)) + 1e-15 and 0 < c <= O.max_abs(g)
    base = O.search_clip(O.gradient_like((1024,), 21, 0.01, 0.01))
    for k in (2.0, 4.0, 0.5):
        r = O.search_clip(np.float32(k) * O.gradient_like((1024,), 21, 0.01, 0.01))
        assert r[0] == np.float32(k) * np.float32(base[0]) and r[1] == base[1]
    with pytest.raises(ValueError):
        O.search_clip(g, 4, 0)


def test_lr_scale_kats():  # test_lr_scale.cpp:8-72
    assert O.scale_factor(0.0) == 1.0
    assert O.scale_factor(0.05) == pytest.approx(np.exp(-1.0), rel=1e-12)
    assert O.scale_factor(1.0) == 0.1
    assert O.scale_factor(0.3, form="linear") == pytest.approx(0.7)
    assert O.scale_factor(0.3, form="quadratic") == pytest.approx(0.91)
    for form in ("exp", "linear", "quadratic"):
        prev = 2.0
        for i in range(201):
            f = O.scale_factor(2.0 * i / 200, form=form)
            assert 0.1 <= f <= 1.0 and f <= prev
            prev = f
    for bad in (dict(dc=-0.1), dict(dc=2.1), dict(dc=0.5, alpha=0.0), dict(dc=0.5, beta=0.0), dict(dc=0.5, beta=1.5)):
        with pytest.raises(ValueError):
            O.scale_factor(**bad)
