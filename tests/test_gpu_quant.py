"""GPU parity: quantisers, reductions, DSGC, DCLR, SGD vs the CPU oracle.

Bit-exact: int8 payloads (nearest and stochastic, incl. the LCG stream state
after the call), max_abs, the chosen clip on grid-only searches.
Tolerance (double sums reduced in a different order): the sums rel 1e-9;
d_c = 1 - cos absolute 1e-9 (the reference's own sequential double sum over
6.4M terms carries ~1e-11 relative error, amplified 1/d_c ~ 200x by the
cancellation); phi rel 1e-8; eps_norm / ghat_sqnorm rel 1e-9; clips from
golden refinement equal or dc(c_gpu) <= dc(c_ref) + 1e-9.
"""
import numpy as np
import pytest
import torch

from oracle import lib as O

pytestmark = pytest.mark.gpu
REL = 1e-9
DC_ABS = 1e-9


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def test_quantize_nearest_bit_exact(ops):
    rng = np.random.default_rng(0)
    for trial in range(20):
        x = (rng.standard_normal(50_000) * rng.uniform(1e-6, 10)).astype(np.float32)
        clip = float(np.abs(x).max() * rng.uniform(0.05, 1.3))
        ref, _ = O.quantize(x, clip)
        got = ops.quantize(t(x), clip).cpu().numpy()
        np.testing.assert_array_equal(got, ref)


def test_quantize_nearest_ties_and_edges(ops):
    # exact half-integer multiples of s (ties away from zero) and neighbours
    for clip in (127.0, 1.27, 0.8, 3e-7, 160.0):
        s = O.quant_scale(clip)
        k = np.arange(-130, 131, dtype=np.float64)
        base = ((k + 0.5) * s).astype(np.float32)
        x = np.concatenate([base, np.nextafter(base, np.float32(np.inf)), np.nextafter(base, np.float32(-np.inf)),
                            np.array([clip, -clip, 2 * clip, 0.0, -0.0], np.float32)]).astype(np.float32)
        ref, _ = O.quantize(x, clip)
        got = ops.quantize(t(x), clip).cpu().numpy()
        np.testing.assert_array_equal(got, ref)


def test_quantize_stochastic_bit_exact_and_stream(ops):
    rng = np.random.default_rng(1)
    for trial, n in enumerate((4, 1000, 65536 * 3 + 4, 1_000_000)):
        x = (rng.standard_normal(n) * 1e-3).astype(np.float32)
        x[rng.random(n) < 0.3] = 0.0
        clip = float(np.abs(x).max() * 0.7)
        seed = 1234 + trial
        ref, st_ref = O.quantize(x, clip, True, seed)
        st = ops.new_lcg_state(seed)
        got = ops.quantize(t(x), clip, stochastic=True, stream_state=st).cpu().numpy()
        np.testing.assert_array_equal(got, ref)
        assert ops.lcg_value(st) == st_ref


def _lcg_draws(seed, n):
    """u_i = X_{i+1} * 2^-32 of the reference LcgStream (quantize.hpp:32-50)."""
    out = np.empty(n, np.float64)
    x = seed & 0xFFFFFFFF
    for i in range(n):
        x = (1664525 * x + 1013904223) & 0xFFFFFFFF
        out[i] = x * 2.0 ** -32
    return out


@pytest.mark.parametrize("clip", [0.9, 3e-5, 127.0])
def test_quantize_stochastic_adversarial(ops, clip):
    """Inputs placed so that frac(x/s) sits on, or within a few ulp of, the
    element's own draw u (the FP32 fast path's decision boundary), plus exact
    multiples of s, the clip edges and values beyond the clip."""
    n, seed = 40_000, 99
    u = _lcg_draws(seed, n)
    s = O.quant_scale(clip)
    rng = np.random.default_rng(5)
    k = rng.integers(-127, 127, n).astype(np.float64)
    x = ((k + u) * s).astype(np.float32)
    kind = rng.integers(0, 6, n)
    x = np.where(kind == 1, np.nextafter(x, np.float32(np.inf)), x)
    x = np.where(kind == 2, np.nextafter(x, np.float32(-np.inf)), x)
    x = np.where(kind == 3, (k * s).astype(np.float32), x)
    edge = np.array([clip, -clip, np.nextafter(np.float32(clip), np.float32(0)), 2 * clip, -3 * clip], np.float32)
    x = np.where(kind == 4, edge[rng.integers(0, len(edge), n)], x).astype(np.float32)
    ref, st_ref = O.quantize(x, clip, True, seed)
    st = ops.new_lcg_state(seed)
    got = ops.quantize(t(x), clip, stochastic=True, stream_state=st).cpu().numpy()
    np.testing.assert_array_equal(got, ref)
    assert ops.lcg_value(st) == st_ref


@pytest.mark.parametrize("clip", [1e-37, 4e-39, 2e-41, 3e38])
def test_quantize_subnormal_scale(ops, clip):
    """clip < 127 * FLT_MIN makes s = float(clip / 127) subnormal: the FP32 fast
    paths do not hold there and the kernels take the FP64 formula."""
    rng = np.random.default_rng(int(np.log2(clip)) % 1000)
    big = float(np.finfo(np.float32).max)
    x = np.clip(rng.standard_normal(30_000) * clip * 0.6, -big, big).astype(np.float32)
    x[:4] = [clip, -clip, min(3 * clip, big), 0.0]
    ref, _ = O.quantize(x, clip)
    np.testing.assert_array_equal(ops.quantize(t(x), clip).cpu().numpy(), ref)
    ref, st_ref = O.quantize(x, clip, True, 7)
    st = ops.new_lcg_state(7)
    np.testing.assert_array_equal(ops.quantize(t(x), clip, stochastic=True, stream_state=st).cpu().numpy(), ref)
    assert ops.lcg_value(st) == st_ref


def test_quantize_stochastic_odd_length(ops):
    x = np.linspace(-1, 1, 1001).astype(np.float32)
    ref, st_ref = O.quantize(x, 0.9, True, 77)
    st = ops.new_lcg_state(77)
    got = ops.quantize(t(x), 0.9, stochastic=True, stream_state=st).cpu().numpy()
    np.testing.assert_array_equal(got, ref)
    assert ops.lcg_value(st) == st_ref


def test_quantize_partitioned(ops):
    rng = np.random.default_rng(3)
    x = rng.standard_normal(1000).astype(np.float32)
    clip = float(np.abs(x).max())
    for parts in (1, 3, 8):
        np.testing.assert_array_equal(ops.quantize_partitioned(t(x), clip, 900, parts).cpu().numpy(),
                                      O.quantize_partitioned(x, clip, 900, parts))


def test_quantize_errors(ops):
    with pytest.raises(ValueError):
        ops.quantize(t(np.ones(4, np.float32)), 0.0)
    with pytest.raises(ValueError):
        ops.quantize(t(np.ones(4, np.float32)), 1.0, stochastic=True)
    ops.quantize(t(np.array([1.0, np.nan, 0, 0], np.float32)), 1.0)
    with pytest.raises(ArithmeticError):
        ops.check()


def test_nchw_to_nhwc_quantize_and_amax(ops):
    rng = np.random.default_rng(4)
    x = rng.standard_normal((3, 5, 7, 6)).astype(np.float32)
    clip = 2.0
    amax = torch.zeros(1, device="cuda")
    q = ops.quantize_act_nhwc(t(x), clip, c_pad=8, amax=amax)
    ref, _ = O.quantize(x, clip)
    qn = q.cpu().numpy()
    np.testing.assert_array_equal(qn[..., :5], ref.transpose(0, 2, 3, 1))
    assert (qn[..., 5:] == 0).all()
    assert float(amax.item()) == O.max_abs(x)


def test_weight_quantizer_layouts(ops):
    rng = np.random.default_rng(5)
    w = rng.standard_normal((6, 5, 3, 3)).astype(np.float32)
    clip = float(np.abs(w).max())
    q1, q2 = ops.quantize_weight(t(w), clip)
    ref, _ = O.quantize(w, clip)
    krsc = q1.cpu().numpy()[:, : 3 * 3 * 8].reshape(6, 3, 3, 8)
    np.testing.assert_array_equal(krsc[..., :5], ref.transpose(0, 2, 3, 1))
    crsk = q2.cpu().numpy()[:, : 3 * 3 * 8].reshape(5, 3, 3, 8)
    np.testing.assert_array_equal(crsk[..., :6], ref.transpose(1, 2, 3, 0))


def test_reductions(ops):
    rng = np.random.default_rng(6)
    x = rng.standard_normal(123_457).astype(np.float32)
    y = rng.standard_normal(123_457).astype(np.float32)
    assert ops.max_abs(t(x)) == O.max_abs(x)
    assert ops.sq_l2_norm(t(x)) == pytest.approx(O.sq_l2_norm(x), rel=REL)
    assert ops.dot(t(x), t(y)) == pytest.approx(O.dot(x, y), rel=1e-8)
    assert not ops.has_nonfinite(t(x))
    x[77] = np.inf
    assert ops.has_nonfinite(t(x))


def test_cosine_kats(ops):
    g = t(np.array([0.5, -1.0, 2.0], np.float32))
    assert abs(ops.cosine_distance(g, g)) < 1e-12
    a, b = t(np.array([1.0, 0.0], np.float32)), t(np.array([0.0, 1.0], np.float32))
    assert ops.cosine_distance(a, b) == pytest.approx(1.0)
    c = t(np.array([1.0, 1.0], np.float32))
    assert ops.cosine_distance(c, a) == pytest.approx(1 - 1 / np.sqrt(2), rel=1e-9)
    z = t(np.zeros(2, np.float32))
    assert ops.cosine_distance(z, z) == 0.0 and ops.cosine_distance(a, z) == 1.0 and ops.cosine_distance(z, a) == 1.0


def test_measure_dc(ops):
    g = O.gradient_like((100_000,), 7, 1e-4, 0.01)
    for clip in (1e-4, 5e-4, float(np.abs(g).max())):
        assert ops.measure_dc(t(g), clip) == pytest.approx(O.measure_dc(g, clip), abs=DC_ABS)


@pytest.mark.parametrize("seed", range(6))
def test_search_clip_grid_only_exact(seed, ops):
    g = O.gradient_like((20_000,), seed, 0.01, 0.01)
    ref = O.search_clip(g, 64, 0)
    got = ops.search_clip(t(g), 64, 0)
    assert got[0] == ref[0]
    assert got[1] == pytest.approx(ref[1], abs=DC_ABS)


@pytest.mark.parametrize("R,seed", [(32, 0), (32, 1), (32, 2), (8, 3), (17, 4), (31, 5), (32, 6), (32, 7)])
def test_search_clip_grid_histogram_exact(R, seed, ops):
    """R <= 32: the grid runs as one boundary-histogram pass (dsgc.cu K4H);
    same clip as the reference's 32 measure_dc calls, d_c within the sums'
    rounding.  Sizes straddle the one-block and many-block grids."""
    n = [20_000, 300_000, 2_000_003, 50_000, 123_457, 1_000, 4_000_000, 77_777][seed]
    g = O.gradient_like((n,), 300 + seed, 1e-3, 0.01)
    ref = O.search_clip(g, R, 0)
    got = ops.search_clip(t(g), R, 0)
    assert got[0] == ref[0]
    assert got[1] == pytest.approx(ref[1], abs=DC_ABS)


def test_search_clip_grid_histogram_adversarial(ops):
    """Elements exactly on (and one ulp either side of) quantisation
    boundaries of every grid candidate, duplicates of max|g|, signed zeros,
    and a constant tensor (every element in the top bin)."""
    rng = np.random.default_rng(11)
    m = np.float32(0.37)
    R = 32
    vals = [m]
    for i in range(1, R + 1):
        c = np.float32(m * np.float32(np.float32(i) / np.float32(R)))
        s = np.float32(c / np.float32(127))
        for q in range(0, 127, 3):
            b = np.float32((q + 0.5) * s)
            vals += [b, np.nextafter(b, np.float32(0)), np.nextafter(b, np.float32(1))]
    v = np.array(vals, np.float32)
    g = np.concatenate([v, -v, rng.choice(v, 200_000), np.full(1000, m, np.float32),
                        np.zeros(100, np.float32), -np.zeros(100, np.float32)]).astype(np.float32)
    rng.shuffle(g)
    for rounds in (0, 2):
        ref = O.search_clip(g, R, rounds)
        got = ops.search_clip(t(g), R, rounds)
        assert got[0] == ref[0] or O.measure_dc(g, got[0]) <= ref[1] + DC_ABS
        assert got[1] == pytest.approx(ref[1], abs=DC_ABS)
    # constant tensor: every candidate's d_c is 0 up to rounding (the pick is a
    # rounding tie-break), so only the objective is compared
    c = np.full(100_000, np.float32(-2.5), np.float32)
    got, ref = ops.search_clip(t(c), R, 0), O.search_clip(c, R, 0)
    assert got[1] == pytest.approx(ref[1], abs=DC_ABS)
    assert O.measure_dc(c, got[0]) <= ref[1] + DC_ABS


@pytest.mark.parametrize("seed", range(6))
def test_search_clip_refined(seed, ops):
    g = O.gradient_like((30_000,), 100 + seed, 1e-4, 0.02)
    ref = O.search_clip(g, 32, 2)
    got = ops.search_clip(t(g), 32, 2)
    assert got[0] == ref[0] or O.measure_dc(g, got[0]) <= ref[1] + DC_ABS
    assert got[1] == pytest.approx(ref[1], abs=DC_ABS)


@pytest.mark.parametrize("mag", [1e-37, 3e-39, 1e37, 3e38])
def test_search_clip_extreme_magnitudes(mag, ops):
    """The candidate pass rebuilds the double x̂ from the float bits with
    power-of-two scalings; scales below FLT_MIN (subnormal x̂) take the multiply
    path, and the largest finite g still scales without overflow."""
    g = O.gradient_like((20_000,), 3, 1e-4, 0.02)
    g = (g / np.abs(g).max() * np.float32(mag)).astype(np.float32)
    assert np.isfinite(g).all() and np.abs(g).max() > 0
    ref = O.search_clip(g, 32, 0)
    got = ops.search_clip(t(g), 32, 0)
    assert got[0] == ref[0]
    assert got[1] == pytest.approx(ref[1], abs=DC_ABS)
    for clip in (ref[0], float(np.abs(g).max()) / 7):
        assert ops.measure_dc(t(g), clip) == pytest.approx(O.measure_dc(g, clip), abs=DC_ABS)


def test_search_clip_kats(ops):
    s = 0.01
    g = (np.arange(-127, 128) * np.float32(s)).astype(np.float32)
    c, dc = ops.search_clip(t(g))
    assert c == O.max_abs(g) and abs(dc) < 1e-12
    # lone outlier, R = 512 (more candidates than one 32-wide pass)
    rng = np.random.default_rng(5)
    g = np.where(rng.random(1000) < 0.5, -0.01, 0.01).astype(np.float32)
    g[999] = 10.0
    ref = O.search_clip(g, 512, 0)
    got = ops.search_clip(t(g), 512, 0)
    assert got[0] == ref[0] and got[0] < 10.0
    assert ops.search_clip(t(np.zeros(64, np.float32)), 32, 2, prev_clip=0.5) == (0.5, 0.0)
    with pytest.raises(ValueError):
        ops.search_clip(t(g), 4, 0)


def test_maybe_update_schedule(ops):
    g = O.gradient_like((512 * 8,), 30, 0.01, 0.01)
    g2 = O.gradient_like((512 * 8,), 31, 0.01, 0.01)
    st = ops.DsgcState(period=100)
    ref = O.new_clip_state(100)
    O.maybe_update(ref, g, 0)
    v = ops.maybe_update(st, t(g), 0)
    assert v.clip == ref.clip and v.iter_of_last_update == 0
    for it in (1, 50, 99):
        O.maybe_update(ref, g2, it)
        v = ops.maybe_update(st, t(g2), it)
        assert v.clip == ref.clip and v.iter_of_last_update == 0
        assert v.last_dc == pytest.approx(ref.last_dc, abs=DC_ABS)
    v = ops.maybe_update(st, t(g2), 100)
    assert v.iter_of_last_update == 100
    with pytest.raises(ValueError):
        ops.maybe_update(st, t(g2), 99)
    # all-zero gradient keeps the clip, d_c = 0
    st1 = ops.DsgcState(period=1)
    v0 = ops.maybe_update(st1, t(g), 0)
    v1 = ops.maybe_update(st1, t(np.zeros_like(g)), 1)
    assert v1.clip == v0.clip and v1.last_dc == 0.0


def _qg_compare(ops, g_nchw, iters, seed=99, search=True, nhwc=True):
    """Run quantize_gradient for several iterations on GPU and oracle."""
    st = ops.DsgcState(period=2)
    ref = O.new_clip_state(2)
    lcg = ops.new_lcg_state(seed)
    stream = seed
    for it in range(iters):
        g = g_nchw[it % len(g_nchw)]
        q_ref, s_ref, stream, stats = O.quantize_gradient(ref, g, it, stream, search=search)
        if nhwc:
            q = ops.quantize_gradient(st, t(g.transpose(0, 2, 3, 1)), it, lcg, nhwc=True, search_enabled=search)
            qn = q.cpu().numpy().transpose(0, 3, 1, 2)
        else:
            qn = ops.quantize_gradient(st, t(g), it, lcg, search_enabled=search).cpu().numpy()
        v = st.sync()
        assert v.clip == ref.clip, (it, v.clip, ref.clip)
        np.testing.assert_array_equal(qn, q_ref, err_msg=f"iter {it}")
        assert ops.lcg_value(lcg) == stream
        assert v.scale == s_ref
        assert v.last_dc == pytest.approx(stats["dc"], abs=DC_ABS)
        assert v.lr_scale == pytest.approx(stats["lr_scale"], rel=1e-8)
        assert v.eps_norm == pytest.approx(stats["eps_norm"], rel=REL)
        assert v.ghat_sqnorm == pytest.approx(stats["ghat_sqnorm"], rel=REL)


def test_quantize_gradient_nhwc_matches_oracle(ops):
    gs = [O.gradient_like((4, 16, 10, 10), s, 1e-4, 0.01) for s in (1, 2, 3)]
    _qg_compare(ops, gs, 5)


def test_quantize_gradient_flat_and_search_disabled(ops):
    gs = [O.gradient_like((2, 8, 6, 6), s, 1e-3, 0.01) for s in (4, 5)]
    _qg_compare(ops, gs, 4, nhwc=False)
    _qg_compare(ops, gs, 3, search=False)


def test_quantize_gradient_zero_skip_consumes_no_draws(ops):
    gs = [O.gradient_like((2, 8, 4, 4), 6, 1e-3, 0.0), np.zeros((2, 8, 4, 4), np.float32)]
    _qg_compare(ops, gs, 4)


def test_quantize_gradient_subnormal_scale(ops):
    for mag in (1e-37, 1e35):
        gs = [(O.gradient_like((2, 8, 6, 6), s, 1e-3, 0.01) * np.float32(mag)).astype(np.float32) for s in (7, 8)]
        _qg_compare(ops, gs, 3)


def test_quantize_gradient_config1_full(ops):
    g = O.gradient_like((32, 64, 56, 56), 11, 1e-4, 0.01)
    _qg_compare(ops, [g], 2)


def test_scale_factor_kats(ops):
    assert ops.scale_factor(0.0) == 1.0
    assert ops.scale_factor(0.05) == pytest.approx(np.exp(-1.0), rel=1e-12)
    assert ops.scale_factor(1.0) == 0.1
    assert ops.scale_factor(0.3, form="linear") == pytest.approx(0.7)
    assert ops.scale_factor(0.3, form="quadratic") == pytest.approx(0.91)
    for bad in ((-0.1,), (2.1,)):
        with pytest.raises(ValueError):
            ops.scale_factor(*bad)
    with pytest.raises(ValueError):
        ops.scale_factor(0.5, alpha=0.0)
    with pytest.raises(ValueError):
        ops.scale_factor(0.5, beta=1.5)
    lr = ops.effective_lr(0.1, {"a": 0.0, "b": 2.0})
    assert lr["a"] == 0.1 and lr["b"] == pytest.approx(0.01)


def test_sgd_dclr_matches_oracle(ops):
    rng = np.random.default_rng(8)
    w = rng.standard_normal(100_003).astype(np.float32)
    gr = (rng.standard_normal(100_003) * 1e-3).astype(np.float32)
    st = ops.DsgcState()
    v = st.view()
    v.lr_scale = 0.37
    st.write(v)
    wt = t(w)
    ops.sgd_dclr_(wt, t(gr), 0.05, st)
    np.testing.assert_array_equal(wt.cpu().numpy(), O.sgd_update(w, gr, 0.05 * 0.37))


@pytest.mark.parametrize("same", [True, False])
def test_quantize_nearest_shared(same, ops):
    """i8t_quantize_nearest_shared: with the reference clip bit-equal the result
    is the reference int8 tensor and the running max is taken over; otherwise
    the plain nearest quantiser of x (payload and running max)."""
    rng = np.random.default_rng(41)
    x = rng.standard_normal(4096 * 3).astype(np.float32)
    xt = t(x)
    ref_clip = torch.tensor([2.5], device="cuda")
    ref_amax = torch.tensor([3.25], device="cuda")
    ref_q = torch.randint(-127, 128, (x.size,), dtype=torch.int8, device="cuda")
    clip = torch.tensor([2.5 if same else 1.75], device="cuda")
    q = torch.empty_like(ref_q)
    amax = torch.tensor([0.5], device="cuda")
    ops.call("i8t_quantize_nearest_shared", ops.ctx(), ops._p(xt), x.size, ops._p(clip), ops._p(ref_clip),
             ops._p(ref_q), ops._p(ref_amax), ops._p(q), ops._p(amax))
    torch.cuda.synchronize()
    if same:
        assert torch.equal(q, ref_q) and float(amax) == 3.25
    else:
        assert np.array_equal(q.cpu().numpy(), O.quantize(x, 1.75)[0])
        assert float(amax) == max(0.5, float(np.abs(x).max()))


@pytest.mark.parametrize("rows", [4096, 4097])
def test_quantize_nearest_rows_rgb_padding(rows, ops):
    """i8t_quantize_nearest_rows for 3-channel pixels padded to 4 (the stem
    input; rows % 4 == 0 takes the four-pixels-per-thread kernel): payload
    equal to the reference quantiser, pad byte 0, running max|x|."""
    rng = np.random.default_rng(81)
    x = (rng.standard_normal((rows, 3)) * 2).astype(np.float32)
    q = torch.full((rows, 4), 77, dtype=torch.int8, device="cuda")
    amax = torch.zeros(1, device="cuda")
    clip = torch.tensor([3.5], device="cuda")
    ops.call("i8t_quantize_nearest_rows", ops.ctx(), ops._p(t(x)), rows, 3, ops._p(clip), ops._p(q), 4, ops._p(amax), 0)
    ref, _ = O.quantize(x, 3.5)
    qn = q.cpu().numpy()
    assert np.array_equal(qn[:, :3], ref.reshape(rows, 3)) and (qn[:, 3] == 0).all()
    assert float(amax) == float(np.abs(x).max())
