"""Randomised cross-check of the C restatement against the compiled reference
(oracle/_ref).  Runs only where the reference was built (this dev
container); the GPU box relies on tests/golden/ instead."""
import numpy as np
import pytest

from oracle import lib as O
from oracle import ref as R

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (needs /root/reference)")


def test_quantize_random():
    rng = np.random.default_rng(0)
    for trial in range(30):
        x = (rng.standard_normal(4000) * rng.uniform(1e-6, 10)).astype(np.float32)
        clip = float(np.abs(x).max() * rng.uniform(0.05, 1.3))
        assert (O.quantize(x, clip)[0] == R.quantize(x, clip)[0]).all()
        qa, sa = O.quantize(x, clip, True, 7 + trial)
        qb, sb = R.quantize(x, clip, True, 7 + trial)
        assert (qa == qb).all() and sa == sb


def test_search_random():
    for seed in range(40):
        g = O.gradient_like((3000,), seed, 10.0 ** -(seed % 6), 0.02)
        assert O.search_clip(g) == R.search_clip(g)
        assert O.search_clip(g, 16, 4) == R.search_clip(g, 16, 4)


def test_conv_random():
    rng = np.random.default_rng(1)
    done = 0
    while done < 30:
        n, c, k, kh = (int(v) for v in (rng.integers(1, 3), rng.integers(1, 6), rng.integers(1, 6), rng.integers(1, 4)))
        s, p, dw = int(rng.integers(1, 3)), int(rng.integers(0, 2)), done % 5 == 4
        k = c if dw else k
        h = (int(rng.integers(1, 5)) - 1) * s + kh - 2 * p
        w = (int(rng.integers(1, 5)) - 1) * s + kh - 2 * p
        if h < 1 or w < 1:
            continue
        gv = R.gvec(n, c, h, w, k, kh, kh, s, p, dw)
        g = O.geom(n, c, h, w, k, kh, kh, s, p, dw, floor_mode=False)
        qa = rng.integers(-127, 128, (n, c, h, w)).astype(np.int8)
        qw = rng.integers(-127, 128, R.w_shape(gv)).astype(np.int8)
        qg = rng.integers(-127, 128, R.out_shape(gv)).astype(np.int8)
        sa, sw, sg = O.quant_scale(0.9), O.quant_scale(3.1), O.quant_scale(1e-3)
        assert (O.conv_fwd(qa, qw, g, sa, sw)[1] == R.conv2d_q(qa, 0.9, qw, 3.1, gv)).all()
        gw, ga = R.conv2d_backward_q(qg, 1e-3, qa, 0.9, qw, 3.1, gv)
        assert (O.conv_dgrad(qg, qw, g, sg, sw)[1] == ga).all()
        assert (O.conv_wgrad(qg, qa, g, sg, sa)[1] == gw).all()
        done += 1


def test_layer_step_multi_iter():
    """Three INT8 Conv2d steps through the reference layer API (period 2) vs the
    restated quantize_gradient + conv ops, stream carried across steps."""
    n, c, h, k = 2, 8, 8, 16
    gv = R.gvec(n, c, h, h, k, 3, 3, 1, 1)
    g = O.geom(n, c, h, h, k, 3, 3, 1, 1, floor_mode=False)
    cs_ref, cs = O.ClipState(0.0, 0.0, -1, 2), O.new_clip_state(2)
    stream_ref = stream = 5
    for it in range(3):
        W = O.gaussian((k, c, 3, 3), 10 + it, 0.2)
        X = O.gaussian((n, c, h, h), 20 + it, 1.0, True)
        GO = O.gradient_like((n, k, h, h), 30 + it, 1e-4, 0.01)
        z, gw, ga, stream_ref, stats = R.conv_layer_step(gv, W, X, GO, it, stream_ref, cs_ref, period=2)
        cw, ca = max(O.max_abs(W), 1e-12), max(O.max_abs(X), 1e-12)
        qw, _ = O.quantize(W, cw)
        qa, _ = O.quantize(X, ca)
        qg, sg, stream, ss = O.quantize_gradient(cs, GO, it, stream)
        assert stream == stream_ref and cs.clip == cs_ref.clip
        assert ss["dc"] == stats[3] and ss["eps_norm"] == stats[5]
        assert (O.conv_dgrad(qg, qw, g, sg, O.quant_scale(cw))[1] == ga).all()
        assert (O.conv_wgrad(qg, qa, g, sg, O.quant_scale(ca))[1] == gw).all()
