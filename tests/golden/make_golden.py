"""Dump golden vectors from the UNMODIFIED reference (oracle/_ref/libi8t_ref.so,
compiled from /root/reference by oracle/Makefile) into tests/golden/golden.npz.

Run here (the dev container, where /root/reference exists):
    make -C oracle ref && python tests/golden/make_golden.py
The fixtures are committed; tests/test_oracle_golden.py checks the C
restatement (oracle/oracle.c) against them anywhere, and the GPU tests check
the CUDA path against the restatement.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import lib as O  # noqa: E402  (input generators only)
from oracle import ref as R  # noqa: E402


def main():
    assert R.build(), "reference not buildable here"
    out = {}
    rng = np.random.default_rng(2024)

    # ---- LCG: first 8 states of a few seeds (quantize.hpp:32-50)
    for seed in (0, 12345, 99, 0xFFFFFFFF):
        import ctypes as C
        s = C.c_uint32(seed)
        out[f"lcg_{seed}"] = np.array([R.lib().ref_lcg_next(C.byref(s)) for _ in range(8)], np.uint32)

    # ---- quantize nearest / stochastic (quantize.cpp:16-43)
    for i in range(6):
        n = int(rng.integers(100, 3000))
        x = (rng.standard_normal(n) * rng.uniform(1e-5, 5)).astype(np.float32)
        x[rng.random(n) < 0.2] = 0.0
        clip = np.float32(np.abs(x).max() * rng.uniform(0.1, 1.2))
        qn, _ = R.quantize(x, float(clip))
        seed = int(rng.integers(0, 2**32))
        qs, st = R.quantize(x, float(clip), True, seed)
        out[f"q{i}_x"] = x
        out[f"q{i}_meta"] = np.array([clip], np.float32)
        out[f"q{i}_seed"] = np.array([seed, st], np.uint32)
        out[f"q{i}_nearest"] = qn
        out[f"q{i}_stoch"] = qs
    # exact ties
    clip = np.float32(1.27)
    s = np.float32(clip / np.float32(127))
    x = ((np.arange(-130, 131) + 0.5) * np.float64(s)).astype(np.float32)
    out["qties_x"] = x
    out["qties_nearest"] = R.quantize(x, float(clip))[0]
    # partitioned
    x = rng.standard_normal(1000).astype(np.float32)
    out["qpart_x"] = x
    out["qpart_q"] = R.quantize_partitioned(x, float(np.abs(x).max()), 900, 8, 4)

    # ---- conv (conv.cpp:108-205), reference geometry rule (exact division)
    gi = 0
    while gi < 16:
        n = int(rng.integers(1, 3)); c = int(rng.integers(1, 5)); kh = int(rng.integers(1, 4))
        s_ = int(rng.integers(1, 3)); p = int(rng.integers(0, 2)); dw = gi % 4 == 3
        k = c if dw else int(rng.integers(1, 5))
        oh = int(rng.integers(1, 5)); h = (oh - 1) * s_ + kh - 2 * p
        ow = int(rng.integers(1, 5)); w = (ow - 1) * s_ + kh - 2 * p
        if h < 1 or w < 1:
            continue
        gv = R.gvec(n, c, h, w, k, kh, kh, s_, p, dw)
        qa = rng.integers(-127, 128, (n, c, h, w)).astype(np.int8)
        qw = rng.integers(-127, 128, R.w_shape(gv)).astype(np.int8)
        qg = rng.integers(-127, 128, R.out_shape(gv)).astype(np.int8)
        z = R.conv2d_q(qa, 1.27, qw, 12.7, gv)
        gw, ga = R.conv2d_backward_q(qg, 0.5, qa, 1.27, qw, 12.7, gv)
        for nm, v in (("g", gv), ("qa", qa), ("qw", qw), ("qg", qg), ("z", z), ("gw", gw), ("ga", ga)):
            out[f"conv{gi}_{nm}"] = v
        gi += 1

    # ---- DSGC (clip.cpp:8-93)
    for i, (seed, grid, rounds) in enumerate([(2, 64, 0), (3, 32, 2), (4, 32, 2), (21, 32, 2), (40, 8, 5)]):
        g = O.gradient_like((2048,), seed, 0.01, 0.01)
        c, d = R.search_clip(g, grid, rounds)
        out[f"search{i}_g"] = g
        out[f"search{i}_cfg"] = np.array([grid, rounds], np.int32)
        out[f"search{i}_res"] = np.array([c, d], np.float64)
        out[f"search{i}_dcs"] = np.array([R.measure_dc(g, float(cc)) for cc in (1e-3, 5e-3, 2e-2)], np.float64)
    g1, g2 = O.gradient_like((512,), 30, 0.01, 0.01), O.gradient_like((512,), 31, 0.01, 0.01)
    st = O.ClipState(0.0, 0.0, -1, 3)
    seq = []
    for it, g in enumerate([g1, g2, g2, g1, np.zeros(512, np.float32), g2, g1]):
        R.maybe_update(st, g, it)
        seq.append([st.clip, st.last_dc, st.iter_of_last_update])
    out["maybe_g1"], out["maybe_g2"] = g1, g2
    out["maybe_seq"] = np.array(seq, np.float64)

    # ---- DCLR (lr_scale.cpp:8-20)
    dcs = np.linspace(0.0, 2.0, 41)
    out["phi"] = np.array([[R.scale_factor(d, 20.0, 0.1, f) for f in (0, 1, 2)] for d in dcs], np.float64)

    # ---- one INT8 Conv2d layer step through the reference layer API (layers.cpp:19-59, 98-126)
    for li, (n, c, h, k, kh, s_, p) in enumerate([(2, 8, 10, 16, 3, 1, 1), (1, 16, 9, 8, 3, 2, 1)]):
        gv = R.gvec(n, c, h, h, k, kh, kh, s_, p)
        W = O.gaussian((k, c, kh, kh), 3 + li, 0.2)
        X = O.gaussian((n, c, h, h), 4 + li, 1.0, True)
        GO = O.gradient_like(R.out_shape(gv), 5 + li, 1e-4, 0.01)
        cs = O.ClipState(0.0, 0.0, -1, 100)
        z, gw, ga, st2, stats = R.conv_layer_step(gv, W, X, GO, 0, 77, cs)
        for nm, v in (("g", gv), ("W", W), ("X", X), ("GO", GO), ("z", z), ("gw", gw), ("ga", ga),
                      ("stats", stats), ("stream", np.array([77, st2], np.uint32))):
            out[f"layer{li}_{nm}"] = v

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
