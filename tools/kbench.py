"""Kernel microbenchmarks on the B200: conv fwd/dgrad/wgrad TOPS on config-1 and
ResNet-50 layer shapes, quantiser GB/s.  CUDA events on the launching stream,
warm-up, inputs larger than L2 or an L2 flush between reps.

    python tools/kbench.py [--batch 256] [--reps 10] [--json out.json]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_12607_b200 import ops  # noqa: E402

L2_FLUSH = None


def flush():
    global L2_FLUSH
    if L2_FLUSH is None:
        L2_FLUSH = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    L2_FLUSH.zero_()


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda._sleep(5_000_000)  # the GPU idles while the host queues flush + launch: no host gap inside s..e
        flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def conv_case(name, n, c, h, k, kh, stride, pad, reps):
    g = ops.geom(n, c, h, h, k, kh, kh, stride, pad)
    p, q = g.out_hw()
    cp, kp = ops.pad4(c), ops.pad4(k)
    qa = torch.randint(-127, 128, (n, h, h, cp), dtype=torch.int8, device="cuda")
    qgz = torch.randint(-127, 128, (n, p, q, kp), dtype=torch.int8, device="cuda")
    w = torch.randn(k, c, kh, kh, device="cuda")
    qw, qwt = ops.quantize_weight(w, float(w.abs().max()), c_pad=cp, k_pad=kp)
    ld_w, ld_wt = qw.shape[1], qwt.shape[1]
    z = torch.empty((n * p * q, k), device="cuda")
    ga = torch.empty((n * h * h, c), device="cuda")
    acc = torch.empty((kh * kh * cp, k), dtype=torch.int64, device="cuda")
    gw = torch.empty((k, c, kh, kh), device="cuda")
    one = torch.ones(1, device="cuda")
    macs = n * p * q * k * c * kh * kh
    res = {"name": name, "shape": [n, c, h, k, kh, stride, pad]}
    res["fwd_ms"] = timeit(lambda: ops.conv_fwd_nhwc(g, qa, cp, qw, ld_w, one, one, z_out=z), reps)
    res["dgrad_ms"] = timeit(lambda: ops.conv_dgrad_nhwc(g, qgz, kp, qwt, ld_wt, one, one, out=ga), reps)
    res["wgrad_ms"] = timeit(lambda: ops.conv_wgrad_nhwc(g, qgz, kp, qa, cp, one, one, acc=acc, gw=gw), reps)
    for kk in ("fwd", "dgrad", "wgrad"):
        res[kk + "_tops"] = 2 * macs / (res[kk + "_ms"] * 1e-3) / 1e12
    res["gop_per_pass"] = 2 * macs / 1e9
    return res


def quant_case(n_elems, reps):
    x = torch.randn(n_elems, device="cuda") * 1e-3
    q = torch.empty(n_elems, dtype=torch.int8, device="cuda")
    clip = torch.tensor([3e-3], device="cuda")
    amax = torch.zeros(1, device="cuda")
    res = {"n": n_elems}
    ms = timeit(lambda: ops.call("i8t_quantize_nearest", ops.ctx(), ops._p(x), n_elems, ops._p(clip), ops._p(q),
                                 ops._p(amax), 1), reps)
    res["nearest_ms"], res["nearest_gbs"] = ms, 5 * n_elems / (ms * 1e-3) / 1e9
    st = ops.DsgcState(period=100)
    lcg = ops.new_lcg_state(1)
    g4 = x.view(-1, 64)  # as NHWC [P, 64]
    ops.quantize_gradient(st, g4.view(1, -1, 1, 64), 0, lcg, nhwc=True)  # search once
    st.sync()
    ms = timeit(lambda: ops.quantize_gradient(st, g4.view(1, -1, 1, 64), 1, lcg, nhwc=True), reps)
    res["grad_fused_ms"], res["grad_fused_gbs"] = ms, 5 * n_elems / (ms * 1e-3) / 1e9
    st2 = ops.DsgcState(period=1)
    ms = timeit(lambda: ops.quantize_gradient(st2, g4.view(1, -1, 1, 64), 0, lcg, nhwc=True), reps)
    res["grad_search_ms"] = ms
    return res


def r50_table(reps):
    """Every distinct ResNet-50 conv shape (batch 256) x multiplicity: measured
    time per direction vs the attainable max(ops/peak, bytes/HBM) time."""
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from r50_roofline import layer_cost, r50_convs
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    peak_ops, peak_bw = 2.0 * peaks["bf16_tflops_sustained"] * 1e12, peaks["hbm_gbs"] * 1e9
    shapes = {}
    for name, n, c, h, k, r, s, p in r50_convs():
        key = (n, c, h, k, r, s, p, name == "stem")
        shapes[key] = shapes.get(key, 0) + 1
    rows, tot_meas, tot_att = [], 0.0, 0.0
    for (n, c, h, k, r, s, p, stem), mult in shapes.items():
        res = conv_case(f"{c}-{k}@{h} {r}x{r}/s{s}", n, c, h, k, r, s, p, reps)
        cost = layer_cost(n, c, h, k, r, s, p, peak_ops, peak_bw, skip_dgrad=stem)
        for d, (o, b, t_att) in cost.items():
            t = res[d + "_ms"] * 1e-3
            tot_meas += mult * t
            tot_att += mult * t_att
            rows.append({"shape": res["name"], "dir": d, "mult": mult, "ms": t * 1e3, "att_ms": t_att * 1e3,
                         "frac_att": t_att / t, "tops": o / t / 1e12,
                         "bound": "tensor" if o / peak_ops >= b / peak_bw else "hbm"})
            print(f"{res['name']:22s} {d:5s} x{mult} {t * 1e3:8.4f} ms  att {t_att * 1e3:8.4f} ms  "
                  f"{100 * t_att / t:5.1f}%  {o / t / 1e12:7.1f} TOPS  {rows[-1]['bound']}", flush=True)
    print(f"TOTAL conv per step: measured {tot_meas * 1e3:.2f} ms, attainable {tot_att * 1e3:.2f} ms "
          f"({100 * tot_att / tot_meas:.1f}%)", flush=True)
    return {"rows": rows, "measured_ms": tot_meas * 1e3, "attainable_ms": tot_att * 1e3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--json", default=None)
    ap.add_argument("--r50", action="store_true", help="per-layer table of all ResNet-50 conv shapes")
    a = ap.parse_args()
    if a.r50:
        out = r50_table(a.reps)
        if a.json:
            with open(a.json, "w") as f:
                json.dump(out, f, indent=1)
        return
    B = a.batch
    cases = [
        ("config1_3x3_64", 32, 64, 56, 64, 3, 1, 1),
        ("r50_l1_1x1_64_256", B, 64, 56, 256, 1, 1, 0),
        ("r50_l1_3x3_64", B, 64, 56, 64, 3, 1, 1),
        ("r50_l1_1x1_256_64", B, 256, 56, 64, 1, 1, 0),
        ("r50_l2_3x3_128", B, 128, 28, 128, 3, 1, 1),
        ("r50_l3_3x3_256", B, 256, 14, 256, 3, 1, 1),
        ("r50_l3_1x1_1024_256", B, 1024, 14, 256, 1, 1, 0),
        ("r50_l4_3x3_512", B, 512, 7, 512, 3, 1, 1),
        ("r50_l4_1x1_512_2048", B, 512, 7, 2048, 1, 1, 0),
    ]
    out = {"convs": [], "quant": None}
    for cs in cases:
        r = conv_case(*cs, a.reps)
        out["convs"].append(r)
        print(json.dumps(r), flush=True)
    out["quant"] = quant_case(32 * 64 * 56 * 56, a.reps)
    print(json.dumps(out["quant"]), flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
