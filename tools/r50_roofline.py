"""Per-layer roofline of the ResNet-50 INT8 convolutions (batch 256): for each
conv and direction, t_tensor = ops / INT8 peak and t_hbm = compulsory bytes /
HBM peak (int8 operands read once, fp32 output written once, int32 wgrad
partials ignored).  Prints the attainable time per step next to the pure
tensor-bound time."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def r50_convs(n=256):
    out = [("stem", n, 3, 224, 64, 7, 2, 3)]
    h, cin = 56, 64
    for width, blocks, stride in [(64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)]:
        for b in range(blocks):
            s = stride if b == 0 else 1
            out.append(("c1", n, cin, h, width, 1, 1, 0))
            out.append(("c2", n, width, h, width, 3, s, 1))
            ho = (h + 2 - 3) // s + 1
            out.append(("c3", n, width, ho, width * 4, 1, 1, 0))
            if b == 0:
                out.append(("ds", n, cin, h, width * 4, 1, s, 0))
            h, cin = ho, width * 4
    return out


def layer_cost(n, c, h, k, r, s, p, peak_ops, peak_bw, skip_dgrad=False):
    P = (h + 2 * p - r) // s + 1
    ops = 2.0 * n * P * P * k * c * r * r
    a8 = n * h * h * max(c, 4)
    g8 = n * P * P * k
    w8 = k * c * r * r
    res = {}
    res["fwd"] = (ops, a8 + w8 + 4.0 * n * P * P * k)
    if not skip_dgrad:
        res["dgrad"] = (ops, g8 + w8 + 4.0 * n * h * h * c)
    res["wgrad"] = (ops, a8 + g8 + 4.0 * w8)
    return {d: (o, b, max(o / peak_ops, b / peak_bw)) for d, (o, b) in res.items()}


def main():
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    peak_ops = 2.0 * peaks["bf16_tflops_sustained"] * 1e12
    peak_bw = peaks["hbm_gbs"] * 1e9
    tot_ops = t_tensor = t_att = 0.0
    for name, n, c, h, k, r, s, p in r50_convs():
        for d, (o, b, t) in layer_cost(n, c, h, k, r, s, p, peak_ops, peak_bw, skip_dgrad=(name == "stem")).items():
            tot_ops += o
            t_tensor += o / peak_ops
            t_att += t
    print(f"ops/step {tot_ops / 1e12:.3f} TOP; tensor-bound {t_tensor * 1e3:.2f} ms; attainable {t_att * 1e3:.2f} ms")


if __name__ == "__main__":
    main()
