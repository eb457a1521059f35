"""bench.py's JSON contract on a small workload (ResNet-20, batch 128): every
key the driver reads is present, the numbers are positive and consistent, and
the timed region launched our kernels."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_line_contract():
    out = subprocess.run([sys.executable, "bench.py", "--model", "resnet20", "--batch", "128", "--steps", "3",
                          "--warmup", "3", "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["value"] == pytest.approx(128 / (line["ms_per_step"] / 1e3), rel=1e-9)
    assert line["e2e"]["h2d_bytes_per_step"] == 128 * 3 * 32 * 32 * 4 + 128 * 8
    assert line["gpu_launches"] > 3 * 20
    r = line["roofline"]
    assert r["bound"] == "tensor" and 0 < r["frac"] < 1 and r["conv_ms_per_step"] < line["ms_per_step"]
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert line["config"]["workload"] == "resnet20_int8_train_step"
