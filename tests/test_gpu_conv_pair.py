"""GPU: the CTA-pair conv path (I8T_CONV_PAIR=1: tcgen05.mma.cta_group::2 on
256-row tiles, TMA operands, 1x1 stride-1 fwd / dgrad with >= 129 output
channels) against the oracle.  The switch is read once per process, so the
ResNet-50 layer-shape tests run in a child process with it set."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_conv_pair_path_matches_oracle():
    env = dict(os.environ, I8T_CONV_PAIR="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_conv.py"), "-k", "resnet50_layer_shapes or fwd_dgrad_wgrad"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " passed" in r.stdout
