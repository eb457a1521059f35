"""Diagnostic only (not part of the product): the achievable dense INT8
tcgen05 GEMM rate on this B200, measured with CUTLASS's own CuTe-DSL
persistent GEMM example (library code shipped in the image), so the conv
kernels' roofline fraction can be read against what a tuned library GEMM
reaches.  Prints TOPS per tile configuration."""
import importlib.util
import sys

import cutlass

PATH = ("/opt/prime-rl/.venv/lib/python3.12/site-packages/flashinfer/data/cutlass/examples/python/CuTeDSL/"
        "blackwell/dense_gemm_persistent.py")
spec = importlib.util.spec_from_file_location("dgp", PATH)
dgp = importlib.util.module_from_spec(spec)
spec.loader.exec_module(dgp)

M = N = K = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
for tile, cluster, two in [((128, 256), (1, 1), False), ((256, 256), (2, 1), True), ((128, 128), (1, 1), False),
                           ((256, 128), (2, 1), True), ((256, 256), (2, 2), True)]:
    t_us = dgp.run((M, N, K, 1), cutlass.Int8, cutlass.Int32, cutlass.Int32, "k", "k", "n", tile, cluster, two, True,
                   1e-1, 3, 20, True, False, True)
    print(f"tile {tile} cluster {cluster} 2cta {two}: {t_us:.1f} us  {2 * M * N * K / t_us / 1e6:.0f} TOPS",
          flush=True)
