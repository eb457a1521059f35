"""paper_1912_12607_b200 -- B200-native (sm_100a) INT8 training hot path of
arXiv 1912.12607 ("Towards Unified INT8 Training for CNNs").

Layers:
  include/i8t_cuda.h        C-ABI (the drop-in boundary; reference i8t API)
  csrc/*.cu                 hand-written sm_100a kernels -> libi8t_cuda.so
  _lib.py                   ctypes binding generated from the header
  ops.py                    torch-facing mirror of the reference operator API
  layers.py / trainer.py    INT8 Conv2d/Dense + the per-step trainer loop
"""
from . import ops  # noqa: F401
from ._lib import ConvGeom, DsgcView  # noqa: F401

__all__ = ["ops", "ConvGeom", "DsgcView"]
