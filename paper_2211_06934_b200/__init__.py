"""B200-native fused differentiable optimizer step (arXiv 2211.06934, TorchOpt
§2.3 "CPU/GPU-accelerated optimizers").

The product is libdiffopt.so (C ABI, include/diffopt.h): hand-written sm_100a
kernels for the Adam / RMSProp / SGD-momentum update and its VJP. This package
is its Python binding (``_lib``: same names as the C entry points), the
autograd wiring and Listing-1 functional API (``functional``), and the two
drivers of SURVEY §8(a): the K-step unrolled sweep (``unroll``) and the
task-sharded MAML meta-batch (``maml``). Importing it without the built
library raises; there is no CPU fallback.
"""
from . import _lib
from ._lib import Tree, DiffoptError, OPT_F32, OPT_BF16, OPT_COMPUTE_DEFAULT, OPT_COMPUTE_F32, \
    OPT_COMPUTE_F64
from .functional import (AdamStep, RmsPropStep, RmsCmStep, SgdStep, ApplyUpdates, FlatTree,
                         adam, rmsprop, sgd, apply_updates)

__all__ = ["Tree", "DiffoptError", "AdamStep", "RmsPropStep", "RmsCmStep", "SgdStep", "ApplyUpdates",
           "FlatTree", "adam", "rmsprop", "sgd", "apply_updates", "OPT_F32", "OPT_BF16",
           "OPT_COMPUTE_DEFAULT", "OPT_COMPUTE_F32", "OPT_COMPUTE_F64"]
from . import implicit, offload, unroll  # noqa: E402  (drivers above the C ABI)
