"""paper_2208_02025_b200 -- B200-native runtime of the programs Ollie (arXiv 2208.02025)
derives for Conv2d / ConvTranspose2d: merged tcgen05 GEMM + OffsetAdd / selective-add
eOperators (standalone or fused into the GEMM epilogue) + a generic scoped eOperator
evaluator, behind the C ABI of include/ollie.h (libollie.so, built in-tree by build.py).

Importing the package loads libollie.so and fails loudly if it is missing: there is no
CPU fallback and the oracle (../oracle) is never imported from here.
"""
from . import ollie  # noqa: F401  (loads libollie.so)
from .layers import DerivedConv  # noqa: F401
from .dilated import DilatedAsDense  # noqa: F401

__all__ = ["ollie", "DerivedConv", "DilatedAsDense"]
