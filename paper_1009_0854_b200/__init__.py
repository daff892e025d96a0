"""paper_1009_0854_b200 — B200-native MACT colour-transform path (arXiv 1009.0854).

Drop-in for the hot path of the reference package ``mact`` 0.1.0:
``fast`` (MACT transforms), ``exact`` (fp64 ground truth + distances),
``lut`` (3D-LUT interpolators) and ``harness`` (error measurement), all
executed by the hand-written sm_100a kernels of ``libmact_cuda.so``
(``csrc/``, C ABI in ``include/mact_cuda.h``).
"""

from .approximants import (Approximant, Polynomial, Rational, TargetFn, eval_poly, eval_rational,
                           registry_get, registry_keys)
from .errors import MactError, UnknownApproximant

__version__ = "0.1.0"

__all__ = ["Approximant", "Polynomial", "Rational", "TargetFn", "eval_poly", "eval_rational",
           "registry_get", "registry_keys",
           "MactError", "UnknownApproximant", "__version__"]
