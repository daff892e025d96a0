"""Coefficient registry of the MACT approximants (data only).

The published coefficient sets (approximants.py:168-265 of the reference;
PAPER.md Tables 1-8) parsed from their decimal strings to the nearest double,
plus the frozen [0,1] refits of arctan(sqrt(3) x) that the reference's HSI
pipeline actually evaluates (fast.py:38-43, recomputed by remez_poly at import
time there; frozen here — tests/test_coeffs.py pins them to the reference).

Nothing in this module evaluates a polynomial on the host: ``eval_poly`` /
``eval_rational`` (approximants.py:55-82), the callable ``Polynomial`` /
``Rational`` / ``Approximant`` and ``TargetFn.exact`` (:101-103) run on the
GPU (``mact_poly_eval`` / ``mact_exact_elem`` of libmact_cuda.so), in numpy's
Horner order and rounding, so they are bit-identical to the reference.  The
classes mirror the reference's public names so code that introspects or calls
a MactConfig's approximants keeps working.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass
from typing import Dict, Tuple, Union

import numpy as np

from .errors import DegenerateDenominator, UnknownApproximant

CBRT_KNEE = 0.008856
ATAN_SQRT3_FIT_HI = 254.0 / 256.0


def _is_scalar(x) -> bool:
    from . import _dev

    return not _dev.is_device_tensor(x) and not isinstance(x, np.ndarray) and np.ndim(x) == 0


def _result(out, on_dev: bool, scalar: bool):
    from . import _dev

    r = _dev.to_caller(out, on_dev)
    return float(r) if scalar else r


class TargetFn(enum.Enum):
    """The elementary functions the bundled approximants replace (approximants.py:85-103)."""

    CBRT = "cbrt"
    ATAN_SQRT3 = "atan_sqrt3"
    ASIN_HALF = "asin_half"
    ACOS_HALF = "acos_half"
    ATAN_F = "atan_f"
    ATAN_G = "atan_g"

    def exact(self, x):
        """Reference libm evaluation of the target function (approximants.py:101-115), on the GPU
        (libdevice cbrt / atan / asin / acos: within an ulp or two of numpy's libm)."""
        import torch

        from . import _dev, _lib
        from .exact import _f64_args

        scalar = _is_scalar(x)
        (t,), on_dev = _f64_args(x)
        out = torch.empty(t.shape, dtype=torch.float64, device=t.device)
        _lib.call("mact_exact_elem", _lib.ELEM_TARGET[self.value], t.data_ptr(), None, None,
                  out.data_ptr(), None, None, t.numel(), _dev.stream_ptr())
        return _result(out, on_dev, scalar)


@dataclass(frozen=True)
class Polynomial:
    """a_0 + a_1 x + ... + a_n x^n (ascending coefficients)."""

    coeffs: Tuple[float, ...]

    def __post_init__(self):
        if not self.coeffs:
            raise ValueError("polynomial needs at least one coefficient")
        object.__setattr__(self, "coeffs", tuple(float(c) for c in self.coeffs))

    @property
    def degree(self) -> int:
        return len(self.coeffs) - 1

    def __call__(self, x):
        return eval_poly(self, x)


@dataclass(frozen=True)
class Rational:
    """Ratio of two polynomials (approximants.py:43-52)."""

    numerator: Polynomial
    denominator: Polynomial

    def __call__(self, x):
        return eval_rational(self, x)


def _poly_eval(num: Polynomial, den, x):
    import torch

    from . import _dev, _lib
    from .exact import _f64_args

    for p in (num, den):
        if p is not None and p.degree >= _lib.POLY_MAX:
            raise ValueError(f"polynomial degree {p.degree} exceeds the device limit {_lib.POLY_MAX - 1}")
    scalar = _is_scalar(x)
    (t,), on_dev = _f64_args(x)
    spec = _lib.MactPolySpec()
    spec.num_deg = num.degree
    for i, c in enumerate(num.coeffs):
        spec.num[i] = c
    spec.den_deg = -1 if den is None else den.degree
    if den is not None:
        for i, c in enumerate(den.coeffs):
            spec.den[i] = c
    out = torch.empty(t.shape, dtype=torch.float64, device=t.device)
    flag = torch.zeros(1, dtype=torch.int32, device=t.device)
    _lib.call("mact_poly_eval", spec, t.data_ptr(), out.data_ptr(), t.numel(), flag.data_ptr(),
              _dev.stream_ptr())
    if den is not None and int(flag.item()):
        if scalar:
            raise DegenerateDenominator(f"denominator vanished at x={x!r}")
        raise DegenerateDenominator("denominator vanished inside evaluation batch")
    return _result(out, on_dev, scalar)


def eval_poly(p: Polynomial, x):
    """Evaluate ``p`` at ``x`` (scalar, ndarray or CUDA tensor) in Horner form (approximants.py:55-72),
    on the GPU with numpy's operation order: bit-identical to the reference."""
    return _poly_eval(p, None, x)


def eval_rational(r: Rational, x):
    """Evaluate ``r`` at ``x``; DegenerateDenominator on a vanishing q(x) (approximants.py:75-82)."""
    return _poly_eval(r.numerator, r.denominator, x)


def target_values(target, x):
    """Evaluate a target given either a TargetFn member or a plain callable (approximants.py:118-120)."""
    return target.exact(x) if isinstance(target, TargetFn) else target(x)


@dataclass(frozen=True)
class Approximant:
    form: Union[Polynomial, Rational]
    interval: Tuple[float, float]
    eps_max: float
    target_fn: TargetFn

    def __post_init__(self):
        lo, hi = self.interval
        if not lo < hi:
            raise ValueError(f"interval must satisfy lo < hi, got {self.interval}")

    def __call__(self, x):
        return self.form(x)

    def measured_max_error(self, num_points: int = 100_000) -> float:
        """Max |approx - exact| over a dense uniform grid of the fit interval (approximants.py:144-149)."""
        import torch

        lo, hi = self.interval
        grid = torch.from_numpy(np.linspace(lo, hi, num_points)).cuda()
        diff = self.form(grid) - torch.as_tensor(target_values(self.target_fn, grid), device=grid.device)
        return float(diff.abs().max())


# (target, degrees) -> (eps_max, coefficient strings...)  — one table, every set.
_P = TargetFn
_TABLE: Dict[Tuple[TargetFn, Tuple[int, ...]], tuple] = {
    (_P.CBRT, (2,)): ("1.271154e-01", ("1.268979e-01", "2.393873", "-1.647669")),
    (_P.CBRT, (3,)): ("9.787829e-02", ("9.787826e-02", "4.057495", "-7.388864", "4.331370")),
    (_P.CBRT, (4,)): ("8.111150e-02", ("8.111133e-02", "5.926004", "-2.017165e+01",
                                       "2.833070e+01", "-1.324728e+01")),
    (_P.CBRT, (5,)): ("7.002956e-02", ("7.002910e-02", "7.961214", "-4.329352e+01",
                                       "1.063182e+02", "-1.135685e+02", "4.358268e+01")),
    (_P.CBRT, (2, 2)): ("2.060996e-03", ("6.309655e-03", "5.785782e-01", "1.591005"),
                        ("4.482646e-02", "1.175862", "9.596879e-01")),
    (_P.CBRT, (2, 3)): ("7.210231e-04", ("2.500705e-03", "3.447113e-01", "1.942708"),
                        ("1.978701e-02", "8.542797e-01", "1.664540", "-2.503267e-01")),
    (_P.CBRT, (3, 2)): ("5.931593e-04", ("1.776519e-03", "2.632323e-01", "1.751297", "3.836709e-01"),
                        ("1.432256e-02", "6.779998e-01", "1.706260")),
    (_P.CBRT, (2, 4)): ("3.107735e-04", ("1.317899e-03", "2.390113e-01", "2.099395"),
                        ("1.124254e-02", "6.726679e-01", "2.184656", "-7.511150e-01",
                         "2.229717e-01")),
    (_P.CBRT, (3, 3)): ("1.858694e-04", ("4.370889e-04", "9.526952e-02", "1.252009", "1.302733"),
                        ("3.912364e-03", "2.954084e-01", "1.717143", "6.343408e-01")),
    (_P.CBRT, (4, 2)): ("2.334688e-04", ("7.589302e-04", "1.519784e-01", "1.663584", "8.368075e-01",
                                         "-1.657269e-01"),
                        ("6.644723e-03", "4.506424e-01", "2.030622")),
    (_P.CBRT, (3, 4)): ("8.539863e-05", ("1.683667e-04", "4.667675e-02", "9.106812e-01", "1.810577"),
                        ("1.610864e-03", "1.617974e-01", "1.494070", "1.218468", "-1.079451e-01")),
    (_P.CBRT, (4, 3)): ("8.052920e-05", ("1.349673e-04", "3.832079e-02", "7.870174e-01", "1.799062",
                                         "2.071170e-01"),
                        ("1.299250e-03", "1.345420e-01", "1.330358", "1.365369")),
    (_P.CBRT, (4, 4)): ("3.856930e-05", ("3.927283e-05", "1.392318e-02", "4.114739e-01", "1.734853",
                                         "8.679223e-01"),
                        ("4.022100e-04", "5.414536e-02", "8.221526e-01", "1.800167", "3.513617e-01")),
    # degree-2 a_2 sign restored as in the reference registry (approximants.py:215-220)
    (_P.ATAN_SQRT3, (2,)): ("6.907910e-03", ("5.959793e-03", "1.782975", "-7.497879e-01")),
    (_P.ATAN_SQRT3, (3,)): ("3.654156e-03", ("-3.654076e-03", "1.884080", "-9.805583e-01",
                                             "1.430580e-01")),
    (_P.ATAN_SQRT3, (4,)): ("1.286371e-03", ("-1.286369e-03", "1.796716", "-4.958969e-01",
                                             "-6.927404e-01", "4.421541e-01")),
    (_P.ATAN_SQRT3, (5,)): ("1.801311e-04", ("-1.801283e-04", "1.739333", "-2.039848e-02",
                                             "-2.065512", "2.052837", "-6.591729e-01")),
    (_P.ASIN_HALF, (4,)): ("2.097814e-05", ("2.097797e-05", "1.412840", "1.429881e-02",
                                            "6.704361e-02", "6.909677e-02")),
    (_P.ASIN_HALF, (5,)): ("2.370540e-06", ("-2.370048e-06", "1.414434", "-3.300037e-03",
                                            "1.354670e-01", "-3.994259e-02", "6.099502e-02")),
    (_P.ACOS_HALF, (4,)): ("1.048949e-05", ("1.570786", "-9.990285e-01", "-1.429899e-02",
                                            "-9.481335e-02", "-1.381942e-01")),
    (_P.ACOS_HALF, (5,)): ("1.186403e-06", ("1.570798", "-1.000156", "3.299810e-03",
                                            "-1.915780e-01", "7.988231e-02", "-1.725177e-01")),
    (_P.ATAN_F, (4,)): ("1.036515e-04", ("-1.036508e-04", "1.003740", "-1.773538e-02",
                                         "-3.390563e-01", "1.386796e-01")),
    (_P.ATAN_F, (5,)): ("2.073939e-05", ("2.073866e-05", "9.982666e-01", "2.352573e-02",
                                         "-4.506862e-01", "2.635050e-01", "-4.920822e-02")),
    (_P.ATAN_G, (4,)): ("1.051643e-04", ("1.570917", "-1.004004", "1.885694e-02",
                                         "3.373159e-01", "-1.377930e-01")),
    (_P.ATAN_G, (5,)): ("2.012104e-05", ("1.570769", "-9.981253e-01", "-2.440212e-02",
                                         "4.528921e-01", "-2.659181e-01", "5.016228e-02")),
}

_INTERVAL = {
    _P.ATAN_SQRT3: (0.0, ATAN_SQRT3_FIT_HI),
    _P.ASIN_HALF: (0.0, 1.0 / math.sqrt(2.0)),
    _P.ACOS_HALF: (0.0, 0.5),
    _P.ATAN_F: (0.0, 254.0 / 255.0),
    _P.ATAN_G: (1.0 / 255.0, 1.0),
}

# [0,1] refit of arctan(sqrt(3) x) = what the reference HSI pipeline evaluates
# (fast.py:38-43, remez_poly(ATAN_SQRT3, (0, 1), n)).  Exact float64 values.
HSI_REFIT: Dict[int, Tuple[Tuple[float, ...], float]] = {
    2: ((0.006284947651693185, 1.780260485842989, -0.7464821732923941), 0.0071342909943101634),
    3: ((-0.003692653108724686, 1.8851978201283177, -0.984841853121039, 0.14684158418931897),
        0.003692653108724797),
    4: ((-0.0013203887844437379, 1.7981353035694578, -0.5047931910004136, -0.6755157658048955,
         0.43201198200133645), 0.001320388784807336),
    5: ((-0.00018962050654047768, 1.7398783026013234, -0.02536381417376224, -2.0498061861186665,
         2.032735308062768, -0.6502460591750653), 0.0001896205065405887),
}


def _make(fn: TargetFn, deg: Tuple[int, ...], entry) -> Approximant:
    eps = float(entry[0])
    if len(deg) == 2:
        form = Rational(Polynomial(tuple(map(float, entry[1]))), Polynomial(tuple(map(float, entry[2]))))
        return Approximant(form, (CBRT_KNEE, 1.0), eps, fn)
    interval = (0.0, 1.0) if fn is TargetFn.CBRT else _INTERVAL[fn]
    return Approximant(Polynomial(tuple(map(float, entry[1]))), interval, eps, fn)


_REGISTRY = {key: _make(key[0], key[1], val) for key, val in _TABLE.items()}


def registry_get(fn: TargetFn, degree_spec: Tuple[int, ...]) -> Approximant:
    """Bundled approximant by target and degrees; UnknownApproximant otherwise
    (reference approximants.py:300-311)."""
    key = (fn, tuple(int(d) for d in degree_spec))
    if key not in _REGISTRY:
        raise UnknownApproximant(f"no bundled coefficients for {fn.value} with degrees {degree_spec}")
    return _REGISTRY[key]


def registry_keys():
    return sorted(_REGISTRY, key=lambda k: (k[0].value, k[1]))


def hsi_refit(degree: int) -> Approximant:
    """The [0,1] arctan(sqrt(3) x) refit used by the HSI pipeline."""
    if degree not in HSI_REFIT:
        raise UnknownApproximant(f"no atan_sqrt3 refit of degree {degree}")
    coeffs, eps = HSI_REFIT[degree]
    return Approximant(Polynomial(coeffs), (0.0, 1.0), eps, TargetFn.ATAN_SQRT3)
