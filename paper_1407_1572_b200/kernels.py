"""Kernel registry (mirror of ifmm/kernels.py) with device kernel ids.

A `Kernel` names one of the device-evaluated radial functions; the GPU
assembly evaluates it (csrc/kfun.cuh).  `evaluate` is a host convenience for
users (e.g. building a right-hand side); the factorize/solve path never calls
it.  Arbitrary Python callables cannot run on the device and are rejected by
`init_operators`.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

DEFAULT_A = 0.001

KERNEL_IDS = {
    "log": 0,
    "laplace3d": 1,
    "biharmonic": 2,
    "bessel-y0": 3,
    "inverse-quadric": 4,
    "inverse-multiquadric": 5,
    "helmholtz3d": 6,
    "gaussian": 7,
    "multiquadric": 8,
    "inv_r": 9,
    "log_r": 10,
}
SMOOTH_KERNELS = ("gaussian", "multiquadric")
KERNEL_NAMES = tuple(KERNEL_IDS)


def _branch(r, a, inner, outer):
    r = np.atleast_1d(np.asarray(r, dtype=float))
    out = np.zeros_like(r)
    lo = (r < a) & (r > 0)
    hi = r >= a
    if lo.any():
        out[lo] = inner(r[lo])
    if hi.any():
        out[hi] = outer(r[hi])
    return out


@dataclass(frozen=True)
class Kernel:
    """Radial kernel f(r) (ifmm/kernels.py:26-47).  `scale`/`shift` apply to
    the BASELINE kernels inv_r = scale/r and log_r = scale (ln r + shift)."""

    name: str
    a: float = DEFAULT_A
    scale: float = 1.0
    shift: float = 0.0

    @property
    def kernel_id(self) -> int:
        if self.name not in KERNEL_IDS:
            raise ValueError(f"kernel {self.name!r} has no device implementation")
        return KERNEL_IDS[self.name]

    def func(self, r):
        a, nm = self.a, self.name
        r = np.atleast_1d(np.asarray(r, dtype=float))
        if nm == "inv_r":
            return np.where(r > 0, self.scale / np.where(r > 0, r, 1.0), 0.0)
        if nm == "log_r":
            return np.where(r > 0, self.scale * (np.log(np.where(r > 0, r, 1.0)) + self.shift), 0.0)
        if nm == "log":
            return _branch(r, a, lambda s: s * (np.log(s) - 1) / (a * (np.log(a) - 1)),
                           lambda s: np.log(s) / np.log(a))
        if nm == "laplace3d":
            return _branch(r, a, lambda s: s / a, lambda s: a / s)
        if nm == "biharmonic":
            return _branch(r, a, lambda s: s**3 * (3 * np.log(s) - 1) / (a**3 * (3 * np.log(a) - 1)),
                           lambda s: s**2 * np.log(s) / (a**2 * np.log(a)))
        if nm == "bessel-y0":
            from scipy.special import y0
            return _branch(r, a, lambda s: (1 + y0(a)) / (1 + y0(s)), lambda s: y0(s) / y0(a))
        if nm == "inverse-quadric":
            return _branch(r, a, lambda s: np.arctan(s) / np.arctan(a), lambda s: (1 + a**2) / (1 + s**2))
        if nm == "inverse-multiquadric":
            return _branch(r, a, lambda s: np.arcsinh(s) / np.arcsinh(a),
                           lambda s: np.sqrt((1 + a**2) / (1 + s**2)))
        if nm == "helmholtz3d":
            return _branch(r, a, lambda s: s / a, lambda s: a * np.cos(s) / (s * np.cos(a)))
        if nm == "gaussian":
            return np.exp(-(r**2) / a)
        if nm == "multiquadric":
            return np.sqrt(1 + r**2 / a**2)
        raise ValueError(f"unknown kernel {nm!r}")

    def evaluate(self, r):
        r = np.asarray(r, dtype=float)
        if np.any(r < 0):
            raise ValueError("negative distance")
        out = self.func(r)
        return float(out[0]) if r.ndim == 0 else out

    def __call__(self, r):
        return self.evaluate(r)


def make_kernel(name: str, a: float = DEFAULT_A, scale: float = 1.0, shift: float = 0.0) -> Kernel:
    """ifmm/kernels.py:173-178 (+ inv_r / log_r)."""
    if name not in KERNEL_IDS:
        raise ValueError(f"unknown kernel {name!r}; choose from {KERNEL_NAMES}")
    if a <= 0:
        raise ValueError("regularization radius a must be positive")
    return Kernel(name=name, a=a, scale=scale, shift=shift)


def baseline_kernel(name: str, n: int) -> Kernel:
    """BASELINE.json kernels on [0,1]^2 with diagonal sqrt(N), mapped to the
    reference box (x' = 2x - 1) and divided by sqrt(N): 1/|x-y| -> (2/r')/sqrt(N),
    log|x-y| -> (ln r' - ln 2)/sqrt(N), unit diagonal."""
    s = 1.0 / math.sqrt(n)
    if name in ("inv_r", "1/r"):
        return Kernel("inv_r", scale=2.0 * s)
    if name in ("log_r", "log|x-y|"):
        return Kernel("log_r", scale=s, shift=-math.log(2.0))
    raise ValueError(name)


def kernel_block(kernel: Kernel, targets: np.ndarray, sources: np.ndarray) -> np.ndarray:
    """Host helper (ifmm/kernels.py:189-194): K(|t_i - s_j|)."""
    d = np.atleast_2d(targets)[:, None, :] - np.atleast_2d(sources)[None, :, :]
    return kernel.evaluate(np.sqrt(np.sum(d * d, axis=2)))
