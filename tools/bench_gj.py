"""Microbenchmark: batched Gauss-Jordan inverse (device time) for IFMM-like pivot shapes."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1407_1572_b200 import _lib as L  # noqa: E402


def saddle(rng, n, r):
    P = rng.standard_normal((n, n))
    P = P + P.T + 0.2 * n * np.eye(n)
    U, _ = np.linalg.qr(rng.standard_normal((n, r)))
    S = np.zeros((n + r, n + r))
    S[:n, :n] = P
    S[:n, n:] = U
    S[n:, :n] = U.T
    return S


rng = np.random.default_rng(0)
cases = [(1820, 64, 48), (455, 240, 80), (114, 330, 150), (28, 450, 300), (4, 500, 250), (1, 800, 0), (1, 1200, 0)]
for count, n, r in cases:
    mats = [saddle(rng, n, r) for _ in range(min(count, 64))]
    mats = (mats * ((count + len(mats) - 1) // len(mats)))[:count]
    sizes = np.array([x.shape[0] for x in mats], dtype=np.int32)
    packed = np.concatenate([x.ravel(order="F") for x in mats])
    ms = ctypes.c_double()
    L.check(L.lib.ifmm_bench_gj_inverse(L.ptr(packed), L.ptr(sizes), count, 3, ctypes.byref(ms)))
    m = n + r
    fl = count * 2.0 * m ** 3
    print(f"count={count:5d} m={m:5d}: {ms.value:8.3f} ms  {fl / ms.value / 1e9:7.2f} TFLOP/s")
