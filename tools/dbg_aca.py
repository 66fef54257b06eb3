"""Debug: run the GPU ACA hook on the oracle's largest reglog_1k fills."""
import sys, numpy as np, ctypes
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from oracle import ifmm_oracle as O
from conftest import load_golden, golden_kernel
g = load_golden("reglog_1k")
pts = O.baseline_points(1024, 0); T = O.build_tree(pts, 2)
fills = []
orig_h = O._squeeze_hybrid
def sh(st, k, p, q, tol, stats):
    F = st.blk["p2l"].get((k, p, q))
    if F is not None:
        fills.append(F.copy())
    return orig_h(st, k, p, q, tol, stats)
O._squeeze_hybrid = sh
st = O.init_operators(T, golden_kernel(g), 4, 1e-10)
O.factorize(st, order="colour9")
from paper_1407_1572_b200 import _lib as L
for F in sorted(fills, key=lambda F: -F.shape[0])[:6]:
    m, n = F.shape
    Lo, Ro, bad = O.aca_block(F, 1e-10)
    _, probes = O.aca_probe_rows(m)
    kmax = min(m, n)
    left = np.empty((m, kmax), order="F"); right = np.empty((n, kmax), order="F")
    rk = np.zeros(1, np.int32); inc = np.zeros(1, np.int32)
    L.check(L.lib.ifmm_test_aca(L.ptr(np.asfortranarray(F)), m, n, 1e-10, L.ptr(probes.astype(np.int32)), kmax,
                                L.ptr(left), L.ptr(right), L.ptr(rk), L.ptr(inc)))
    k = int(rk[0]); ap = left[:, :k] @ right[:, :k].T
    s = np.linalg.svd(F, compute_uv=False)
    print(F.shape, "oracle rank", Lo.shape[1], "gpu crosses", k, "inc", inc[0], "err", np.linalg.norm(ap - F) / np.linalg.norm(F),
          "svd rank@1e-10", int(np.sum(s / s[0] >= 1e-10)))
