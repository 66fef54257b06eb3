"""Debug: GPU Gauss-Jordan inverse accuracy on a dumped pivot vs an 80-bit reference."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1407_1572_b200 import _lib as L
raw = open(sys.argv[1], 'rb').read()
n, r = np.frombuffer(raw[:8], dtype=np.int32); m = int(n + r)
S = np.frombuffer(raw[8:], dtype=np.float64).reshape((m, m), order='F').copy()
def gj_inv(A):
    A = A.copy(); k = A.shape[0]; Ainv = np.eye(k, dtype=A.dtype)
    for c in range(k):
        p = c + np.argmax(np.abs(A[c:, c]))
        if p != c:
            A[[c, p]] = A[[p, c]]; Ainv[[c, p]] = Ainv[[p, c]]
        piv = A[c, c]; A[c] /= piv; Ainv[c] /= piv
        f = A[:, c].copy(); f[c] = 0
        A -= np.outer(f, A[c]); Ainv -= np.outer(f, Ainv[c])
    return Ainv
ref = gj_inv(S.astype(np.longdouble)).astype(np.float64)
a = S.ravel(order='F').copy(); info = np.zeros(1, np.int32)
L.check(L.lib.ifmm_test_gj_inverse(L.ptr(a), L.ptr(np.array([m], np.int32)), 1, L.ptr(info)))
g = a.reshape((m, m), order='F')
lu = np.linalg.inv(S)
for name, X in [("gpu GJ", g), ("LAPACK", lu)]:
    e = lambda sl: np.linalg.norm((X - ref)[sl], 1) / np.linalg.norm(ref[sl], 1)
    print(f"{name}: rel err {np.linalg.norm(X-ref,1)/np.linalg.norm(ref,1):.3e}  G {e(np.s_[:n,:n]):.2e} S12 {e(np.s_[:n,n:]):.2e} S22 {e(np.s_[n:,n:]):.2e}")
