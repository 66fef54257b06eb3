"""Debug: oracle augmentation trace (colour9) -- per fill: kind p q rank +wq -> rq (+wp)."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from oracle import ifmm_oracle as O
from conftest import load_golden, golden_kernel
g = load_golden(sys.argv[1] if len(sys.argv) > 1 else "reglog_1k")
N, depth, p, tol = int(g["N"]), int(g["depth"]), int(g["p"]), float(g["tol"])
pts = O.baseline_points(N, 0); T = O.build_tree(pts, depth)
orig_aug = O._augment
ev = []
def aug(st, k, q, W):
    ev.append((q, W.shape[1], st.U[(k, q)].shape[1] + W.shape[1]))
    return orig_aug(st, k, q, W)
O._augment = aug
oh, on = O._squeeze_hybrid, O._squeeze_near
def sh(st, k, p_, q, tl, stats):
    ev.clear(); r0 = st.r(k, q); oh(st, k, p_, q, tl, stats)
    w = sum(e[1] for e in ev if e[0] == q)
    print(f"augq kind=0 p={p_} q={q} +{w} -> {st.r(k, q)}")
def sn(st, k, p_, q, tl, stats):
    ev.clear(); oh2 = on(st, k, p_, q, tl, stats)
    wq = sum(e[1] for e in ev if e[0] == q); wp = sum(e[1] for e in ev if e[0] == p_)
    print(f"augq kind=1 p={p_} q={q} +{wq} -> {st.r(k, q)} | p +{wp} -> {st.r(k, p_)}")
O._squeeze_hybrid, O._squeeze_near = sh, sn
st = O.init_operators(T, golden_kernel(g), p, tol)
O.factorize(st, order="colour9")
