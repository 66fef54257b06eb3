"""Debug: oracle fill sequence (colour9) for a golden case: kind p q rows cols aca_crosses rank."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from oracle import ifmm_oracle as O
from conftest import load_golden, golden_kernel
g = load_golden(sys.argv[1] if len(sys.argv) > 1 else "reglog_1k")
N, depth, p, tol = int(g["N"]), int(g["depth"]), int(g["p"]), float(g["tol"])
pts = O.baseline_points(N, 0); T = O.build_tree(pts, depth)
orig_aca = O.aca_block
cur = {}
def aca(F, t):
    L, R, bad = orig_aca(F, t)
    cur["r"] = (F.shape, L.shape[1], bad)
    return L, R, bad
O.aca_block = aca
oh, on = O._squeeze_hybrid, O._squeeze_near
def sh(st, k, p_, q, tl, stats):
    cur.clear(); oh(st, k, p_, q, tl, stats)
    if cur: print(f"fill k={k} kind=0 p={p_} q={q} shape={cur['r'][0]} rank={cur['r'][1]}")
def sn(st, k, p_, q, tl, stats):
    cur.clear(); on(st, k, p_, q, tl, stats)
    if cur: print(f"fill k={k} kind=1 p={p_} q={q} shape={cur['r'][0]} rank={cur['r'][1]}")
O._squeeze_hybrid, O._squeeze_near = sh, sn
st = O.init_operators(T, golden_kernel(g), p, tol)
O.factorize(st, order="colour9")
