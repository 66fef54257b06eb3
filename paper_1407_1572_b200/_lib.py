"""ctypes binding of libifmm_b200.so (include/ifmm_b200.h).

There is no fallback: if the shared library is missing this module raises at
import, and compute entry points raise RuntimeError when no CUDA device is
present.  Status codes map onto the reference's exception types
(ValueError, SingularPivotError, RuntimeError, MemoryError).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libifmm_b200.so")

OK, INVALID, SINGULAR, CUDA, OOM, NO_DEVICE = range(6)
PTR_HOST, PTR_DEVICE = 0, 1

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: build the CUDA library first "
        "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_1407_1572_b200)")

lib = ctypes.CDLL(LIB_PATH)

_c = ctypes
_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_d = ctypes.c_double
_pi32 = ctypes.POINTER(ctypes.c_int32)
_pi64 = ctypes.POINTER(ctypes.c_int64)
_pd = ctypes.POINTER(ctypes.c_double)

# name -> (restype, argtypes); every symbol declared in include/ifmm_b200.h
SIGNATURES = {
    "ifmm_last_error": (ctypes.c_char_p, []),
    "ifmm_last_singular": (_i32, [_pi32, _pi32, _pd]),
    "ifmm_version": (_i32, []),
    "ifmm_device_count": (_i32, []),
    "ifmm_set_device": (_i32, [_i32]),
    "ifmm_release_cached_memory": (_i32, []),
    "ifmm_tree_build": (_i32, [_p, _i64, _i32, _i32, _i32, ctypes.POINTER(_p)]),
    "ifmm_tree_build_sparse": (_i32, [_p, _i64, _i32, _i32, _i32, ctypes.POINTER(_p)]),
    "ifmm_tree_info": (_i32, [_p, _pi64, _pi32, _pi32]),
    "ifmm_tree_permutation": (_i32, [_p, _p]),
    "ifmm_tree_leaf_offsets": (_i32, [_p, _p]),
    "ifmm_tree_lists": (_i32, [_p, _i32, _p, _p, _p, _p, _p]),
    "ifmm_tree_colours": (_i32, [_p, _i32, _p]),
    "ifmm_tree_free": (None, [_p]),
    "ifmm_store_init": (_i32, [_p, _i32, _d, _d, _d, _i32, _d, _p, _i32, ctypes.POINTER(_p)]),
    "ifmm_store_max_init_rank": (_i32, [_p, _pi32]),
    "ifmm_store_dims": (_i32, [_p, _i32, _p, _p]),
    "ifmm_store_basis": (_i32, [_p, _i32, _i32, _p]),
    "ifmm_store_m2l": (_i32, [_p, _i32, _i32, _i32, _p]),
    "ifmm_store_p2p": (_i32, [_p, _i32, _i32, _p]),
    "ifmm_store_bytes": (_i32, [_p, _p]),
    "ifmm_store_set_basis": (_i32, [_p, _i32, _i32, _p]),
    "ifmm_store_set_m2l": (_i32, [_p, _i32, _i32, _i32, _p]),
    "ifmm_store_set_p2p": (_i32, [_p, _i32, _i32, _p]),
    "ifmm_extended_layout": (_i32, [_p, _pi64, _p, _p, _p, _p]),
    "ifmm_extended_dense": (_i32, [_p, _i64, _pi64, _p]),
    "ifmm_matvec": (_i32, [_p, _p, _p, _i64, _i32]),
    "ifmm_store_free": (None, [_p]),
    "ifmm_factorize": (_i32, [_p, _d, _i32, _d, ctypes.POINTER(_p)]),
    "ifmm_factorize_rank_control": (_i32, [_p, _d, _i32, _d, _d, ctypes.POINTER(_p)]),
    "ifmm_factor_rank_control": (_i32, [_p, _p]),
    "ifmm_factor_info": (_i32, [_p, _pi32, _pi32, _pi64, _pd]),
    "ifmm_factor_level_stats": (_i32, [_p, _i32, _p]),
    "ifmm_factor_level_cond": (_i32, [_p, _i32, _pd]),
    "ifmm_factor_singular": (_i32, [_p, _i64, _p, _p, _p, _pi64]),
    "ifmm_factor_record": (_i32, [_p, _i64, _p, _p, _p]),
    "ifmm_factor_record_lu": (_i32, [_p, _i64, _p, _p]),
    "ifmm_factor_top": (_i32, [_p, _p, _p, _p]),
    "ifmm_factor_records": (_i32, [_p, _p]),
    "ifmm_factor_work": (_i32, [_p, _p]),
    "ifmm_factor_timing": (_i32, [_p, _p, _p]),
    "ifmm_factor_timing_level": (_i32, [_p, _i32, _p]),
    "ifmm_launch_count": (_i64, []),
    "ifmm_solve": (_i32, [_p, _p, _p, _i64, _i32]),
    "ifmm_solve_refined": (_i32, [_p, _p, _p, _p, _i64, _i32, _i32, _d, _p, _p]),
    "ifmm_factor_free": (None, [_p]),
    "ifmm_comm_nccl_unique_id": (_i32, [_p]),
    "ifmm_comm_nccl_version": (_i32, [_pi32]),
    "ifmm_comm_nccl_init": (_i32, [_p, _i32, _i32, ctypes.POINTER(_p)]),
    "ifmm_comm_host_init": (_i32, [_i32, _i32, _p, _p, _p, ctypes.POINTER(_p)]),
    "ifmm_comm_free": (None, [_p]),
    "ifmm_comm_selftest": (_i32, [_p, _i64, _pi32]),
    "ifmm_factorize_sharded": (_i32, [_p, _p, _d, _i32, _d, ctypes.POINTER(_p)]),
    "ifmm_factorize_emulated": (_i32, [_p, _i32, _d, _i32, _d, _p]),
    "ifmm_factorize_sharded_rank_control": (_i32, [_p, _p, _d, _i32, _d, _d, ctypes.POINTER(_p)]),
    "ifmm_factorize_emulated_rank_control": (_i32, [_p, _i32, _d, _i32, _d, _d, _p]),
    "ifmm_solve_emulated": (_i32, [_p, _i32, _p, _p, _i64, _i32]),
    "ifmm_factor_shard_info": (_i32, [_p, _p, _p]),
    "ifmm_partition": (_i32, [_i32, _i32, _i32, _i32, _p, _p]),
    "ifmm_partition_halo_counts": (_i32, [_i32, _i32, _i32, _i32, _i32, _i32, _p, _p]),
    "ifmm_test_lu": (_i32, [_p, _p, _i32, _p, _p, _p]),
    "ifmm_test_lu_solve_x": (_i32, [_p, _p, _i32, _i32, _p, _i32, _p, _p]),
    "ifmm_test_gemm": (_i32, [_i32, _i32, _i32, _i32, _i32, _d, _p, _i32, _p, _i32, _d, _p, _i32, _i32]),
    "ifmm_test_set_group": (_i32, [_i32]),
    "ifmm_test_recompress": (_i32, [_p, _i32, _i32, _d, _p, _i32, _p, _p, _p, _p, _p]),
    "ifmm_test_jacobi": (_i32, [_p, _i32, _i32, _p, _p]),
    "ifmm_test_qr": (_i32, [_p, _i32, _i32, _p, _p]),
    "ifmm_test_aca": (_i32, [_p, _i32, _i32, _d, _p, _i32, _p, _p, _p, _p]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class SingularPivotError(RuntimeError):
    """Numerically singular pivot block (ifmm/solver.py:53-60)."""

    def __init__(self, level: int, index: int, cond: float):
        super().__init__(
            f"pivot for cluster {index} at level {level} is numerically "
            f"singular (condition estimate {cond:.2e})")
        self.level = level
        self.index = index


def check(status: int) -> None:
    if status == OK:
        return
    msg = lib.ifmm_last_error().decode(errors="replace")
    if status == INVALID:
        raise ValueError(msg)
    if status == SINGULAR:
        lv, ix, cd = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
        lib.ifmm_last_singular(ctypes.byref(lv), ctypes.byref(ix), ctypes.byref(cd))
        raise SingularPivotError(lv.value, ix.value, cd.value)
    if status == OOM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def as_input(x, rows: int):
    """Normalise a (rows,) / (rows, k) numpy array or CUDA torch tensor.

    Returns (pointer, ptr_kind, nrhs, keepalive, is_torch, was_1d)."""
    if type(x).__module__.startswith("torch"):
        import torch  # only when the caller already uses torch
        t = x.detach()
        if t.dim() not in (1, 2) or t.shape[0] != rows:
            raise ValueError(f"expected shape ({rows},) or ({rows}, k), got {tuple(t.shape)}")
        t = t.to(torch.float64).contiguous()
        nr = 1 if t.dim() == 1 else int(t.shape[1])
        kind = PTR_DEVICE if t.is_cuda else PTR_HOST
        if kind == PTR_DEVICE:
            # the library reads device buffers on its own stream: wait for torch's
            # stream to finish producing this tensor (and the copy made above)
            if t.device.index != torch.cuda.current_device():
                raise ValueError(f"tensor on {t.device}, but the library runs on cuda:{torch.cuda.current_device()}")
            torch.cuda.current_stream(t.device).synchronize()
        if kind == PTR_HOST:
            a = t.numpy()
            return ptr(a), PTR_HOST, nr, a, True, t.dim() == 1
        return ctypes.c_void_p(t.data_ptr()), PTR_DEVICE, nr, t, True, t.dim() == 1
    a = np.ascontiguousarray(np.asarray(x, dtype=float))
    if a.ndim not in (1, 2) or a.shape[0] != rows:
        raise ValueError(f"expected shape ({rows},) or ({rows}, k), got {a.shape}")
    nr = 1 if a.ndim == 1 else a.shape[1]
    return ptr(a), PTR_HOST, nr, a, False, a.ndim == 1


def alloc_output(like, kind: int, rows: int, nrhs: int, one_d: bool):
    """Output buffer matching an input normalised by as_input."""
    if kind == PTR_DEVICE:
        import torch
        out = torch.empty((rows, nrhs), dtype=torch.float64, device=like.device)
        return out, ctypes.c_void_p(out.data_ptr())
    out = np.empty((rows, nrhs))
    return out, ptr(out)


ACA_PROBE_STRIDE = 22


def aca_probe_row(m: int) -> np.ndarray:
    """One row of the ACA probe table for an m-row fill: the reference's probe
    draw np.random.default_rng(0).choice(m, size=min(10, m), replace=False)
    (ifmm/lowrank.py:196-197), then the PCG64 state it leaves (state, increment
    as hi/lo 64-bit words, has_uint32, uinteger) -- the stream the reference's
    random restart rows continue (ifmm/lowrank.py:224-226)."""
    row = np.zeros(ACA_PROBE_STRIDE, dtype=np.int32)
    rng = np.random.default_rng(0)
    d = rng.choice(m, size=min(10, m), replace=False)
    row[:len(d)] = d
    st = rng.bit_generator.state
    mask = (1 << 64) - 1
    s, inc = st["state"]["state"], st["state"]["inc"]
    words = np.array([s >> 64, s & mask, inc >> 64, inc & mask, st["has_uint32"], st["uinteger"]], dtype=np.uint64)
    row[10:] = words.view(np.int32)
    return row


def aca_probe_table(maxm: int = 4096) -> np.ndarray:
    """Probe rows (+ generator state) of the reference's ACA for every fill
    height m <= maxm (rows of aca_probe_row)."""
    global _PROBES
    if _PROBES is not None and _PROBES.shape[0] > maxm:
        return _PROBES
    tab = np.zeros((maxm + 1, ACA_PROBE_STRIDE), dtype=np.int32)
    for m in range(1, maxm + 1):
        tab[m] = aca_probe_row(m)
    _PROBES = tab
    return tab


_PROBES = None
