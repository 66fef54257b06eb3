"""CPU-only checks of the boundary: the C-ABI library loads, exports every
symbol include/ifmm_b200.h declares, and compute entry points refuse to run
(no CPU fallback) when there is no CUDA device."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "ifmm_b200.h")).read()
    return sorted(set(re.findall(r"\b(ifmm_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    from paper_1407_1572_b200 import _lib
    names = _declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(_lib.lib, n), n
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_1407_1572_b200", "libifmm_b200.so")
    blob = open(so, "rb").read()
    assert b"sm_100a" in blob


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1407_1572_b200 as ifmm
    pts = np.random.default_rng(0).uniform(-1, 1, (64, 2))
    with pytest.raises(RuntimeError, match="no CUDA device"):
        ifmm.build_tree(ifmm.PointSet(2, pts), 2)


def test_host_side_validation():
    import paper_1407_1572_b200 as ifmm
    with pytest.raises(ValueError):
        ifmm.PointSet(2, np.array([[0.0, 2.0]]))
    with pytest.raises(ValueError):
        ifmm.PointSet(4, np.zeros((3, 4)))
    with pytest.raises(ValueError):
        ifmm.make_kernel("nope")
    with pytest.raises(RuntimeError):
        ifmm.IfmmSolver().solve(np.zeros(3))


def test_probe_table_matches_reference_draw():
    from paper_1407_1572_b200 import _lib
    from oracle import ifmm_oracle as O
    tab = _lib.aca_probe_table(300)
    for m in (1, 2, 9, 10, 11, 57, 300):
        _, probes = O.aca_probe_rows(m)
        assert list(tab[m, :len(probes)]) == [int(v) for v in probes]


def test_probe_table_carries_the_generator_state():
    """Rows of the probe table continue the reference's generator: a Generator rebuilt
    from the stored PCG64 words draws what np.random.default_rng(0) draws after the probe
    choice (the random ACA restart rows, ifmm/lowrank.py:224-226)."""
    from paper_1407_1572_b200 import _lib
    for m in (1, 7, 10, 64, 513):
        row = _lib.aca_probe_row(m)
        w = [int(x) for x in row[10:].view(np.uint64)]
        g = np.random.Generator(np.random.PCG64())
        g.bit_generator.state = {"bit_generator": "PCG64", "state": {"state": (w[0] << 64) | w[1],
                                                                     "inc": (w[2] << 64) | w[3]},
                                 "has_uint32": w[4], "uinteger": w[5]}
        ref = np.random.default_rng(0)
        ref.choice(m, size=min(10, m), replace=False)
        for k in (1, 2, 5, m, 3 * m + 1):
            assert g.choice(list(range(k))) == ref.choice(list(range(k)))


def test_kernel_host_eval_matches_oracle():
    import paper_1407_1572_b200 as ifmm
    from oracle import ifmm_oracle as O
    r = np.linspace(0, 2, 101)
    for name in ifmm.KERNEL_NAMES:
        k = ifmm.make_kernel(name, a=0.01, scale=0.5, shift=0.25)
        spec = O.KernelSpec(name, a=0.01, scale=0.5, shift=0.25)
        assert np.allclose(k.func(r), O.kernel_eval(spec, r), rtol=1e-15, atol=0)
