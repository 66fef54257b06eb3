"""B200-native IFMM factorize/solve (drop-in for the reference `ifmm` hot path).

Same public names as the reference package (ifmm/__init__.py:73-104) for the
factorize/solve path; every numerical step runs in hand-written sm_100a CUDA
(libifmm_b200.so, include/ifmm_b200.h).  There is no CPU fallback.
"""
from ._lib import SingularPivotError
from .estimator import IfmmSolver, default_depth
from .geometry import ClusterTree, Cluster, PointSet, build_tree, compute_lists, morton_decode, morton_encode
from .kernels import KERNEL_NAMES, Kernel, baseline_kernel, kernel_block, make_kernel
from .operators import (OperatorStore, assemble_extended_dense, dump_extended, extended_layout, extended_restrict_x,
                        extended_rhs, fmm_matvec, init_operators, load_operator_blocks)
from .solver import IfmmFactorization, LevelStats, factorize, solve
from . import distributed  # noqa: E402  (sharded factorize / solve)

__all__ = [
    "Cluster",
    "ClusterTree",
    "IfmmFactorization",
    "IfmmSolver",
    "KERNEL_NAMES",
    "Kernel",
    "LevelStats",
    "OperatorStore",
    "PointSet",
    "SingularPivotError",
    "baseline_kernel",
    "build_tree",
    "assemble_extended_dense",
    "compute_lists",
    "dump_extended",
    "extended_layout",
    "extended_restrict_x",
    "extended_rhs",
    "default_depth",
    "factorize",
    "fmm_matvec",
    "init_operators",
    "kernel_block",
    "load_operator_blocks",
    "make_kernel",
    "morton_decode",
    "morton_encode",
    "solve",
]

__version__ = "0.1.0"
