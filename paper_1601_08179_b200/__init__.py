"""B200-native condensed spectral-element Helmholtz solver (arXiv 1601.08179, TPT + BT).

The product is libsc.so (csrc/, C-ABI in include/sc.h): hand-written sm_100a CUDA
kernels for the condensed operator, the BT-PCG loop and the per-solve pre/post steps.
This package is the thin Python binding (``capi``: ctypes declarations with the C
names; ``solver.Context``: workspace owned by torch).  It never imports ``oracle``.
"""
from . import capi
from .capi import SC_PERM, SC_PRIMAL, SC_DUAL, ScError

__all__ = ["capi", "SC_PERM", "SC_PRIMAL", "SC_DUAL", "ScError", "Context", "context_for_grid",
           "basis_1d_host", "layout_query", "LoopbackGroup"]


def __getattr__(name):
    if name in ("Context", "context_for_grid", "basis_1d_host", "layout_query", "LoopbackGroup"):
        from . import solver
        return getattr(solver, name)
    raise AttributeError(name)
