"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/sc.h
declares, validates arguments, and its host-side L0 (1-D transformed basis) matches
the oracle's independent construction."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "sc.h")


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1601_08179_b200 import capi
    return capi.load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sc_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(lib):
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    from paper_1601_08179_b200 import capi
    assert set(names) == set(capi.SIGNATURES), set(names) ^ set(capi.SIGNATURES)


def test_library_is_sm100a(lib):
    from paper_1601_08179_b200 import capi
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", capi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_setup_rejects_invalid_without_side_effects(lib):
    from paper_1601_08179_b200.capi import ScParams, SC_EINVAL
    h = np.ones(4)
    def call(p=4, ne=(2, 2, 2), lam=1.0, hval=1.0, nranks=1, rank=0):
        hh = np.full(4, hval)
        prm = ScParams()
        prm.p = p
        for d in range(3):
            prm.ne[d] = ne[d]
            prm.h[d] = hh.ctypes.data
        prm.lam = lam
        prm.device = 0
        prm.nccl_comm = None
        prm.rank = rank
        prm.nranks = nranks
        ctx = ctypes.c_void_p()
        st = lib.sc_setup(ctypes.byref(prm), ctypes.byref(ctx))
        return st, ctx
    for kw in (dict(p=1), dict(p=33), dict(ne=(0, 2, 2)), dict(lam=-1.0), dict(lam=float("nan")),
               dict(hval=0.0), dict(hval=float("inf")), dict(nranks=2, rank=0), dict(rank=1)):
        st, ctx = call(**kw)
        assert st == SC_EINVAL, kw
        assert not ctx.value
    assert lib.sc_basis_1d_host(1, None, None, None, None, None, None) == SC_EINVAL
    assert lib.sc_basis_1d_host(33, None, None, None, None, None, None) == SC_EINVAL
    del h


@pytest.mark.parametrize("p", [2, 3, 4, 5, 8, 12, 16, 24, 32])
def test_host_basis_matches_oracle(lib, p):
    """Convention-free comparison (ascending Lambda, a0 > 0 rule applied on both sides)."""
    from paper_1601_08179_b200 import basis_1d_host
    from oracle import basis
    B = basis_1d_host(p)
    lam, S = basis.interior_eigen(p)
    x, w, K = basis.mass_stiffness(p)
    assert np.allclose(B["w"], w, rtol=1e-14, atol=0)
    assert np.abs(B["lam"] - lam).max() <= 1e-13 * lam.max()
    assert np.abs(B["S"] - S).max() <= 1e-10
    a0 = S @ K[1:p, 0]
    assert np.abs(B["a0"] - a0).max() <= 1e-10 * a0.max()
    assert abs(B["K00"] - K[0, 0]) <= 1e-13 * abs(K[0, 0]) * p
    assert abs(B["K0p"] - K[0, p]) <= 1e-13 * abs(K[0, 0]) * p
    assert abs(B["w0"] - w[0]) < 1e-16
    # parity of the eigenvectors: |ap| = |a0| to rounding in long double
    assert B["parity_err"] < 1e-15
    assert np.all(B["a0"] > 0)
    # S M S^T = I and S K S^T = Lambda with the library's own S
    MII = np.diag(w[1:p])
    assert np.allclose(B["S"] @ MII @ B["S"].T, np.eye(p - 1), atol=1e-13)
    assert np.allclose(B["S"] @ K[1:p, 1:p] @ B["S"].T, np.diag(B["lam"]), atol=1e-12 * lam.max())
