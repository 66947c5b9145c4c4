"""Python front end of the C-ABI: one context per (grid, rank) with torch-owned workspace.

Marshalling only -- every step of the hot path runs in libsc.so's CUDA kernels.
"""
import ctypes

import numpy as np
import torch

from . import capi
from .capi import ScParams, ScLayoutInfo, ScPcgReport, ScError, ptr, stream_handle


def _check(lib, ctx, fn, st):
    if st != capi.SC_OK:
        msg = lib.sc_last_error(ctx).decode() if ctx else ""
        raise ScError(fn, st, msg)


def basis_1d_host(p):
    """L0 1-D transformed basis computed by the library's host code (no GPU needed)."""
    lib = capi.load()
    ni = p - 1
    lam, a0, ap = (np.zeros(ni) for _ in range(3))
    S = np.zeros(ni * ni)
    w = np.zeros(p + 1)
    kt = np.zeros(4)
    dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    st = lib.sc_basis_1d_host(p, dp(lam), dp(a0), dp(ap), dp(S), dp(w), dp(kt))
    if st != capi.SC_OK:
        raise ScError("sc_basis_1d_host", st)
    return dict(lam=lam, a0=a0, ap=ap, S=S.reshape(ni, ni), w=w, K00=kt[0], K0p=kt[1], w0=kt[2],
                parity_err=kt[3])


def layout_query(p, ne, widths, lam, rank=0, nranks=1):
    """sc_layout_query: the slab layout sc_setup would use on this rank (host only, no GPU)."""
    lib = capi.load()
    hs = [np.ascontiguousarray(np.asarray(w, dtype=np.float64)) for w in widths]
    prm = ScParams()
    prm.p = int(p)
    for d in range(3):
        prm.ne[d] = int(ne[d])
        prm.h[d] = hs[d].ctypes.data
    prm.lam = float(lam)
    prm.device = 0
    prm.nccl_comm = None
    prm.rank = int(rank)
    prm.nranks = int(nranks)
    L = ScLayoutInfo()
    st = lib.sc_layout_query(ctypes.byref(prm), ctypes.byref(L))
    if st != capi.SC_OK:
        raise ScError("sc_layout_query", st)
    return L


class Context:
    """sc_setup + workspace.  widths: (hx[nx], hy[ny], hz[nz]) global element widths."""

    def __init__(self, p, ne, widths, lam, device=0, nccl_comm=None, rank=0, nranks=1):
        self.lib = capi.load()
        self.device = torch.device("cuda", device)
        self._h = [np.ascontiguousarray(np.asarray(w, dtype=np.float64)) for w in widths]
        prm = ScParams()
        prm.p = int(p)
        for d in range(3):
            prm.ne[d] = int(ne[d])
            prm.h[d] = self._h[d].ctypes.data
        prm.lam = float(lam)
        prm.device = int(device)
        prm.nccl_comm = nccl_comm
        prm.rank = int(rank)
        prm.nranks = int(nranks)
        ctx = ctypes.c_void_p()
        st = self.lib.sc_setup(ctypes.byref(prm), ctypes.byref(ctx))
        _check(self.lib, None, "sc_setup", st)
        self.ctx = ctx
        L = ScLayoutInfo()
        _check(self.lib, ctx, "sc_layout", self.lib.sc_layout(ctx, ctypes.byref(L)))
        self.layout = L
        self.p = p
        self.n_total = int(L.n_total)
        self.n_lattice = int(L.n_lattice)
        nbytes = int(self.lib.sc_workspace_bytes(ctx))
        self.workspace = torch.empty(nbytes // 8 + 32, dtype=torch.float64, device=self.device)
        base = self.workspace.data_ptr()
        aligned = (base + 255) // 256 * 256
        _check(self.lib, ctx, "sc_bind_workspace",
               self.lib.sc_bind_workspace(ctx, aligned, nbytes))

    # -- vectors -----------------------------------------------------------
    def skeleton(self, fill=0.0):
        return torch.full((self.n_total,), fill, dtype=torch.float64, device=self.device)

    def lattice(self, fill=0.0):
        return torch.full((self.n_lattice,), fill, dtype=torch.float64, device=self.device)

    # -- C-ABI calls (same names) ------------------------------------------
    def _s(self, stream):
        return stream_handle(stream if stream is not None else torch.cuda.current_stream(self.device))

    def sc_apply_condensed(self, x, y, stream=None):
        _check(self.lib, self.ctx, "sc_apply_condensed",
               self.lib.sc_apply_condensed(self.ctx, ptr(x), ptr(y), self._s(stream)))

    def sc_pcg_solve(self, b, x, rtol=1e-10, maxit=1000, stream=None):
        rep = ScPcgReport()
        st = self.lib.sc_pcg_solve(self.ctx, ptr(b), ptr(x), float(rtol), int(maxit), ctypes.byref(rep),
                                   self._s(stream))
        _check(self.lib, self.ctx, "sc_pcg_solve", st)
        return rep

    def sc_pcg_solve_host(self, h_b, h_x, rtol=1e-10, maxit=1000, stream=None):
        rep = ScPcgReport()
        st = self.lib.sc_pcg_solve_host(self.ctx, ptr(h_b), ptr(h_x), float(rtol), int(maxit),
                                        ctypes.byref(rep), self._s(stream))
        _check(self.lib, self.ctx, "sc_pcg_solve_host", st)
        return rep

    def sc_pcg_start(self, b, x, rtol=0.0, maxit=1 << 30, stream=None):
        _check(self.lib, self.ctx, "sc_pcg_start",
               self.lib.sc_pcg_start(self.ctx, ptr(b), ptr(x), float(rtol), int(maxit), self._s(stream)))

    def sc_pcg_iterate(self, niter, stream=None):
        _check(self.lib, self.ctx, "sc_pcg_iterate", self.lib.sc_pcg_iterate(self.ctx, int(niter), self._s(stream)))

    def sc_pcg_status(self, stream=None):
        rep = ScPcgReport()
        _check(self.lib, self.ctx, "sc_pcg_status", self.lib.sc_pcg_status(self.ctx, ctypes.byref(rep),
                                                                            self._s(stream)))
        return rep

    def sc_profile_enable(self, on=True):
        _check(self.lib, self.ctx, "sc_profile_enable", self.lib.sc_profile_enable(self.ctx, int(bool(on))))

    def sc_profile_read(self):
        ms = ctypes.c_double()
        n = ctypes.c_longlong()
        _check(self.lib, self.ctx, "sc_profile_read", self.lib.sc_profile_read(self.ctx, ctypes.byref(ms),
                                                                                ctypes.byref(n)))
        return ms.value, n.value

    def sc_condense_rhs(self, f, b, stream=None):
        _check(self.lib, self.ctx, "sc_condense_rhs",
               self.lib.sc_condense_rhs(self.ctx, ptr(f), ptr(b), self._s(stream)))

    def sc_recover(self, f, x, u, stream=None):
        _check(self.lib, self.ctx, "sc_recover",
               self.lib.sc_recover(self.ctx, ptr(f), ptr(x), ptr(u), self._s(stream)))

    def sc_condense_rhs_dirichlet(self, f, g, b, stream=None):
        _check(self.lib, self.ctx, "sc_condense_rhs_dirichlet",
               self.lib.sc_condense_rhs_dirichlet(self.ctx, ptr(f), ptr(g), ptr(b), self._s(stream)))

    def sc_recover_dirichlet(self, f, g, x, u, stream=None):
        _check(self.lib, self.ctx, "sc_recover_dirichlet",
               self.lib.sc_recover_dirichlet(self.ctx, ptr(f), ptr(g), ptr(x), ptr(u), self._s(stream)))

    def sc_to_transformed(self, v_lat, v_skel, mode, stream=None):
        _check(self.lib, self.ctx, "sc_to_transformed",
               self.lib.sc_to_transformed(self.ctx, ptr(v_lat), ptr(v_skel), int(mode), self._s(stream)))

    def sc_from_transformed(self, v_skel, v_lat, mode, stream=None):
        _check(self.lib, self.ctx, "sc_from_transformed",
               self.lib.sc_from_transformed(self.ctx, ptr(v_skel), ptr(v_lat), int(mode), self._s(stream)))

    def sc_fill_random(self, seed, v_skel, stream=None):
        _check(self.lib, self.ctx, "sc_fill_random",
               self.lib.sc_fill_random(self.ctx, int(seed), ptr(v_skel), self._s(stream)))

    def sc_dot(self, a, b, stream=None):
        out = ctypes.c_double()
        _check(self.lib, self.ctx, "sc_dot", self.lib.sc_dot(self.ctx, ptr(a), ptr(b), ctypes.byref(out),
                                                              self._s(stream)))
        return out.value

    def sc_preconditioner(self, out, stream=None):
        _check(self.lib, self.ctx, "sc_preconditioner",
               self.lib.sc_preconditioner(self.ctx, ptr(out), self._s(stream)))

    # -- PAPER.md §7 operator variants (nodal basis) --------------------------
    def sc_apply_tpc(self, x, y, stream=None):
        _check(self.lib, self.ctx, "sc_apply_tpc", self.lib.sc_apply_tpc(self.ctx, ptr(x), ptr(y), self._s(stream)))

    def sc_mmc_bytes(self):
        return int(self.lib.sc_mmc_bytes(self.ctx))

    def sc_mmc_bind(self, buf=None, stream=None):
        """Precompute the MMC element matrices into `buf` (a device tensor of >= sc_mmc_bytes bytes;
        allocated here when None).  The buffer is kept referenced by the context."""
        nbytes = self.sc_mmc_bytes()
        if buf is None:
            buf = torch.empty(nbytes // 8 + 1, dtype=torch.float64, device=self.device)
        self._mmc_buf = buf
        _check(self.lib, self.ctx, "sc_mmc_bind",
               self.lib.sc_mmc_bind(self.ctx, ptr(buf), buf.numel() * buf.element_size(), self._s(stream)))

    def sc_apply_mmc(self, x, y, stream=None):
        _check(self.lib, self.ctx, "sc_apply_mmc", self.lib.sc_apply_mmc(self.ctx, ptr(x), ptr(y), self._s(stream)))

    def sc_pcg_solve_nodal(self, b, x, op="tpc", prec="block", rtol=1e-10, maxit=1000, stream=None):
        """Solvers UC / DC / BC (prec "none" / "diag" / "block") on the nodal condensed system."""
        rep = ScPcgReport()
        opc = {"tpc": capi.SC_OP_TPC, "mmc": capi.SC_OP_MMC}[op]
        pc = {"none": capi.SC_PREC_NONE, "diag": capi.SC_PREC_DIAG, "block": capi.SC_PREC_BLOCK}[prec]
        st = self.lib.sc_pcg_solve_nodal(self.ctx, opc, pc, ptr(b), ptr(x), float(rtol), int(maxit),
                                         ctypes.byref(rep), self._s(stream))
        _check(self.lib, self.ctx, "sc_pcg_solve_nodal", st)
        return rep

    def sc_basis_1d(self):
        ni = self.p - 1
        lam, a0, ap = (np.zeros(ni) for _ in range(3))
        S = np.zeros(ni * ni)
        w = np.zeros(self.p + 1)
        kt = np.zeros(4)
        dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        _check(self.lib, self.ctx, "sc_basis_1d",
               self.lib.sc_basis_1d(self.ctx, dp(lam), dp(a0), dp(ap), dp(S), dp(w), dp(kt)))
        return dict(lam=lam, a0=a0, ap=ap, S=S.reshape(ni, ni), w=w, K00=kt[0], K0p=kt[1], w0=kt[2])

    def operator_kernel(self):
        return self.lib.sc_operator_kernel(self.ctx).decode()

    def launch_count(self):
        return int(self.lib.sc_launch_count(self.ctx))

    # -- convenience (nodal lattice <-> transformed skeleton) ---------------
    def to_lattice_nodal(self, v_skel, dual=False):
        out = self.lattice()
        self.sc_from_transformed(v_skel, out, capi.SC_DUAL if dual else capi.SC_PRIMAL)
        return out

    def from_lattice_nodal(self, v_lat, dual=False):
        out = self.skeleton()
        self.sc_to_transformed(v_lat, out, capi.SC_DUAL if dual else capi.SC_PRIMAL)
        return out

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.sc_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackGroup:
    """sc_loopback_comms_create: nranks in-process communicator handles for ranks that are host
    threads of this process (tests of the multi-rank path on one GPU).  comms[r] goes into
    Context(..., nccl_comm=comms[r], rank=r, nranks=nranks)."""

    def __init__(self, nranks):
        self.lib = capi.load()
        self.nranks = int(nranks)
        self._arr = (ctypes.c_void_p * self.nranks)()
        st = self.lib.sc_loopback_comms_create(self.nranks, self._arr)
        if st != capi.SC_OK:
            raise ScError("sc_loopback_comms_create", st)
        self.comms = [ctypes.c_void_p(self._arr[r]) for r in range(self.nranks)]

    def close(self):
        if self._arr is not None:
            self.lib.sc_loopback_comms_destroy(self._arr, self.nranks)
            self._arr = None


def context_for_grid(grid, device=0, **kw):
    """Context from a synth.Grid (p, ne, hx, hy, hz, lam)."""
    return Context(grid.p, grid.ne, (grid.hx, grid.hy, grid.hz), grid.lam, device=device, **kw)
