"""Thin ctypes binding of include/sc.h (argument marshalling only).

Every entry point of the C-ABI is exposed under the same name.  Device vectors are
passed as torch CUDA tensors (fp64, contiguous) or raw integer device pointers;
streams as torch.cuda.Stream or raw cudaStream_t integers.  There is no fallback:
if libsc.so is missing or fails to load, ``load()`` raises.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SC_LIB_PATH", os.path.join(HERE, "_lib", "libsc.so"))

SC_OK, SC_EINVAL, SC_ENOMEM, SC_ECUDA, SC_ENCCL, SC_EBREAKDOWN, SC_ESTATE = range(7)
SC_PERM, SC_PRIMAL, SC_DUAL = 0, 1, 2
SC_OP_TPC, SC_OP_MMC = 1, 2
SC_PREC_NONE, SC_PREC_DIAG, SC_PREC_BLOCK = 0, 1, 2
STATUS_NAMES = {0: "SC_OK", 1: "SC_EINVAL", 2: "SC_ENOMEM", 3: "SC_ECUDA", 4: "SC_ENCCL",
                5: "SC_EBREAKDOWN", 6: "SC_ESTATE"}


class ScParams(ctypes.Structure):
    _fields_ = [("p", ctypes.c_int), ("ne", ctypes.c_int * 3), ("h", ctypes.c_void_p * 3),
                ("lam", ctypes.c_double), ("device", ctypes.c_int), ("nccl_comm", ctypes.c_void_p),
                ("rank", ctypes.c_int), ("nranks", ctypes.c_int)]


class ScLayoutInfo(ctypes.Structure):
    _fields_ = [("n_total", ctypes.c_longlong), ("n_free", ctypes.c_longlong),
                ("n_lattice", ctypes.c_longlong), ("n_lattice_global", ctypes.c_longlong),
                ("off_face", ctypes.c_longlong * 3), ("n_faces", ctypes.c_longlong * 3),
                ("off_edge", ctypes.c_longlong * 3), ("n_edges", ctypes.c_longlong * 3),
                ("off_vertex", ctypes.c_longlong), ("n_vertices", ctypes.c_longlong),
                ("ne_local", ctypes.c_int * 3), ("z_begin", ctypes.c_int), ("z_end", ctypes.c_int),
                ("p", ctypes.c_int), ("n_i", ctypes.c_int)]


class ScPcgReport(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int), ("converged", ctypes.c_int), ("relres", ctypes.c_double),
                ("r0norm", ctypes.c_double), ("t_solve_s", ctypes.c_double)]


_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
SIGNATURES = {
    "sc_setup": ([ctypes.POINTER(ScParams), ctypes.POINTER(_P)], ctypes.c_int),
    "sc_destroy": ([_P], ctypes.c_int),
    "sc_layout_query": ([ctypes.POINTER(ScParams), ctypes.POINTER(ScLayoutInfo)], ctypes.c_int),
    "sc_layout": ([_P, ctypes.POINTER(ScLayoutInfo)], ctypes.c_int),
    "sc_workspace_bytes": ([_P], ctypes.c_size_t),
    "sc_bind_workspace": ([_P, _P, ctypes.c_size_t], ctypes.c_int),
    "sc_basis_1d": ([_P, _D, _D, _D, _D, _D, _D], ctypes.c_int),
    "sc_basis_1d_host": ([ctypes.c_int, _D, _D, _D, _D, _D, _D], ctypes.c_int),
    "sc_apply_condensed": ([_P, _P, _P, _P], ctypes.c_int),
    "sc_pcg_solve": ([_P, _P, _P, ctypes.c_double, ctypes.c_int, ctypes.POINTER(ScPcgReport), _P], ctypes.c_int),
    "sc_pcg_solve_host": ([_P, _P, _P, ctypes.c_double, ctypes.c_int, ctypes.POINTER(ScPcgReport), _P],
                          ctypes.c_int),
    "sc_pcg_start": ([_P, _P, _P, ctypes.c_double, ctypes.c_int, _P], ctypes.c_int),
    "sc_pcg_iterate": ([_P, ctypes.c_int, _P], ctypes.c_int),
    "sc_pcg_status": ([_P, ctypes.POINTER(ScPcgReport), _P], ctypes.c_int),
    "sc_profile_enable": ([_P, ctypes.c_int], ctypes.c_int),
    "sc_profile_read": ([_P, _D, ctypes.POINTER(ctypes.c_longlong)], ctypes.c_int),
    "sc_condense_rhs": ([_P, _P, _P, _P], ctypes.c_int),
    "sc_recover": ([_P, _P, _P, _P, _P], ctypes.c_int),
    "sc_condense_rhs_dirichlet": ([_P, _P, _P, _P, _P], ctypes.c_int),
    "sc_operator_kernel": ([_P], ctypes.c_char_p),
    "sc_recover_dirichlet": ([_P, _P, _P, _P, _P, _P], ctypes.c_int),
    "sc_to_transformed": ([_P, _P, _P, ctypes.c_int, _P], ctypes.c_int),
    "sc_from_transformed": ([_P, _P, _P, ctypes.c_int, _P], ctypes.c_int),
    "sc_fill_random": ([_P, ctypes.c_uint64, _P, _P], ctypes.c_int),
    "sc_dot": ([_P, _P, _P, _D, _P], ctypes.c_int),
    "sc_preconditioner": ([_P, _P, _P], ctypes.c_int),
    "sc_nccl_unique_id": ([ctypes.c_char_p], ctypes.c_int),
    "sc_nccl_comm_init": ([ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)],
                          ctypes.c_int),
    "sc_nccl_comm_destroy": ([_P], ctypes.c_int),
    "sc_loopback_comms_create": ([ctypes.c_int, ctypes.POINTER(_P)], ctypes.c_int),
    "sc_loopback_comms_destroy": ([ctypes.POINTER(_P), ctypes.c_int], ctypes.c_int),
    "sc_apply_tpc": ([_P, _P, _P, _P], ctypes.c_int),
    "sc_mmc_bytes": ([_P], ctypes.c_size_t),
    "sc_mmc_bind": ([_P, _P, ctypes.c_size_t, _P], ctypes.c_int),
    "sc_apply_mmc": ([_P, _P, _P, _P], ctypes.c_int),
    "sc_pcg_solve_nodal": ([_P, ctypes.c_int, ctypes.c_int, _P, _P, ctypes.c_double, ctypes.c_int,
                            ctypes.POINTER(ScPcgReport), _P], ctypes.c_int),
    "sc_launch_count": ([_P], ctypes.c_longlong),
    "sc_last_error": ([_P], ctypes.c_char_p),
    "sc_version": ([], ctypes.c_char_p),
}

_lib = None


def load():
    """Load libsc.so (raises OSError / RuntimeError if it is missing -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libsc.so not built: {LIB_PATH} missing (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


class ScError(RuntimeError):
    def __init__(self, fn, status, msg=""):
        super().__init__(f"{fn} -> {STATUS_NAMES.get(status, status)} {msg}")
        self.status = status


def ptr(t):
    """Device/host pointer of a torch tensor, or pass through ints / None."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def stream_handle(s):
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream
