"""Preconditioned conjugate gradients (ORACLE, test infrastructure only).

PAPER.md P:594: "a conjugate gradient solver suffices [Hestenes & Stiefel]".
Standard PCG, x0 = 0, stopping rule of SURVEY §8(c) c6: stop as soon as
norm(r_k) <= rtol * norm(r_0) for the recursively updated residual; the
iteration count is the number of operator applications A p in the loop.
"""
import numpy as np


class PCGResult:
    def __init__(self, x, iters, converged, history, breakdown=False):
        self.x = x
        self.iters = iters
        self.converged = converged
        self.history = history
        self.breakdown = breakdown


def pcg(apply_A, apply_Pinv, b, rtol=1e-10, maxit=1000, norm=None, dot=None, fixed_iters=None):
    """Solve A x = b; apply_Pinv(r) returns z = P^{-1} r.

    norm(r): the residual norm used by the stopping rule (default Euclidean).
    dot(a, b): inner product (default np.dot).
    fixed_iters: if given, run exactly that many iterations (no stopping test).
    """
    if norm is None:
        norm = lambda v: float(np.sqrt(np.dot(v, v)))
    if dot is None:
        dot = lambda a, c: float(np.dot(a, c))
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    r = b.copy()
    z = apply_Pinv(r)
    p = z.copy()
    rz = dot(r, z)
    r0 = norm(r)
    history = [r0]
    if r0 == 0.0:
        return PCGResult(x, 0, True, history)
    nmax = fixed_iters if fixed_iters is not None else maxit
    k = 0
    converged = False
    while k < nmax:
        q = apply_A(p)
        pq = dot(p, q)
        if pq <= 0.0:
            return PCGResult(x, k, False, history, breakdown=True)
        alpha = rz / pq
        x += alpha * p
        r -= alpha * q
        k += 1
        rn = norm(r)
        history.append(rn)
        if fixed_iters is None and rn <= rtol * r0:
            converged = True
            break
        z = apply_Pinv(r)
        rz_new = dot(r, z)
        beta = rz_new / rz
        p = z + beta * p
        rz = rz_new
    return PCGResult(x, k, converged, history)
