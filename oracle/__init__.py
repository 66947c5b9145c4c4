"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (fp64, numpy/scipy) of what
the hot path of arXiv 1601.08179 computes: the statically condensed
spectral-element Helmholtz operator, defined as the dense Schur complement
H_BB - H_BI H_II^{-1} H_IB of the element matrix on GLL points (PAPER.md
P:198-225), assembled over a Cartesian grid, inside a
block-Jacobi preconditioned conjugate-gradient solve.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_1601_08179_b200``): it never uses the fast-diagonalisation
(FDM), the transformed factorisation (TPT) or any GPU-path helper.  The single
exception is ``basis.interior_eigen`` (the generalized eigenproblem of Eq.
eq:generalized_eigenvalues, solved with scipy.linalg.eigh), used only to
express vectors in the transformed basis for basis-convention checks
(SURVEY.md §8(c) c2, c6, c8).

Modules
-------
basis     GLL rule, Lagrange derivative matrix, 1-D M and K
element   metric coefficients d_e, dense element matrix, B/I split, Schur complement
          
mesh      Cartesian lattice numbering, gather R / scatter R^T, skeleton + Dirichlet masks
          
operator  assembled condensed operator y = R Hhat R^T x (MMC-style DGEMM)
pcg       conjugate gradients with a preconditioner callback (Hestenes-Stiefel)
solve     Alg. 1 pipeline: condensed RHS, block-Jacobi preconditioner, recovery (P:226-246,
          P:597-607)

Parity status: every function here is pinned by ``tests/test_oracle_*.py``
(closed forms, invariants, brute force); nothing is "parity unpinned" except
PCG iteration counts beyond the oracle's own PCG (the paper prints none,
SURVEY.md §8(c) "Pins per oracle part").
"""
