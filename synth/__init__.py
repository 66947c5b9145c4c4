"""Seeded synthetic inputs shared by the oracle-side tests and the GPU-side tests.

This module holds NONE of the method's arithmetic (no GLL, no operators, no
condensation).  It only defines:

* the counter-based splitmix64 uniform[-1, 1] generator keyed by
  (seed, global GLL-lattice index) -- SURVEY.md §8(c) reading c17;
* the workload grids of BASELINE.json (element counts, widths, lambda, p);
* the manufactured right-hand sides used by the configs
  (u = sin(pi x) sin(pi y) sin(pi z), f = (lambda + 3 pi^2) u) and the paper's E3 solution
  (Eq. eq:solution, k = 5) with its graded meshes.

The CUDA library implements the same counter-based generator on its own
(``sc_fill_random``); tests check the two agree bit for bit.
"""
from .splitmix import splitmix64, uniform_pm1, lattice_random, lattice_shape
from .grids import Grid, cfg1, cfg2, cfg3, cfg4, cfg5, small_grid, CFG3_P, nonuniform_grid, graded_widths, e3_grid
from .manufactured import sine_u, sine_f, e3_u, e3_f

__all__ = [
    "splitmix64", "uniform_pm1", "lattice_random", "lattice_shape",
    "Grid", "cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "small_grid", "CFG3_P",
    "sine_u", "sine_f", "nonuniform_grid", "graded_widths", "e3_grid", "e3_u", "e3_f",
]
