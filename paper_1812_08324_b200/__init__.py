"""B200-native Crank-Nicolson H-matrix solver for 1D Levy-generator equations.

Drop-in for the hot path of the reference package `levyh` (arxiv 1812.08324):
operator assembly (entry generation), compression, H-LU and time stepping,
with the reference's public Python names.  All arithmetic runs in
hand-written sm_100a CUDA kernels behind the C ABI in include/levyh_b200.h;
there is no CPU fallback.
"""
from . import _lib  # noqa: F401
from .fractional import (FracConfig, LevyMeasure, assemble_fractional_poisson_1d, cgmy_measure,  # noqa: F401
                         frac_kernel_constant, frac_stencil_1d, frac_symbol_1d, power_measure,
                         quartic_window, tail_mass_power_1d, windowed_second_moment, eval_i1, eval_i2,
                         eval_i3, frac_apply_1d, frac_apply_2d, windowed_second_moment_radial_2d,
                         tail_mass_square_2d, lshape_grid, lshape_boundary_distance, variable_order_field,
                         three_bump_source, assemble_variable_order, write_field_csv)
from .geometry import (ClusterNode, ClusterTree, Permutation, PointSet, admissible,  # noqa: F401
                       build_cluster_tree)
from .hmatrix import (HConfig, HMatrix, KernelExpansion, ToeplitzEntries, build_from_dense,  # noqa: F401
                      bcast_factors, build_from_expansion, build_toeplitz, build_toeplitz_nccl,
                      derive_toeplitz, dump_structure,
                      export_blocks, gaussian_expansion_1d, gaussian_expansion_2d, Cn2dEntries, h_entry, memory_report,
                      rank_bound_gaussian, structure_summary, to_dense)
from .hops import (SOLVE_METHODS, HFactorization, hlu, lowrank_add_recompress, matvec,  # noqa: F401
                   mul_dense, solve, trisolve_lower, trisolve_upper_right)
from .levy import (CNSystem, CNSystem2D, FracCNSystem, UniformGrid1D, UniformGrid2D, assemble_cn_1d,  # noqa: F401
                   assemble_cn_2d, gaussian_measure, run_cn, step_cn)
from .checkpoint import load_hmatrix, save_hmatrix  # noqa: F401
from .formats import (cache_load, cache_store, fit_loglog_slope, fit_order, median_time, read_csv,  # noqa: F401
                      write_csv)
from .solvers import IterationLog, gmres_restarted, operator, pcg  # noqa: F401

__version__ = "0.1.0"
