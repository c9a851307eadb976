"""B200-native BAMG setup + AMG-preconditioned GMRES for Markov-chain steady states.

Drop-in for the hot path of arxiv/paper_1402_4005 (`markovmg`): the names and
signatures below mirror markovmg/__init__.py:39-60 for that path; the compute
runs in libbamg_sm100.so (hand-written sm_100a kernels, C ABI in
include/bamg_sm100.h).  There is no CPU fallback: without the built library
or a CUDA device the entry points raise `BamgUnavailable`.
"""

from ._lib import BamgError, BamgUnavailable
from .bootstrap import (Hierarchy, Level, SetupConfig, SetupResult, TripletSet, bootstrap_cycle,
                        coarsest_triplets, complexities, export_hierarchy, init_test_vectors,
                        levels_at_least, run_setup, triplet_residual)
from .chains import (ChainProblem, birth_death, make_chain, molloy_net, petri_reachability,
                     random_planar, tandem_queue, uniform_2d)
from .coarsen import (CfSplitting, CoarseningConfig, cr_coarsen, geometric_coarsen, make_splitting,
                      splitting_from_mask)
from .dense import PinvOperator
from .device import DeviceCSR
from .fov import (FovResult, ProjectedSystem, eigenvalue_dots, elman_bound, fov_boundary, project_range,
                  projected_preconditioned, theorem2_bound)
from .interp import (InterpConfig, WeightedTestSet, build_interpolation, build_restriction,
                     singular_test_weights)
from .presets import PRESETS, build_problem, default_setup_config
from .relax import SmootherConfig, degenerate_rows, jacobi_sweep, jacobi_sweep_transpose
from .solver import (GmresConfig, SolveReport, VCycleOperator, gmres, report_to_json,
                     residuals_to_csv, solve_steady_state)
from .sparse import (adjacency_structure, make_csr, spmv, spmv_transpose, transpose,
                     triple_product)

__version__ = "0.1.0"
