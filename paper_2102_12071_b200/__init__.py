"""B200-native learned-smoother multigrid (hot path of arXiv 2102.12071).

Drop-in facade for the reference package's solver API (mgsmooth 0.1.0,
__init__.py:9-35) restricted to the hot path: grids and stencil fields, full
coarsening transfers and Galerkin products, the stencil -> smoother CNN, the
per-point smoother, the V-cycle and the solve loop.  Everything numeric runs
in hand-written sm_100a CUDA kernels behind the C-ABI in include/mgb.h
(libmgb.so, built by ``python -m paper_2102_12071_b200.build``).
"""

from .errors import (ConfigError, ContractError, MgError, NonConvergedError, NumericError,
                     SingularMatrixError, TrainingError, UnsupportedOperationError)
from .grid import (ConvKernel, GridFunction, GridSpec, StencilField, apply_stencil, compose_kernels,
                   constant_stencil, convolve, delta_kernel, from_active, full_spec, pad_kernel, to_active, zeros)
from .transfer import TransferPair, coarsen_full, galerkin_product, prolong, restrict
from .smoothers import (ConvSmoother, InferredSmoother, JacobiSmoother, KernelInferenceNet, conv_smoother,
                        effective_kernel, infer_kernels, inference_net, jacobi, load_model, model_from_dict,
                        model_to_dict, representative_diagonal, save_model)
from .hierarchy import (Level, MultigridHierarchy, RepeatedSmoother, SolveReport, build_hierarchy,
                        build_hierarchy_batch, build_hierarchy_classed, coarse_solve, cycle_correction, equip_classical,
                        equip_conv_init, equip_inferred, equip_trained, retarget, solve, v_cycle)
from .autodiff import grad_check
from .problems import ProblemSpec, build_geometry
from .training import (LossRecord, TrainConfig, TrainingSample, forward_loss, make_dataset, retrain_with_injection,
                       train_adaptive, train_independent, train_inference_net, train_level, train_mixture)
from .krylov import (CyclePreconditioner, FgmresConfig, GridAction, KrylovReport, cycle_preconditioner, fgmres,
                     gmres, grid_action)

__version__ = "0.1.0"
