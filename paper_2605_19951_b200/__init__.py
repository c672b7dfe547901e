"""B200-native shifted-solve Gauss-Newton path of arXiv 2605.19951.

Drop-in for the reference package ``rbainv`` on the hot path: the same
public names (shifted / forward / sensitivity / inversion / regularization /
synthetic / rba data types), backed by sm_100a CUDA kernels in libdrba.so
(C ABI: include/rba_b200.h).  Importing the package does not need a GPU;
the device entry points raise if libdrba.so or the GPU is missing (there is
no CPU fallback).
"""

from .problem import Grid, Model, Problem
from .mesh3d import BoxSpec, build_box_problem, build_config, config_spec, spectral_bound
from .rba import (RationalApproximant, TimeChannels, config_approximant, load_approximant,
                  save_approximant)
from .shifted import (CacheCounters, CacheMissError, PoleWorkerPool, ShiftedFactorCache,
                      SolveError, default_worker_count, factorize_all_poles,
                      resolve_with_cache, solve_all_poles)
from .forward import ForwardResult, forward_response, response_from_pole_solutions
from .sensitivity import JacobianOperator, TaylorReport, adjoint_test, taylor_test
from .regularization import RegOperator, apply_sqrt, apply_sqrt_t, build_reg, reg_value_grad
from .inversion import (InversionConfig, InversionState, IterationRecord, LineSearchResult,
                        LsqrConfig, chi_squared, default_lambda0, gn_step, line_search,
                        run_inversion)
from .synthetic import DataSet, NoiseSpec, load_dataset, make_dataset, save_dataset
from .reporting import (RunReport, TimingModel, consolidate_report, fit_timing_model, load_state,
                        pole_solution_checksum, scaling_benchmark, write_run_artifacts)

__version__ = "0.1.0"
