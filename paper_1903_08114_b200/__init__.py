"""B200-native exact-GP BBMM hot path (arXiv 1903.08114), a drop-in for the
blockgp reference package's kernel / partitioned-MVM / mBCG / preconditioner /
MLL / prediction API.

All O(n) and O(n^2) work runs in hand-written sm_100a CUDA kernels behind the
C ABI in include/gpbbmm.h (built in-tree as _lib/libgpbbmm.so); Python keeps
only the reference's host-side orchestration. There is no CPU fallback.
"""

from .errors import ConvergenceError, NumericError, TrainingError
from .kernels import (KernelModel, default_model, kernel_block, kernel_block_grad, kernel_eval,
                      load_model, model_from_text, model_to_raw, model_to_text, raw_to_model,
                      save_model)
from .partition import (PartitionPlan, WorkerPool, partitioned_mvm, plan_from_budget,
                        plan_partitions, track_allocations)
from .precond import (PivotedFactor, PreconditionerCache, build_preconditioner,
                      partial_pivoted_cholesky, precond_apply, precond_sample)
from .cg import SolveReport, SolveRequest, Tridiagonal, mbcg_solve, slq_logdet
from .likelihood import CgConfig, MLLResult, mll_value_and_grad
from .predictor import (CgPredictor, PredictionCache, PredOutput, build_cache, load_cache,
                        predict, predict_mean, predict_variance, save_cache, verify_cache)
from .data import Dataset, RawTable, split_and_whiten
from .love import LoveCache, build_love_cache, predict_variance_love
from .trainer import AdamConfig, LbfgsConfig, MllObjective, TrainConfig, TrainTrace, train

__version__ = "0.1.0"
