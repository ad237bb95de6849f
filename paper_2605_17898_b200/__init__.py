"""B200-native matrix-free K_y.V / CG / SLQ hot path of LightGP (arXiv 2605.17898).

Drop-in for the CG path of the reference package ``minigp``: same kernel
classes, grammar and hyper-parameter interface, same ``matrix_free_matvec``,
``cg_solve``, ``slq_logdet``, ``gp_fit(..., "cg")``, ``gp_predict`` and
``log_marginal_likelihood``; the compute runs in hand-written sm_100a CUDA
behind the C ABI in ``include/lightgp.h`` (``_lib/liblightgp.so``).
"""

__version__ = "0.1.0"

from .errors import (
    DimensionMismatchError,
    KernelParseError,
    MiniGpError,
    NonFiniteError,
    NonSquareError,
    NonSymmetricError,
    NotPositiveDefiniteError,
    OperatorNotSpdError,
    SingularTriangularError,
)
from .linalg import LEDGER, AllocationLedger, as_matrix, as_vector, tracked
from .kernels import (
    RBF,
    Kernel,
    Linear,
    Matern12,
    Matern32,
    Matern52,
    Periodic,
    Product,
    Scale,
    Sum,
    flatten_params,
    format_kernel,
    is_stationary,
    kernel_diag,
    kernel_eval,
    lower,
    n_params,
    parse_kernel,
    slab_buffer_count,
    unflatten_params,
)
from .solvers import (
    CgConfig,
    CgResult,
    KernelOperator,
    cg_solve,
    matrix_free_matvec,
    probe_block,
    slq_logdet,
)
from .models import (
    AUTO_CHOLESKY_MAX,
    CG_FIT_BLOCK,
    DENSE_OPERATOR_MAX,
    FIT_CG_TOLERANCE,
    ExactState,
    OptimizerConfig,
    exact_evidence_objective,
    flatten_model_params,
    gp_fit,
    gp_predict,
    log_marginal_likelihood,
    metrics,
    optimize_hyperparams,
    unflatten_model_params,
)

__all__ = [name for name in dir() if not name.startswith("_")]
