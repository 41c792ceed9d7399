"""B200-native (sm_100a) LR-PD-SDP hot path: a drop-in for the reference
``pdsdp`` package's ``solve_lr_pd_sdp`` (arXiv 1810.05231, Algorithm 2).

Public names mirror the reference's ``pdsdp/__init__.py:9-81`` for the hot
path; the per-iteration arithmetic runs in ``libpdsdp_b200.so`` (hand-written
CUDA for sm_100a behind the C ABI in ``include/pdsdp_b200.h``).
"""

from .config import (
    Checkpoint,
    ProgressInfo,
    RankController,
    SolutionReport,
    SolveResult,
    SolveStatus,
    SolverConfig,
    rank_certificate_satisfied,
    stall_detected,
    update_rank,
)
from .io import (
    ParseError,
    load_problem,
    parse_extended,
    parse_sdpa,
    read_solution,
    write_extended,
    write_sdpa,
    write_solution,
)
from .layout import EigenDecomposition, SymMatrix, approx_error_bound, packed_index, packed_length, smat, svec
from .model import SdpProblem, SparseRow, as_problem
from .operators import apply_M, apply_M_adjoint, aproj_psd
from .solver import (
    check_solution,
    estimate_operator_norm,
    solve_lr_pd_sdp,
    solve_lr_pd_sdp_batch,
    solve_pd_sdp,
    step_size,
)

__all__ = [
    "Checkpoint", "EigenDecomposition", "ProgressInfo", "RankController", "SdpProblem",
    "SolveResult", "SolveStatus", "SolverConfig", "SparseRow", "SymMatrix", "apply_M",
    "apply_M_adjoint", "aproj_psd", "as_problem", "approx_error_bound", "estimate_operator_norm",
    "SolutionReport", "check_solution", "solve_pd_sdp",
    "ParseError", "load_problem", "parse_extended", "parse_sdpa", "read_solution", "write_extended",
    "write_sdpa", "write_solution",
    "packed_index", "packed_length", "rank_certificate_satisfied", "smat", "solve_lr_pd_sdp", "solve_lr_pd_sdp_batch",
    "stall_detected", "step_size", "svec", "update_rank",
]

__version__ = "0.1.0"
