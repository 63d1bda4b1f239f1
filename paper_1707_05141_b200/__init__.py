"""paper_1707_05141_b200: B200-native batched QR / one-sided Jacobi SVD / randomized SVD.

Drop-in for the reference package ``batchfact`` (/root/reference/pkg/src/batchfact)
on its batched hot path. The Python layer mirrors the reference's names, options,
result dataclasses and error conventions; every factorisation runs in hand-written
sm_100a CUDA kernels behind the C ABI in include/batchfact_b200.h
(``libbatchfact_b200.so``, loaded with ctypes). There is no CPU fallback.
"""

from ._lib import BackendUnavailable
from .blockjacobi import BlockJacobiOptions, BlockSvdResult, batch_block_svd, block_svd, block_svd_tensor
from .core import BatchError, as_matrix, read_matrix_text, write_matrix_text
from .helpers import (
    batch_apply,
    frobenius,
    gemm,
    householder_vector,
    jacobi_rotation,
    off_orthogonality,
    scaled_offdiag,
    syrk,
)
from .jacobi import (
    JacobiOptions,
    PairSchedule,
    SvdResult,
    batch_svd,
    round_robin_schedule,
    svd,
    svd_tensor,
)
from .qr import QrResult, batch_qr, qr, qr_tensor
from .rsvd import RsvdOptions, TruncatedSvd, batch_rsvd, gaussian_matrix, gaussian_tensor, rsvd, rsvd_tensor
from .testmat import make_matrix_tensor

__version__ = "0.1.0"

__all__ = [
    "BackendUnavailable",
    "BatchError",
    "BlockJacobiOptions",
    "BlockSvdResult",
    "JacobiOptions",
    "PairSchedule",
    "QrResult",
    "RsvdOptions",
    "SvdResult",
    "TruncatedSvd",
    "as_matrix",
    "batch_apply",
    "frobenius",
    "gemm",
    "householder_vector",
    "jacobi_rotation",
    "off_orthogonality",
    "read_matrix_text",
    "scaled_offdiag",
    "syrk",
    "write_matrix_text",
    "batch_block_svd",
    "batch_qr",
    "batch_rsvd",
    "batch_svd",
    "block_svd",
    "block_svd_tensor",
    "gaussian_matrix",
    "gaussian_tensor",
    "make_matrix_tensor",
    "qr",
    "qr_tensor",
    "round_robin_schedule",
    "rsvd",
    "rsvd_tensor",
    "svd",
    "svd_tensor",
]
