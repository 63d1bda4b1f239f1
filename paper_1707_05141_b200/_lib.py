"""ctypes binding of the in-tree C-ABI library ``libbatchfact_b200.so`` (include/batchfact_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is visible,
every compute entry point raises :class:`BackendUnavailable`.
"""

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
# BATCHFACT_B200_LIB overrides the library path (kernel experiments only)
LIB_PATH = os.environ.get("BATCHFACT_B200_LIB") or os.path.join(HERE, "libbatchfact_b200.so")
CSRC = os.path.join(HERE, "csrc")


class BackendUnavailable(RuntimeError):
    """The sm_100a library (or a CUDA device) is not available."""


class _Opts(ctypes.Structure):
    _fields_ = [
        ("tolerance", ctypes.c_double),
        ("max_sweeps", ctypes.c_int32),
        ("ordering", ctypes.c_int32),
        ("accumulate_v", ctypes.c_int32),
        ("tier", ctypes.c_int32),
    ]


class _BlockOpts(ctypes.Structure):
    _fields_ = [
        ("tolerance", ctypes.c_double),
        ("block_width", ctypes.c_int32),
        ("method", ctypes.c_int32),
        ("max_sweeps", ctypes.c_int32),
        ("accumulate_v", ctypes.c_int32),
    ]


JacobiOptsC = _Opts
BlockOptsC = _BlockOpts

BF_OK = 0
BF_ERR_ARG = -1
BF_ERR_WORKSPACE = -2
BF_ERR_UNSUPPORTED = -3

# every symbol include/batchfact_b200.h declares
EXPORTS = (
    "bf_gemm_batched_f64",
    "bf_gemm_batched_f32",
    "bf_last_error",
    "bf_version",
    "bf_qr_workspace_size",
    "bf_qr_batched_f64",
    "bf_qr_batched_f32",
    "bf_svd_workspace_size",
    "bf_svd_batched_f64",
    "bf_svd_batched_f32",
    "bf_block_svd_workspace_size",
    "bf_block_svd_batched_f64",
    "bf_block_svd_batched_f32",
    "bf_block_svd_batched_ex_f64",
    "bf_block_svd_batched_ex_f32",
    "bf_rsvd_workspace_size",
    "bf_rsvd_batched_f64",
    "bf_rsvd_batched_f32",
    "bf_gaussian_batched_f64",
    "bf_gaussian_batched_f32",
    "bf_householder_batched_f64",
    "bf_householder_batched_f32",
    "bf_jacobi_rotation_batched_f64",
    "bf_off_orthogonality_batched_f64",
    "bf_off_orthogonality_batched_f32",
    "bf_scaled_offdiag_batched_f64",
    "bf_scaled_offdiag_batched_f32",
    "bf_syrk_batched_f64",
    "bf_syrk_batched_f32",
    "bf_frobenius_batched_f64",
    "bf_frobenius_batched_f32",
    "bf_axpby_f64",
    "bf_axpby_f32",
    "bf_make_matrix_workspace_size",
    "bf_make_matrix_batched_f64",
)

_lib = None


def build(force=False, jobs=8):
    """Compile the CUDA library in-tree for sm_100a (nvcc; no GPU needed)."""
    args = ["make", "-s", "-C", CSRC, f"-j{jobs}"]
    if force:
        subprocess.run(["make", "-s", "-C", CSRC, "clean"], check=True)
    subprocess.run(args, check=True)


def load():
    """Load (once) and type the library. Raises BackendUnavailable if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise BackendUnavailable(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U64, D, SZ = (
        ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_size_t,
    )
    L.bf_last_error.restype = ctypes.c_char_p
    L.bf_version.restype = ctypes.c_char_p
    L.bf_qr_workspace_size.argtypes = [I64, I32, I32, I32]
    L.bf_qr_workspace_size.restype = SZ
    for name in ("bf_qr_batched_f64", "bf_qr_batched_f32"):
        f = getattr(L, name)
        f.argtypes = [I64, I32, I32, P, P, P, I32, P, SZ, P]
        f.restype = ctypes.c_int
    L.bf_svd_workspace_size.argtypes = [I64, I32, I32, I32, ctypes.POINTER(_Opts)]
    L.bf_svd_workspace_size.restype = SZ
    for name in ("bf_svd_batched_f64", "bf_svd_batched_f32"):
        f = getattr(L, name)
        f.argtypes = [I64, I32, I32, P, P, P, P, P, P, P, ctypes.POINTER(_Opts), P, SZ, P]
        f.restype = ctypes.c_int
    L.bf_block_svd_workspace_size.argtypes = [I64, I32, I32, I32, ctypes.POINTER(_BlockOpts)]
    L.bf_block_svd_workspace_size.restype = SZ
    for name in ("bf_block_svd_batched_f64", "bf_block_svd_batched_f32"):
        f = getattr(L, name)
        f.argtypes = [I64, I32, I32, P, P, P, P, P, P, P, ctypes.POINTER(_BlockOpts), P, SZ, P]
        f.restype = ctypes.c_int
    for name in ("bf_block_svd_batched_ex_f64", "bf_block_svd_batched_ex_f32"):
        f = getattr(L, name)
        f.argtypes = [I64, I32, I32, P, P, P, P, P, P, P, P, ctypes.POINTER(_BlockOpts), P, SZ, P]
        f.restype = ctypes.c_int
    L.bf_rsvd_workspace_size.argtypes = [I64, I32, I32, I32, I32, I32]
    L.bf_rsvd_workspace_size.restype = SZ
    for name in ("bf_rsvd_batched_f64", "bf_rsvd_batched_f32"):
        f = getattr(L, name)
        f.argtypes = [I64, I32, I32, I32, I32, U64, U64, I64, P, P, P, P, P, P, SZ, P]
        f.restype = ctypes.c_int
    for name in ("bf_gaussian_batched_f64", "bf_gaussian_batched_f32"):
        f = getattr(L, name)
        f.argtypes = [I64, I32, I32, U64, U64, I64, I32, P, P]
        f.restype = ctypes.c_int
    L.bf_make_matrix_workspace_size.argtypes = [I64, I32, I32]
    L.bf_make_matrix_workspace_size.restype = SZ
    L.bf_make_matrix_batched_f64.argtypes = [I64, I32, I32, I32, D, I32, U64, U64, I64, P, P, P, SZ, P]
    L.bf_make_matrix_batched_f64.restype = ctypes.c_int
    for name in ("bf_gemm_batched_f64", "bf_gemm_batched_f32"):
        f = getattr(L, name)
        f.argtypes = [I64, I32, I32, I32, P, I32, I64, I32, P, I32, I64, I32, P, I32, I64, P]
        f.restype = ctypes.c_int
    F = ctypes.c_float
    for suf, R in (("f64", D), ("f32", F)):
        getattr(L, f"bf_householder_batched_{suf}").argtypes = [I64, I32, P, P, P, P]
        getattr(L, f"bf_off_orthogonality_batched_{suf}").argtypes = [I64, I32, I32, P, P, P]
        getattr(L, f"bf_scaled_offdiag_batched_{suf}").argtypes = [I64, I32, P, P, P]
        getattr(L, f"bf_syrk_batched_{suf}").argtypes = [I64, I32, I32, P, P, P]
        getattr(L, f"bf_frobenius_batched_{suf}").argtypes = [I64, I32, I32, P, P, P]
        getattr(L, f"bf_axpby_{suf}").argtypes = [I64, R, P, R, P, P, P]
        for nm in ("householder_batched", "off_orthogonality_batched", "scaled_offdiag_batched", "syrk_batched",
                   "frobenius_batched", "axpby"):
            getattr(L, f"bf_{nm}_{suf}").restype = ctypes.c_int
    L.bf_jacobi_rotation_batched_f64.argtypes = [I64, P, P, P, P, P, P]
    L.bf_jacobi_rotation_batched_f64.restype = ctypes.c_int
    _lib = L
    return L


def last_error():
    return load().bf_last_error().decode()


def check(rc, what):
    """Map a C-ABI status to the reference's exception types."""
    if rc == BF_OK:
        return
    msg = last_error()
    if rc == BF_ERR_ARG:
        raise ValueError(msg)
    if rc == BF_ERR_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: status {rc}: {msg}")
