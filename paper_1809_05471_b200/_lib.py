"""ctypes binding of libigs_b200.so (the C-ABI declared in include/igs_capi.h).

This is the binding a maintainer of the reference package would add
(INTEGRATION.md): plain ctypes structs mirroring igs_dir / igs_problem,
status codes mapped onto the reference's exception classes (errors.py:4-17).
There is no CPU fallback: a missing library or a missing GPU raises.
"""

import ctypes
import os

from .errors import CapacityError, DomainError, UnsupportedDerivativeError

_PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# IGS_LIB_PATH: development A/B timing of two builds (tools/ab_time.sh)
LIB_PATH = os.environ.get("IGS_LIB_PATH") or os.path.join(_PKG_DIR, "libigs_b200.so")

MAX_DIM = 3
MAX_DERIV_SET = 8
MAX_ORDER = 16

OP_ASSEMBLE, OP_APPLY, OP_EVAL_FIELD, OP_PATTERN = 1, 2, 3, 4
FLAG_DEFAULT, FLAG_FORCE_GENERIC, FLAG_ACCUMULATE = 0, 1, 2
FLAG_KERNEL_ONLY, FLAG_TWO_PASS, FLAG_SPLIT_BOUNDARY, FLAG_THREE_PASS = 4, 8, 16, 32

IGS_OK, IGS_EARG, IGS_EDOMAIN, IGS_EDERIV, IGS_ECAPACITY, IGS_ECUDA, IGS_ENCCL, IGS_EWORKSPACE = range(8)

_c_double_p = ctypes.c_void_p
_c_int64_p = ctypes.c_void_p


class IgsDir(ctypes.Structure):
    _fields_ = [
        ("order", ctypes.c_int32),
        ("num_basis", ctypes.c_int32),
        ("num_points", ctypes.c_int32),
        ("max_deriv", ctypes.c_int32),
        ("values", ctypes.c_void_p),
        ("first_active", ctypes.c_void_p),
        ("weights", ctypes.c_void_p),
        ("csupp_lo", ctypes.c_void_p),
        ("csupp_hi", ctypes.c_void_p),
        ("points", ctypes.c_void_p),
        ("num_elements", ctypes.c_int32),
        ("points_per_element", ctypes.c_int32),
        ("uniform", ctypes.c_int32),
    ]


class IgsProblem(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32),
        ("trial", IgsDir * MAX_DIM),
        ("test", IgsDir * MAX_DIM),
        ("n_theta", ctypes.c_int32),
        ("n_eta", ctypes.c_int32),
        ("theta", (ctypes.c_int8 * MAX_DIM) * MAX_DERIV_SET),
        ("eta", (ctypes.c_int8 * MAX_DIM) * MAX_DERIV_SET),
        ("plane_of", (ctypes.c_int8 * MAX_DERIV_SET) * MAX_DERIV_SET),
        ("n_planes", ctypes.c_int32),
        ("plane_stride", ctypes.c_int64),
        ("dir_order", ctypes.c_int32 * MAX_DIM),
        ("num_pairs", ctypes.c_int64 * MAX_DIM),
        ("slab_lo", ctypes.c_int32),
        ("slab_hi", ctypes.c_int32),
    ]


class IgsPullbackArgs(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32),
        ("npts", ctypes.c_int64),
        ("val", ctypes.c_void_p * MAX_DIM),
        ("grad", (ctypes.c_void_p * MAX_DIM) * MAX_DIM),
        ("wval", ctypes.c_void_p),
        ("wgrad", ctypes.c_void_p * MAX_DIM),
        ("reaction", ctypes.c_void_p),
        ("reaction_stride", ctypes.c_int64),
        ("convection", ctypes.c_void_p * MAX_DIM),
        ("convection_stride", ctypes.c_int64),
        ("diffusion", (ctypes.c_void_p * MAX_DIM) * MAX_DIM),
        ("diffusion_stride", ctypes.c_int64),
        ("rtol", ctypes.c_double),
    ]


class IgsGeometryMap(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32),
        ("order", ctypes.c_int32 * MAX_DIM),
        ("num_basis", ctypes.c_int32 * MAX_DIM),
        ("num_points", ctypes.c_int64 * MAX_DIM),
        ("values", ctypes.c_void_p * MAX_DIM),
        ("first_active", ctypes.c_void_p * MAX_DIM),
        ("control", ctypes.c_void_p),
        ("weights", ctypes.c_void_p),
    ]


# (name, restype, argtypes) for every symbol declared in include/igs_capi.h.
_SIGNATURES = [
    ("igs_last_error", ctypes.c_char_p, []),
    ("igs_status_string", ctypes.c_char_p, [ctypes.c_int]),
    ("igs_abi_version", ctypes.c_int32, []),
    ("igs_fused_path", ctypes.c_int32, [ctypes.POINTER(IgsProblem), ctypes.c_int32]),
    ("igs_gauss_rule", ctypes.c_int,
     [ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    ("igs_tabulate", ctypes.c_int,
     [ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    ("igs_pattern_1d", ctypes.c_int,
     [ctypes.POINTER(IgsProblem), ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
      ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p]),
    ("igs_pattern", ctypes.c_int,
     [ctypes.POINTER(IgsProblem), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
      ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]),
    ("igs_workspace_bytes", ctypes.c_size_t, [ctypes.POINTER(IgsProblem), ctypes.c_int32, ctypes.c_int32]),
    ("igs_assemble_values", ctypes.c_int,
     [ctypes.POINTER(IgsProblem), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
      ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
      ctypes.c_size_t, ctypes.c_int32, ctypes.c_void_p]),
    ("igs_apply", ctypes.c_int,
     [ctypes.POINTER(IgsProblem), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
      ctypes.c_size_t, ctypes.c_int32, ctypes.c_void_p]),
    ("igs_eval_field", ctypes.c_int,
     [ctypes.POINTER(IgsProblem), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
      ctypes.c_size_t, ctypes.c_void_p]),
    ("igs_fill_synthetic", ctypes.c_int,
     [ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64,
      ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]),
    ("igs_layers_copy", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p]),
    ("igs_write_matrix_market", ctypes.c_int,
     [ctypes.c_char_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    ("igs_assemble_naive", ctypes.c_int,
     [ctypes.POINTER(IgsProblem), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
      ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
      ctypes.c_void_p]),
    ("igs_geometry_planes", ctypes.c_int,
     [ctypes.POINTER(IgsGeometryMap), ctypes.POINTER(IgsPullbackArgs), ctypes.c_void_p, ctypes.c_int32,
      ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
      ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    ("igs_geometry_pullback", ctypes.c_int,
     [ctypes.POINTER(IgsPullbackArgs), ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64,
      ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p, ctypes.c_size_t,
      ctypes.c_void_p]),
    ("igs_nccl_unique_id", ctypes.c_int, [ctypes.c_void_p]),
    ("igs_nccl_comm_init", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]),
    ("igs_nccl_comm_destroy", ctypes.c_int, [ctypes.c_void_p]),
    ("igs_nccl_check", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32]),
    ("igs_apply_sharded_workspace", ctypes.c_size_t,
     [ctypes.POINTER(IgsProblem), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    ("igs_apply_sharded", ctypes.c_int,
     [ctypes.POINTER(IgsProblem), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
      ctypes.c_size_t, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
      ctypes.c_void_p]),
]

EXPORTED = tuple(name for name, _, _ in _SIGNATURES)

_LIB = None


def load():
    """Load (once) and return the library.  Raises if it was never built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1809_05471_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in _SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(status, what=""):
    """Raise the reference-equivalent exception for a non-zero status."""
    if status == IGS_OK:
        return
    lib = load()
    msg = lib.igs_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == IGS_EDOMAIN:
        raise DomainError(text)
    if status == IGS_EDERIV:
        raise UnsupportedDerivativeError(text)
    if status == IGS_ECAPACITY:
        raise CapacityError(text)
    if status in (IGS_EARG, IGS_EWORKSPACE):
        raise ValueError(text)
    raise RuntimeError(text)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_1809_05471_b200 computes on a CUDA device; none is available")
    load()
    return torch


def stream_handle():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())
