"""ctypes binding of the C ABI in include/optfuse_b200.h (liboptfuse_b200.so).

The product path has exactly one implementation: the sm_100a kernels in
``csrc/optfuse_kernels.cu``.  If the shared library is missing this module
raises ``NativeLibraryError`` -- there is no CPU or PyTorch fallback.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import NativeLibraryError

LIB_NAME = "liboptfuse_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

OF_OK, OF_ERR_INVALID, OF_ERR_UNSUPPORTED, OF_ERR_CUDA = 0, 1, 2, 3
OF_F32, OF_F64, OF_BF16 = 0, 1, 2
OF_FLAG_ZERO_GRAD = 0x1
OF_FLAG_SHADOW_BF16 = 0x2
OF_FLAG_DEVICE_STEP = 0x4
OF_FLAG_SCALE_F64 = 0x8
ABI_VERSION = 4

# of_kind (optim.py:22 minus newton, plus adamw)
KIND_CODES = {"sgd": 0, "sgd-momentum": 1, "adagrad": 2, "rmsprop": 3, "adadelta": 4,
              "adam": 5, "adamw": 6}

# every symbol include/optfuse_b200.h declares (checked by tests/test_native_abi.py)
SYMBOLS = ("of_abi_version", "of_status_string", "of_last_error", "of_launch_count",
           "of_policy_step_mt", "of_sgdm_mt", "of_adam_mt", "of_step_advance", "of_dp_step_peer",
           "of_sqnorm_workspace_len", "of_sqnorm_mt", "of_clip_coef", "of_exact_matmul",
           "of_copy_mt", "of_dp_step_multicast", "of_wgrad_step", "of_dp_sqnorm_peer")

_vp = ctypes.c_void_p
_PP = ctypes.POINTER(ctypes.c_void_p)


class OfHparams(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("max_ctas", ctypes.c_int32),
                ("eta", ctypes.c_double), ("alpha", ctypes.c_double),
                ("weight_decay", ctypes.c_double), ("epsilon", ctypes.c_double),
                ("beta1", ctypes.c_double), ("beta2", ctypes.c_double), ("rho", ctypes.c_double),
                ("bias_correction1", ctypes.c_double), ("bias_correction2", ctypes.c_double),
                ("step_offset_dev", _vp), ("step_table_dev", _vp),
                ("step_table_rows", ctypes.c_int64), ("t_base", ctypes.c_int64)]


class OfTensorList(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("param_dtype", ctypes.c_int32),
                ("grad_dtype", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("param", _PP), ("grad", _PP), ("state0", _PP), ("state1", _PP),
                ("shadow", _PP), ("numel", ctypes.POINTER(ctypes.c_int64))]


OF_MAX_PEERS = 16


class OfPeerBucket(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("param_dtype", ctypes.c_int32), ("grad_dtype", ctypes.c_int32),
                ("peer_grad", _PP), ("peer_param", _PP), ("master", _vp),
                ("state0", _vp), ("state1", _vp),
                ("shard_begin", ctypes.c_int64), ("shard_len", ctypes.c_int64)]


class OfMcBucket(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("param_dtype", ctypes.c_int32), ("grad_dtype", ctypes.c_int32),
                ("mc_grad", _vp), ("mc_param", _vp), ("local_param", _vp),
                ("state0", _vp), ("state1", _vp),
                ("shard_begin", ctypes.c_int64), ("shard_len", ctypes.c_int64)]


class OfWgradArgs(ctypes.Structure):
    _fields_ = [("out_features", ctypes.c_int64), ("in_features", ctypes.c_int64),
                ("tokens", ctypes.c_int64), ("grad_out_rows", _vp), ("input", _vp),
                ("param", _vp), ("state0", _vp), ("state1", _vp), ("shadow", _vp),
                ("grad_dump", _vp)]


_lib = None


def lib():
    """Load the kernel library once; raise NativeLibraryError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("OPTFUSE_B200_LIB", LIB_PATH))
    if not path.exists():
        raise NativeLibraryError(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the fused-optimizer path has no CPU fallback)")
    try:
        so = ctypes.CDLL(str(path))
    except OSError as e:
        raise NativeLibraryError(f"cannot load {path}: {e}") from e
    so.of_abi_version.restype = ctypes.c_int
    # version first: a stale library must fail here, not on a missing symbol
    if so.of_abi_version() != ABI_VERSION:
        raise NativeLibraryError(f"{path}: ABI version {so.of_abi_version()} != {ABI_VERSION} "
                                 "(stale build: rerun __graft_entry__.build())")
    so.of_status_string.restype = ctypes.c_char_p
    so.of_status_string.argtypes = [ctypes.c_int]
    so.of_last_error.restype = ctypes.c_char_p
    so.of_launch_count.restype = ctypes.c_uint64
    so.of_policy_step_mt.restype = ctypes.c_int
    so.of_policy_step_mt.argtypes = [ctypes.POINTER(OfTensorList), ctypes.POINTER(OfHparams),
                                     _vp, ctypes.c_uint32, _vp]
    so.of_sgdm_mt.restype = ctypes.c_int
    so.of_sgdm_mt.argtypes = [ctypes.POINTER(OfTensorList), ctypes.c_double, ctypes.c_double,
                              ctypes.c_double, _vp, ctypes.c_uint32, _vp]
    so.of_adam_mt.restype = ctypes.c_int
    so.of_adam_mt.argtypes = [ctypes.POINTER(OfTensorList)] + [ctypes.c_double] * 7 + [
        ctypes.c_int, _vp, ctypes.c_uint32, _vp]
    so.of_step_advance.restype = ctypes.c_int
    so.of_step_advance.argtypes = [_vp, ctypes.c_int64, _vp]
    so.of_dp_step_peer.restype = ctypes.c_int
    so.of_dp_step_peer.argtypes = [ctypes.POINTER(OfPeerBucket), ctypes.POINTER(OfHparams), _vp,
                                   ctypes.c_uint32, _vp]
    so.of_dp_sqnorm_peer.restype = ctypes.c_int
    so.of_dp_sqnorm_peer.argtypes = [ctypes.POINTER(OfPeerBucket), _vp, ctypes.c_int64, _vp,
                                     ctypes.c_int, _vp]
    so.of_dp_step_multicast.restype = ctypes.c_int
    so.of_dp_step_multicast.argtypes = [ctypes.POINTER(OfMcBucket), ctypes.POINTER(OfHparams), _vp,
                                        ctypes.c_uint32, _vp]
    so.of_wgrad_step.restype = ctypes.c_int
    so.of_wgrad_step.argtypes = [ctypes.POINTER(OfWgradArgs), ctypes.POINTER(OfHparams),
                                 ctypes.c_uint32, _vp]
    so.of_copy_mt.restype = ctypes.c_int
    so.of_copy_mt.argtypes = [_PP, _PP, ctypes.POINTER(ctypes.c_int64), ctypes.c_int, _vp]
    so.of_exact_matmul.restype = ctypes.c_int
    so.of_exact_matmul.argtypes = [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_int, _vp]
    so.of_sqnorm_workspace_len.restype = ctypes.c_int64
    so.of_sqnorm_mt.restype = ctypes.c_int
    so.of_sqnorm_mt.argtypes = [ctypes.POINTER(OfTensorList), _vp, ctypes.c_int64, _vp,
                                ctypes.c_int, _vp]
    so.of_clip_coef.restype = ctypes.c_int
    so.of_clip_coef.argtypes = [_vp, ctypes.c_double, _vp, _vp, _vp]
    _lib = so
    return so


def check(status: int, what: str) -> None:
    if status != OF_OK:
        so = lib()
        msg = so.of_last_error().decode(errors="replace")
        raise NativeLibraryError(
            f"{what}: {so.of_status_string(status).decode()} ({msg})")


def launch_count() -> int:
    """Kernels launched by liboptfuse_b200.so in this process."""
    return int(lib().of_launch_count())
