"""Thin host wrappers around the C ABI: tensor lists and launches.

A ``TensorList`` is the host-memory ``of_tensor_list`` for one fixed set of
parameters (a layer, a bucket, or the whole model); its ctypes pointer arrays
are allocated once and only the device pointers are rewritten per launch, so
issuing a multi-tensor update from a hook costs one ctypes call.
"""

from __future__ import annotations

import ctypes

import torch

from . import _native as nat
from .errors import ConfigError

_DTYPE_CODES = {torch.float32: nat.OF_F32, torch.float64: nat.OF_F64,
                torch.bfloat16: nat.OF_BF16}


def dtype_code(dt: torch.dtype) -> int:
    try:
        return _DTYPE_CODES[dt]
    except KeyError:
        raise ConfigError(f"dtype {dt} is not supported by the update kernels "
                          "(float32, float64; bfloat16 gradients into float32 params)")


class TensorList:
    """Cached ``of_tensor_list`` with room for ``n`` tensors."""

    __slots__ = ("n", "param", "grad", "state0", "state1", "shadow", "numel", "struct", "ref")

    def __init__(self, n: int):
        self.n = n
        self.param = (ctypes.c_void_p * max(n, 1))()
        self.grad = (ctypes.c_void_p * max(n, 1))()
        self.state0 = (ctypes.c_void_p * max(n, 1))()
        self.state1 = (ctypes.c_void_p * max(n, 1))()
        self.shadow = (ctypes.c_void_p * max(n, 1))()
        self.numel = (ctypes.c_int64 * max(n, 1))()
        pp = nat._PP
        self.struct = nat.OfTensorList(
            n, nat.OF_F32, nat.OF_F32, 0,
            ctypes.cast(self.param, pp), ctypes.cast(self.grad, pp),
            ctypes.cast(self.state0, pp), ctypes.cast(self.state1, pp),
            ctypes.cast(self.shadow, pp), ctypes.cast(self.numel, ctypes.POINTER(ctypes.c_int64)))
        self.ref = ctypes.byref(self.struct)

    def set_dtypes(self, param_dtype: torch.dtype, grad_dtype: torch.dtype) -> None:
        self.struct.param_dtype = dtype_code(param_dtype)
        self.struct.grad_dtype = dtype_code(grad_dtype)

    def set(self, i: int, param, grad, state0=None, state1=None, shadow=None) -> None:
        self.param[i] = param.data_ptr() if param is not None else None
        self.grad[i] = grad.data_ptr()
        self.state0[i] = state0.data_ptr() if state0 is not None else None
        self.state1[i] = state1.data_ptr() if state1 is not None else None
        self.shadow[i] = shadow.data_ptr() if shadow is not None else None
        self.numel[i] = grad.numel()


def hparams(kind: str, eta: float, alpha: float, weight_decay: float, epsilon: float,
            beta1: float, beta2: float, rho: float, t: int, max_ctas: int = 0,
            device_step=None) -> nat.OfHparams:
    """of_hparams for step index t; bias corrections in double (optim.py:145-146).
    ``device_step`` (a DeviceStep): fill the OF_FLAG_DEVICE_STEP fields, with
    t as the base index the device offset is added to."""
    bc1 = bc2 = 1.0
    if kind in ("adam", "adamw"):
        bc1 = 1 - beta1 ** t
        bc2 = 1 - beta2 ** t
    hp = nat.OfHparams(nat.KIND_CODES[kind], max_ctas, eta, alpha, weight_decay, epsilon,
                       beta1, beta2, rho, bc1, bc2)
    if device_step is not None:
        hp.step_offset_dev = device_step.offset.data_ptr()
        hp.step_table_dev = device_step.table.data_ptr()
        hp.step_table_rows = device_step.table.shape[0]
        hp.t_base = t
    return hp


def step_advance(offset: torch.Tensor, delta: int = 1, stream=None) -> None:
    """of_step_advance: offset += delta on the device (stream-ordered)."""
    st = nat.lib().of_step_advance(offset.data_ptr(), int(delta), _handle(stream))
    nat.check(st, "of_step_advance")


def policy_step(tl: TensorList, hp: nat.OfHparams, grad_scale, flags: int, stream) -> None:
    """of_policy_step_mt on ``stream`` (a torch.cuda.Stream or raw handle).
    ``grad_scale``: None or a 0-dim f32 / f64 device tensor (f64: the flag
    OF_FLAG_SCALE_F64 is added)."""
    gs = None
    if grad_scale is not None:
        gs = grad_scale.data_ptr()
        if grad_scale.dtype == torch.float64:
            flags |= nat.OF_FLAG_SCALE_F64
    st = nat.lib().of_policy_step_mt(tl.ref, ctypes.byref(hp), gs, flags, _handle(stream))
    if st:
        nat.check(st, "of_policy_step_mt")


class PeerBucket:
    """Host ``of_peer_bucket`` of one data-parallel bucket (pointers fixed at
    construction: the symmetric buffers never move)."""

    __slots__ = ("grads", "params", "struct", "ref")

    def __init__(self, world: int, rank: int, param_dtype, grad_dtype, peer_grad_ptrs,
                 peer_param_ptrs, master, state0, state1, shard_begin: int, shard_len: int):
        self.grads = (ctypes.c_void_p * world)(*peer_grad_ptrs)
        self.params = (ctypes.c_void_p * world)(*peer_param_ptrs)
        pp = nat._PP

        def ptr(t):
            return t.data_ptr() if t is not None else None
        self.struct = nat.OfPeerBucket(world, rank, dtype_code(param_dtype), dtype_code(grad_dtype),
                                       ctypes.cast(self.grads, pp), ctypes.cast(self.params, pp),
                                       ptr(master), ptr(state0), ptr(state1), shard_begin, shard_len)
        self.ref = ctypes.byref(self.struct)


def dp_step_peer(pb: PeerBucket, hp: nat.OfHparams, grad_scale, flags: int, stream) -> None:
    """of_dp_step_peer: reduce-scatter + update + all-gather of one bucket in one kernel."""
    gs = grad_scale.data_ptr() if grad_scale is not None else None
    st = nat.lib().of_dp_step_peer(pb.ref, ctypes.byref(hp), gs, flags, _handle(stream))
    if st:
        nat.check(st, "of_dp_step_peer")


def dp_sqnorm_peer(pb: PeerBucket, workspace: torch.Tensor, out: torch.Tensor, accumulate: bool,
                   stream) -> None:
    """of_dp_sqnorm_peer: Σ over this rank's shard of the peer-summed gradient squared (f64)."""
    st = nat.lib().of_dp_sqnorm_peer(pb.ref, workspace.data_ptr(), workspace.numel(), out.data_ptr(),
                                     int(accumulate), _handle(stream))
    if st:
        nat.check(st, "of_dp_sqnorm_peer")


class McBucket:
    """Host ``of_mc_bucket`` of one data-parallel bucket over NVLS multicast
    (multicast addresses of the flat gradient/parameter buffers, fixed)."""

    __slots__ = ("struct", "ref")

    def __init__(self, world: int, rank: int, mc_grad_ptr: int, mc_param_ptr: int, local_param,
                 state0, state1, shard_begin: int, shard_len: int, dtype=torch.float32):
        def ptr(t):
            return t.data_ptr() if t is not None else None
        code = dtype_code(dtype)
        self.struct = nat.OfMcBucket(world, rank, code, code, mc_grad_ptr, mc_param_ptr, ptr(local_param),
                                     ptr(state0), ptr(state1), shard_begin, shard_len)
        self.ref = ctypes.byref(self.struct)


def dp_step_multicast(mb: McBucket, hp: nat.OfHparams, grad_scale, flags: int, stream) -> None:
    """of_dp_step_multicast: the bucket step with an in-switch reduced gradient
    load and multicast parameter/gradient stores (fp32)."""
    gs = grad_scale.data_ptr() if grad_scale is not None else None
    st = nat.lib().of_dp_step_multicast(mb.ref, ctypes.byref(hp), gs, flags, _handle(stream))
    if st:
        nat.check(st, "of_dp_step_multicast")


def wgrad_step(grad_out, inp, param, state0, state1, hp: nat.OfHparams, *, shadow=None,
               flags: int = 0, stream=None, grad_dump=None) -> None:
    """of_wgrad_step: dW = grad_out^T @ inp (bf16 [T, M] and [T, N]) on the tensor
    cores with the optimizer update applied from the accumulator to the fp32
    ``param`` [M, N] and its history (and the bf16 ``shadow``); the gradient
    is not materialised unless ``grad_dump`` (fp32 [M, N]) is given."""
    T, M = grad_out.shape
    N = inp.shape[1]
    if inp.shape[0] != T or tuple(param.shape) != (M, N):
        raise ConfigError(f"wgrad: shapes {tuple(grad_out.shape)}, {tuple(inp.shape)}, "
                          f"{tuple(param.shape)} do not form dW = dY^T X")
    for t, dt in ((grad_out, torch.bfloat16), (inp, torch.bfloat16), (param, torch.float32)):
        if t.dtype != dt or not t.is_contiguous():
            raise ConfigError(f"wgrad: expected contiguous {dt}, got {t.dtype}")

    def ptr(t):
        return t.data_ptr() if t is not None else None
    if shadow is not None:
        flags |= nat.OF_FLAG_SHADOW_BF16
    args = nat.OfWgradArgs(M, N, T, grad_out.data_ptr(), inp.data_ptr(), param.data_ptr(),
                           ptr(state0), ptr(state1), ptr(shadow), ptr(grad_dump))
    st = nat.lib().of_wgrad_step(ctypes.byref(args), ctypes.byref(hp), flags, _handle(stream))
    if st:
        nat.check(st, "of_wgrad_step")


class CopyList:
    """Fixed (dst, src) tensor pairs for ``of_copy_mt`` (pointers captured once)."""

    __slots__ = ("n", "dst", "src", "nbytes", "keep")

    def __init__(self, dsts, srcs, checked: bool = False):
        if len(dsts) != len(srcs):
            raise ConfigError("copy list: dst and src lengths differ")
        self.n = len(dsts)
        self.dst = (ctypes.c_void_p * max(self.n, 1))(*[d.data_ptr() for d in dsts])
        self.src = (ctypes.c_void_p * max(self.n, 1))(*[s.data_ptr() for s in srcs])
        self.nbytes = (ctypes.c_int64 * max(self.n, 1))(*[d.numel() * d.element_size() for d in dsts])
        if not checked:
            for d, s in zip(dsts, srcs):
                if not same_layout(d, s):
                    raise ConfigError("copy list: a pair differs in size or layout")
        self.keep = (list(dsts), list(srcs))


def same_layout(a, b) -> bool:
    """Same dtype, shape and element order in memory (strides of size-1
    dimensions are arbitrary), both dense: a byte copy moves a into b."""
    if a.dtype != b.dtype or a.shape != b.shape:
        return False
    if any(sa != sb for n, sa, sb in zip(a.shape, a.stride(), b.stride()) if n > 1):
        return False
    return is_dense(a) and is_dense(b)


def is_dense(t) -> bool:
    """Non-overlapping and dense: the dimensions of size > 1, ordered by
    stride, tile [0, numel) exactly (contiguous, channels-last, any permutation)."""
    dims = sorted((st, n) for n, st in zip(t.shape, t.stride()) if n > 1)
    expect = 1
    for st, n in dims:
        if st != expect:
            return False
        expect *= n
    return True


def copy_mt(cl: CopyList, stream=None) -> None:
    st = nat.lib().of_copy_mt(ctypes.cast(cl.dst, nat._PP), ctypes.cast(cl.src, nat._PP),
                              cl.nbytes, cl.n, _handle(stream))
    nat.check(st, "of_copy_mt")


def sqnorm(tl: TensorList, workspace: torch.Tensor, out: torch.Tensor, accumulate: bool,
           stream) -> None:
    st = nat.lib().of_sqnorm_mt(tl.ref, workspace.data_ptr(), workspace.numel(), out.data_ptr(),
                                int(accumulate), _handle(stream))
    nat.check(st, "of_sqnorm_mt")


def clip_coef(sq: torch.Tensor, max_norm: float, coef: torch.Tensor, factor: torch.Tensor,
              stream) -> None:
    st = nat.lib().of_clip_coef(sq.data_ptr(), float(max_norm), coef.data_ptr(),
                                factor.data_ptr(), _handle(stream))
    nat.check(st, "of_clip_coef")


def sqnorm_workspace_len() -> int:
    return int(nat.lib().of_sqnorm_workspace_len())


def _handle(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream
