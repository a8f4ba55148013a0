"""The C-ABI library loads and exports every symbol include/optfuse_b200.h
declares; argument validation rejects bad calls before anything is launched
(no GPU needed: nothing here reaches the CUDA runtime)."""

import ctypes

import torch
import re
from pathlib import Path

import pytest

from paper_2104_00237_b200 import _native as nat
from paper_2104_00237_b200 import kernels

HEADER = Path(__file__).resolve().parent.parent / "include" / "optfuse_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|uint64_t|const char\*)\s+(of_\w+)\(",
                                 text, re.M)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(nat.SYMBOLS)


def test_library_exports_every_symbol():
    so = nat.lib()
    for name in declared_symbols():
        assert hasattr(so, name), name
    assert so.of_abi_version() == nat.ABI_VERSION == 4
    assert so.of_status_string(0) == b"ok"
    assert so.of_sqnorm_workspace_len() >= 148


def test_library_is_sm100a_only():
    data = nat.LIB_PATH.read_bytes()
    assert b"sm_100a" in data


def _hp(kind=1, eta=0.1):
    return nat.OfHparams(kind, 0, eta, 0.9, 0.0, 1e-8, 0.9, 0.999, 0.9, 1.0, 1.0)


def test_invalid_arguments_rejected_before_launch():
    so = nat.lib()
    before = so.of_launch_count()
    hp = _hp()
    assert so.of_policy_step_mt(None, ctypes.byref(hp), None, 0, None) == nat.OF_ERR_INVALID
    assert b"NULL" in so.of_last_error()
    tl = kernels.TensorList(1)
    tl.param[0] = 0x1000
    tl.grad[0] = None
    tl.state0[0] = 0x2000
    tl.numel[0] = 7
    assert so.of_policy_step_mt(tl.ref, ctypes.byref(hp), None, 0, None) == nat.OF_ERR_INVALID
    assert b"grad" in so.of_last_error()
    bad = _hp(kind=42)
    assert so.of_policy_step_mt(tl.ref, ctypes.byref(bad), None, 0, None) == nat.OF_ERR_INVALID
    neg = _hp(eta=-1.0)
    assert so.of_policy_step_mt(tl.ref, ctypes.byref(neg), None, 0, None) == nat.OF_ERR_INVALID
    assert so.of_policy_step_mt(tl.ref, ctypes.byref(hp), None, 0x80, None) == nat.OF_ERR_INVALID
    # ABI 3: an f64 grad scale needs the scale pointer
    assert so.of_policy_step_mt(tl.ref, ctypes.byref(hp), None, nat.OF_FLAG_SCALE_F64,
                                None) == nat.OF_ERR_INVALID
    assert b"SCALE_F64" in so.of_last_error()
    tl.struct.param_dtype = nat.OF_BF16
    tl.grad[0] = 0x3000
    assert so.of_policy_step_mt(tl.ref, ctypes.byref(hp), None, 0, None) == nat.OF_ERR_UNSUPPORTED
    adam = nat.OfHparams(5, 0, 1e-3, 0.9, 0.0, 1e-8, 0.9, 0.999, 0.9, 0.0, 0.0)
    tl.struct.param_dtype = nat.OF_F32
    tl.state1[0] = 0x4000
    assert so.of_policy_step_mt(tl.ref, ctypes.byref(adam), None, 0, None) == nat.OF_ERR_INVALID
    assert b"bias" in so.of_last_error()
    # OF_FLAG_DEVICE_STEP needs the device offset and table (and ignores the
    # host bias corrections, which are zero here)
    dev = nat.OF_FLAG_DEVICE_STEP
    assert so.of_policy_step_mt(tl.ref, ctypes.byref(adam), None, dev, None) == nat.OF_ERR_INVALID
    assert b"DEVICE_STEP" in so.of_last_error()
    adam.step_offset_dev, adam.step_table_dev, adam.step_table_rows = 0x5000, 0x6000, 1
    assert so.of_policy_step_mt(tl.ref, ctypes.byref(adam), None, dev, None) == nat.OF_ERR_INVALID
    assert b"rows" in so.of_last_error()
    assert so.of_step_advance(None, 1, None) == nat.OF_ERR_INVALID
    # the data-parallel peer step validates world/rank/shard/pointers first
    pb = kernels.PeerBucket(2, 0, torch.float32, torch.float32, [0x1000, 0x2000], [0x3000, 0x4000],
                            None, None, None, 0, 8)
    sgdm = _hp()
    assert so.of_dp_step_peer(pb.ref, ctypes.byref(sgdm), None, 0, None) == nat.OF_ERR_INVALID
    assert b"state0" in so.of_last_error()
    pb.struct.state0 = 0x5000
    pb.struct.rank = 2
    assert so.of_dp_step_peer(pb.ref, ctypes.byref(sgdm), None, 0, None) == nat.OF_ERR_INVALID
    pb.struct.rank = 0
    pb.struct.shard_len = 6
    assert so.of_dp_step_peer(pb.ref, ctypes.byref(sgdm), None, 0, None) == nat.OF_ERR_INVALID
    pb.struct.shard_len = 8
    pb.struct.world = nat.OF_MAX_PEERS + 1
    assert so.of_dp_step_peer(pb.ref, ctypes.byref(sgdm), None, 0, None) == nat.OF_ERR_INVALID
    pb.struct.world = 2
    pb.struct.param_dtype = nat.OF_BF16      # bf16 params need bf16 grads and a master
    assert so.of_dp_step_peer(pb.ref, ctypes.byref(sgdm), None, 0, None) == nat.OF_ERR_INVALID
    assert so.of_dp_step_peer(pb.ref, ctypes.byref(sgdm), None, nat.OF_FLAG_ZERO_GRAD,
                              None) == nat.OF_ERR_INVALID
    # ABI 4: the peer transport's clip reduction validates the same fields first
    ws = 0x7000
    assert so.of_dp_sqnorm_peer(None, ws, 16, 0x8000, 0, None) == nat.OF_ERR_INVALID
    assert so.of_dp_sqnorm_peer(pb.ref, None, 0, 0x8000, 0, None) == nat.OF_ERR_INVALID
    assert b"workspace" in so.of_last_error()
    assert so.of_dp_sqnorm_peer(pb.ref, ws, 16, None, 0, None) == nat.OF_ERR_INVALID
    pb.struct.rank = 5
    assert so.of_dp_sqnorm_peer(pb.ref, ws, 16, 0x8000, 0, None) == nat.OF_ERR_INVALID
    pb.struct.rank = 0
    pb.struct.shard_begin = 2
    assert so.of_dp_sqnorm_peer(pb.ref, ws, 16, 0x8000, 0, None) == nat.OF_ERR_INVALID
    assert b"multiples of 4" in so.of_last_error()
    pb.struct.shard_begin = 0
    # the (experimental) multicast step is fp32 only (ABI 3 dtype fields)
    mb = kernels.McBucket(1, 0, 0x1000, 0x2000, None, None, None, 0, 8, dtype=torch.bfloat16)
    mb.struct.local_param = 0x3000
    mb.struct.state0 = 0x4000
    assert so.of_dp_step_multicast(mb.ref, ctypes.byref(sgdm), None, 0, None) == nat.OF_ERR_UNSUPPORTED
    assert b"fp32" in so.of_last_error()
    assert so.of_copy_mt(None, None, None, 3, None) == nat.OF_ERR_INVALID
    nb = (ctypes.c_int64 * 1)(-4)
    one = (ctypes.c_void_p * 1)(0x10)
    assert so.of_copy_mt(ctypes.cast(one, nat._PP), ctypes.cast(one, nat._PP), nb, 1,
                         None) == nat.OF_ERR_INVALID
    assert so.of_copy_mt(None, None, None, 0, None) == nat.OF_OK
    assert so.of_exact_matmul(None, 0x10, 0x20, 2, 2, 2, nat.OF_F32, None) == nat.OF_ERR_INVALID
    assert so.of_exact_matmul(0x10, 0x10, 0x20, 70000, 2, 2, nat.OF_F32, None) == nat.OF_ERR_INVALID
    assert so.of_exact_matmul(0x10, 0x10, 0x20, 2, 2, 2, nat.OF_BF16, None) == nat.OF_ERR_UNSUPPORTED
    empty = kernels.TensorList(0)
    assert so.of_policy_step_mt(empty.ref, ctypes.byref(hp), None, 0, None) == nat.OF_OK
    assert so.of_clip_coef(None, 1.0, None, None, None) == nat.OF_ERR_INVALID
    assert so.of_sqnorm_mt(empty.ref, None, 0, None, 0, None) == nat.OF_ERR_INVALID
    assert so.of_launch_count() == before, "a rejected call must not launch"


def test_check_raises_native_error():
    from paper_2104_00237_b200.errors import NativeLibraryError
    so = nat.lib()
    so.of_policy_step_mt(None, None, None, 0, None)
    with pytest.raises(NativeLibraryError, match="invalid"):
        nat.check(nat.OF_ERR_INVALID, "of_policy_step_mt")


def test_no_host_function_compiled_to_an_exit_stub():
    """nvcc compiles a host function template that calls a __device__-only
    helper into `exit(1)` without an error; such a launcher would kill the
    process silently on its first call.  Every host function of the library's
    own code must therefore be free of calls to exit()."""
    import shutil
    import subprocess
    if shutil.which("objdump") is None:
        pytest.skip("objdump not installed")
    out = subprocess.run(["objdump", "-d", "--no-show-raw-insn", "-C", str(nat.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    stubs, fn = [], None
    for line in out.splitlines():
        m = re.match(r"^[0-9a-f]+ <(.*)>:$", line)
        if m:
            fn = m.group(1)
        elif fn and "exit@plt" in line and ("ofk::" in fn or "anonymous namespace" in fn
                                             or fn.startswith("of_")):
            stubs.append(fn)
    assert not stubs, stubs[:5]
