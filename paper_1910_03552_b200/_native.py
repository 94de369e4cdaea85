"""ctypes binding of libbeast_b200.so (the C ABI in include/beast_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every op raises.  Build with `python -m paper_1910_03552_b200.build`
(or `__graft_entry__.build()`).
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from .errors import NativeError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbeast_b200.so")

_lib = None

P = C.c_void_p
I = C.c_int
I64 = C.c_int64
F = C.c_float
SZ = C.c_size_t

# name -> (restype, argtypes); every symbol include/beast_b200.h declares
SIGNATURES: dict[str, tuple] = {
    "bp_abi_version": (I, []),
    "bp_last_error": (C.c_char_p, []),
    "bp_launch_count": (C.c_ulonglong, []),
    "bp_vtrace_from_logits_f32": (I, [P, P, P, P, P, P, P, I, I, I, F, F, F, P, P, P, P, P, P, P]),
    "bp_vtrace_from_importance_weights_f32": (I, [P, P, P, P, P, I, I, F, F, F, P, P, P, P, P]),
    "bp_learner_loss_workspace_bytes": (SZ, [I, I, I]),
    "bp_learner_loss_f32": (I, [P, P, P, P, P, P, I, I, I, F, F, F, F, F, F, F, I,
                                P, P, P, P, P, P, P, P, P]),
    "bp_sumsq_workspace_bytes": (SZ, [I64]),
    "bp_sumsq_f32": (I, [P, I64, P, P, P]),
    "bp_rmsprop_clip_f32": (I, [P, P, P, I64, P, F, I, F, P, F, F, I, P, P, P, P, P]),
    "bp_loss_workspace_bytes": (SZ, []),
    "bp_pg_loss_f32": (I, [P, P, P, C.c_longlong, I, P, P, P, P, P]),
    "bp_baseline_loss_f32": (I, [P, C.c_longlong, P, P, P, P]),
    "bp_entropy_loss_f32": (I, [P, C.c_longlong, I, P, P, P, P, P]),
    "bp_pg_loss_bwd_f32": (I, [P, P, P, C.c_longlong, I, P, P, P]),
    "bp_baseline_loss_bwd_f32": (I, [P, C.c_longlong, P, P, P]),
    "bp_entropy_loss_bwd_f32": (I, [P, C.c_longlong, I, P, P, P]),
    "bp_atari_param_count": (I64, [I, I]),
    "bp_atari_param_offsets": (I, [I, I, P]),
    "bp_atari_workspace_bytes": (SZ, [I, I]),
    "bp_atari_pack_weights": (I, [P, P, P]),
    "bp_atari_forward": (I, [P, I, P, P, P, P, P, P, P]),
    "bp_atari_set_conv1_u8": (I, [I]),
    "bp_atari_set_wgrad_window": (I, [I]),
    "bp_gemm_trace_next": (I, [P, I, I]),
    "bp_atari_forward_planes": (I, [P, I, P, P, I, P, P, P, P, P, P]),
    "bp_atari_backward": (I, [P, I, P, P, P, P, P, P]),
    "bp_atari_backward_frames": (I, [P, I, P, P, I, P, P, P, P]),
    "bp_lstm_partial_floats": (SZ, [I]),
    "bp_lstm_trace": (I, [P]),
    "bp_lstm_set_mode": (I, [I]),
    "bp_lstm_cluster_active": (I, []),
    "bp_lstm_cluster_capacity": (I, []),
    "bp_atari_lstm_forward": (I, [P, P, I, I, P, P, P, P, P, P, P, P, P, P, P, P]),
    "bp_atari_lstm_forward_planes": (I, [P, P, I, I, P, P, I, P, P, P, P, P, P, P, P, P, P, P]),
    "bp_atari_lstm_backward": (I, [P, P, I, I, P, P, P, P, P, P, P]),
    "bp_sample_actions_f32": (I, [P, I, I, C.c_uint64, I, P, P]),
    "bp_atari_forward_sample": (I, [P, I, P, P, I, P, P, P, C.c_uint64, P, I, P, P, P, P]),
    "bp_atari_lstm_forward_sample": (I, [P, P, I, I, P, P, I, P, P, P, P, P, P, C.c_uint64, P, I,
                                         P, P, P, P, P, P]),
    "bp_pack_stats": (I, [P, P, P, I, P, P, P, P, P]),
    "bp_host_wait_seq": (I, [P, C.c_uint, C.c_longlong]),
    "bp_copy_many": (I, [P, P, P, I, P]),
    "bp_infeed_put": (I, [P, P, C.c_size_t, P, P, P]),
    "bp_infeed_get": (I, [P, P, P]),
    "bp_gemm_bf16_test": (I, [P, P, P, I, I, I, I, I, I, I, P]),
    "bp_gemm_shift_test": (I, [P, P, P, I, I, I, I, P, I, P, I, P]),
}


BP_NET_NO_X0 = 1


class BpAtariNet(C.Structure):
    """Mirror of `BpAtariNet` in include/beast_b200.h (field order matters)."""

    _fields_ = [("num_actions", C.c_int), ("max_frames", C.c_int), ("use_lstm", C.c_int)] + [
        (name, C.c_void_p) for name in (
            "wbf", "whf", "x0", "x1", "x2", "x3", "core", "m1", "m2", "m3", "mc", "g", "d_fc",
            "d_pre3", "d_pre2", "d_pre1", "ws")
    ] + [("ws_bytes", C.c_size_t), ("flags", C.c_int), ("fc_grad_ready", C.c_void_p)]


class BpLstmCore(C.Structure):
    """Mirror of `BpLstmCore` in include/beast_b200.h (field order matters)."""

    _fields_ = [("hidden", C.c_int), ("max_rows", C.c_int)] + [
        (name, C.c_void_p) for name in (
            "wih", "gx", "gates", "cseq", "hprev", "out", "hx", "part", "dgates", "dh", "dx", "wpart")
    ]


def load(path: str = LIB_PATH):
    """Load (once) and type the library. Raises NativeError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeError(
            f"{path} not built; run `python -m paper_1910_03552_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    return _lib if _lib is not None else load()


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().bp_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed (code {rc}): {msg}")


def ptr(t) -> int | None:
    """Device pointer of a tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def require_cuda(*tensors) -> None:
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device: the B200 kernels have no CPU fallback")
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise NativeError("expected CUDA tensors")
