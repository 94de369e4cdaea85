"""TorchBeast-compatible V-trace API on the fused sm_100a kernels.

Drop-in for upstream `torchbeast.core.vtrace` [upstream, not vendored]:
`from_logits`, `from_importance_weights`, `VTraceFromLogitsReturns`,
`VTraceReturns`, `action_log_probs`.  The in-tree reference arithmetic is
beastpipe `action_log_rhos` + `vtrace_targets`
(/root/reference/pkg/src/beastpipe/vtrace.py:51-128).

All tensors are time-major (T, B[, A]) on the current CUDA device; the
kernel runs on the current torch stream.  Results carry no autograd graph
(upstream computes vs / pg_advantages under no_grad as well).

Error behaviour: the kernels OR violations (action out of range, non-finite
input, negative discount) into a device status word.  `from_logits` leaves it
unchecked to stay asynchronous (upstream does no validation either); call
`check_status()` or pass `check=True` to raise `SchemaError` /
`NonFiniteError` like beastpipe does.
"""
from __future__ import annotations

import collections
import math

import torch

from . import _native as N
from ._tensors import expect_shape, status_word, to_cuda

VTraceFromLogitsReturns = collections.namedtuple(
    "VTraceFromLogitsReturns",
    ["vs", "pg_advantages", "log_rhos", "behavior_action_log_probs", "target_action_log_probs"],
)
VTraceReturns = collections.namedtuple("VTraceReturns", "vs pg_advantages")


def _clip(v) -> float:
    return math.inf if v is None else float(v)


def check_status(device=None) -> None:
    """Raise SchemaError / NonFiniteError if any V-trace launch flagged bad input."""
    status_word(torch.device(device or "cuda")).check("vtrace")


def from_logits(behavior_policy_logits, target_policy_logits, actions, discounts, rewards, values,
                bootstrap_value, clip_rho_threshold=1.0, clip_pg_rho_threshold=1.0, *,
                clip_c_threshold=1.0, check=False):
    """V-trace for softmax policies, one fused kernel (log-softmax x2, gather,
    clipped rho / c, reverse scan over T, pg advantages)."""
    beh, _ = to_cuda(behavior_policy_logits, torch.float32)
    dev = beh.device
    tgt, _ = to_cuda(target_policy_logits, torch.float32, dev)
    if beh.dim() != 3:
        raise N.NativeError("policy logits must be (T, B, A)")
    T, B, A = beh.shape
    expect_shape("target_policy_logits", tgt, (T, B, A))
    act, _ = to_cuda(actions, torch.int64, dev)
    disc, _ = to_cuda(discounts, torch.float32, dev)
    rew, _ = to_cuda(rewards, torch.float32, dev)
    val, _ = to_cuda(values, torch.float32, dev)
    boot, _ = to_cuda(bootstrap_value, torch.float32, dev)
    for name, t in (("actions", act), ("discounts", disc), ("rewards", rew), ("values", val)):
        expect_shape(name, t, (T, B))
    expect_shape("bootstrap_value", boot, (B,))
    outs = torch.empty((5, T, B), dtype=torch.float32, device=dev)
    vs, pg, lr, blp, tlp = outs.unbind(0)
    sw = status_word(dev)
    N.check(N.lib().bp_vtrace_from_logits_f32(
        N.ptr(beh), N.ptr(tgt), N.ptr(act), N.ptr(disc), N.ptr(rew), N.ptr(val), N.ptr(boot),
        T, B, A, _clip(clip_rho_threshold), _clip(clip_pg_rho_threshold), _clip(clip_c_threshold),
        N.ptr(vs), N.ptr(pg), N.ptr(lr), N.ptr(blp), N.ptr(tlp), sw.ptr(),
        N.stream_handle(dev)), "bp_vtrace_from_logits_f32")
    if check:
        sw.check("from_logits")
    return VTraceFromLogitsReturns(vs=vs, pg_advantages=pg, log_rhos=lr,
                                   behavior_action_log_probs=blp, target_action_log_probs=tlp)


def from_importance_weights(log_rhos, discounts, rewards, values, bootstrap_value,
                            clip_rho_threshold=1.0, clip_pg_rho_threshold=1.0, *,
                            clip_c_threshold=1.0, check=False, return_clipped_rhos=False):
    """V-trace from log importance weights (reverse scan over T, parallel over B)."""
    lr, _ = to_cuda(log_rhos, torch.float32)
    dev = lr.device
    if lr.dim() != 2:
        raise N.NativeError("log_rhos must be (T, B)")
    T, B = lr.shape
    disc, _ = to_cuda(discounts, torch.float32, dev)
    rew, _ = to_cuda(rewards, torch.float32, dev)
    val, _ = to_cuda(values, torch.float32, dev)
    boot, _ = to_cuda(bootstrap_value, torch.float32, dev)
    for name, t in (("discounts", disc), ("rewards", rew), ("values", val)):
        expect_shape(name, t, (T, B))
    expect_shape("bootstrap_value", boot, (B,))
    outs = torch.empty((3, T, B), dtype=torch.float32, device=dev)
    vs, pg, cr = outs.unbind(0)
    sw = status_word(dev)
    N.check(N.lib().bp_vtrace_from_importance_weights_f32(
        N.ptr(lr), N.ptr(disc), N.ptr(rew), N.ptr(val), N.ptr(boot), T, B,
        _clip(clip_rho_threshold), _clip(clip_pg_rho_threshold), _clip(clip_c_threshold),
        N.ptr(vs), N.ptr(pg), N.ptr(cr), sw.ptr(), N.stream_handle(dev)),
        "bp_vtrace_from_importance_weights_f32")
    if check:
        sw.check("from_importance_weights")
    if return_clipped_rhos:
        return VTraceReturns(vs=vs, pg_advantages=pg), cr
    return VTraceReturns(vs=vs, pg_advantages=pg)


def action_log_probs(policy_logits, actions):
    """log softmax(policy_logits)[actions], shape of `actions` (upstream helper).

    Computed by the fused kernel (behaviour side of a from_logits call against
    itself); the gather is exact.
    """
    r = from_logits(policy_logits, policy_logits, actions,
                    torch.zeros(actions.shape, device=policy_logits.device),
                    torch.zeros(actions.shape, device=policy_logits.device),
                    torch.zeros(actions.shape, device=policy_logits.device),
                    torch.zeros(actions.shape[1:], device=policy_logits.device))
    return r.target_action_log_probs
