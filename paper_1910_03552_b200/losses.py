"""The north-star loss helpers on fused sm_100a reduction kernels, with autograd.

Drop-in for upstream TorchBeast `monobeast.compute_baseline_loss(advantages)`,
`compute_entropy_loss(logits)` and `compute_policy_gradient_loss(logits, actions,
advantages)` [upstream, not vendored]: same signatures, sum-reduced 0-dim float32 results,
gradients through `loss.backward()`.  The in-tree arithmetic they restate is beastpipe
`losses_from_targets` (/root/reference/pkg/src/beastpipe/vtrace.py:169-221):
pg = -sum adv * log pi(a) (:194), baseline = 0.5 sum (vs - V)^2 (:195),
entropy_loss = -sum H = sum pi log pi (:196, model.py:212-215), and the exact gradients
(:208-214).  Each forward is one kernel (logits read once, deterministic f64 reduction),
each backward one elementwise kernel reading the upstream gradient on device (no sync).

Errors: an action outside [0, A) in the pg loss ORs BP_STATUS_ACTION_RANGE into the
per-device status word (F.nll_loss rejects it); pass check=True (one sync) to raise
SchemaError immediately, or call vtrace.check_status() later.
"""
from __future__ import annotations

import torch

from . import _native as N
from ._tensors import status_word
from .errors import SchemaError

_ws: dict = {}


def _workspace(device, which: str) -> torch.Tensor:
    key = (device.index, which)
    ws = _ws.get(key)
    if ws is None:
        ws = torch.zeros(N.lib().bp_loss_workspace_bytes(), dtype=torch.uint8, device=device)
        _ws[key] = ws
    return ws


def _f32(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        N.require_cuda()
        raise SchemaError(f"{name}: expected a CUDA tensor")
    return t.detach().float().contiguous()


class _BaselineLoss(torch.autograd.Function):
    @staticmethod
    def forward(ctx, advantages):
        adv = _f32(advantages, "advantages")
        out = torch.empty((), dtype=torch.float32, device=adv.device)
        N.check(N.lib().bp_baseline_loss_f32(N.ptr(adv), adv.numel(), N.ptr(out), None,
                                             N.ptr(_workspace(adv.device, "baseline")),
                                             N.stream_handle(adv.device)), "bp_baseline_loss_f32")
        ctx.save_for_backward(adv)
        ctx.shape = advantages.shape
        return out

    @staticmethod
    def backward(ctx, grad):
        (adv,) = ctx.saved_tensors
        g = grad.float().contiguous()
        d = torch.empty_like(adv)
        N.check(N.lib().bp_baseline_loss_bwd_f32(N.ptr(adv), adv.numel(), N.ptr(g), N.ptr(d),
                                                 N.stream_handle(adv.device)), "bp_baseline_loss_bwd_f32")
        return d.view(ctx.shape)


class _EntropyLoss(torch.autograd.Function):
    @staticmethod
    def forward(ctx, logits):
        x = _f32(logits, "logits")
        A = x.shape[-1]
        rows = x.numel() // A if A else 0
        out = torch.empty((), dtype=torch.float32, device=x.device)
        N.check(N.lib().bp_entropy_loss_f32(N.ptr(x), rows, A, N.ptr(out), None,
                                            N.ptr(_workspace(x.device, "entropy")),
                                            status_word(x.device).ptr(), N.stream_handle(x.device)),
                "bp_entropy_loss_f32")
        ctx.save_for_backward(x)
        return out

    @staticmethod
    def backward(ctx, grad):
        (x,) = ctx.saved_tensors
        A = x.shape[-1]
        g = grad.float().contiguous()
        d = torch.empty_like(x)
        N.check(N.lib().bp_entropy_loss_bwd_f32(N.ptr(x), x.numel() // A, A, N.ptr(g), N.ptr(d),
                                                N.stream_handle(x.device)), "bp_entropy_loss_bwd_f32")
        return d


class _PolicyGradientLoss(torch.autograd.Function):
    @staticmethod
    def forward(ctx, logits, actions, advantages):
        x = _f32(logits, "logits")
        A = x.shape[-1]
        rows = x.numel() // A
        act = actions.detach().to(torch.int64).contiguous()
        adv = _f32(advantages, "advantages")
        if act.numel() != rows or adv.numel() != rows:
            raise SchemaError(f"logits {tuple(logits.shape)}, actions {tuple(actions.shape)} and advantages "
                              f"{tuple(advantages.shape)} disagree on the (T, B) rows")
        out = torch.empty((), dtype=torch.float32, device=x.device)
        N.check(N.lib().bp_pg_loss_f32(N.ptr(x), N.ptr(act), N.ptr(adv), rows, A, N.ptr(out), None,
                                       N.ptr(_workspace(x.device, "pg")), status_word(x.device).ptr(),
                                       N.stream_handle(x.device)), "bp_pg_loss_f32")
        ctx.save_for_backward(x, act, adv)
        return out

    @staticmethod
    def backward(ctx, grad):
        x, act, adv = ctx.saved_tensors
        A = x.shape[-1]
        g = grad.float().contiguous()
        d = torch.empty_like(x)
        N.check(N.lib().bp_pg_loss_bwd_f32(N.ptr(x), N.ptr(act), N.ptr(adv), x.numel() // A, A, N.ptr(g),
                                           N.ptr(d), N.stream_handle(x.device)), "bp_pg_loss_bwd_f32")
        return d, None, None  # upstream: cross_entropy * advantages.detach()


def compute_baseline_loss(advantages: torch.Tensor) -> torch.Tensor:
    """0.5 * sum(advantages ** 2)  (beastpipe vtrace.py:195 with advantages = vs - V)."""
    return _BaselineLoss.apply(advantages)


def compute_entropy_loss(logits: torch.Tensor, *, check: bool = False) -> torch.Tensor:
    """sum(softmax(logits) * log_softmax(logits)): the negative entropy (vtrace.py:196)."""
    out = _EntropyLoss.apply(logits)
    if check:
        status_word(out.device).check("compute_entropy_loss")
    return out


def compute_policy_gradient_loss(logits: torch.Tensor, actions: torch.Tensor, advantages: torch.Tensor, *,
                                 check: bool = False) -> torch.Tensor:
    """sum(nll(log_softmax(logits), actions) * advantages.detach())  (vtrace.py:194)."""
    out = _PolicyGradientLoss.apply(logits, actions, advantages)
    if check:
        status_word(out.device).check("compute_policy_gradient_loss")
    return out
