"""beastpipe-compatible learner ops on the fused sm_100a kernels.

Same names, argument meaning and error behaviour as the in-tree reference
(/root/reference/pkg/src/beastpipe/vtrace.py):

    VtraceConfig, VtraceResult, LossBundle            vtrace.py:18-48
    action_log_rhos(behavior, target, actions)        vtrace.py:51-69
    vtrace_targets(log_rhos, ..., cfg)                vtrace.py:94-128
    compute_losses(batch, logits, baseline, cfg)      vtrace.py:224-255

Inputs may be numpy arrays (copied to the GPU, results returned as float32
numpy -- the reference's training precision) or CUDA tensors (results stay
on the device).  The arithmetic is fp32 on the GPU; the stated tolerance vs
the fp64 oracle is 1e-5 relative.  Data-dependent violations are
raised synchronously here (SchemaError / NonFiniteError), matching the
reference which raises immediately.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._tensors import out_like, status_word, to_cuda
from .errors import SchemaError
from .vtrace import from_importance_weights, from_logits


@dataclass(frozen=True)
class VtraceConfig:
    """vtrace.py:18-33, plus the upstream knobs the fused kernel exposes.

    pg_rho_bar None -> same as rho_bar (beastpipe); reward_clip -> upstream
    `reward_clipping == "abs_one"`; row_shift 0 -> beastpipe row alignment
    (actions / behaviour logits from rows 0..T-1, vtrace.py:243-244), 1 ->
    upstream learn() (`batch[1:]`).
    """

    discount: float = 0.99
    rho_bar: float = 1.0
    c_bar: float = 1.0
    baseline_cost: float = 0.5
    entropy_cost: float = 0.01
    pg_cost: float = 1.0
    pg_rho_bar: float | None = None
    reward_clip: bool = False
    row_shift: int = 0

    def __post_init__(self):
        if not 0.0 < self.discount <= 1.0:
            raise ValueError(f"discount must be in (0, 1], got {self.discount}")
        if not self.rho_bar >= self.c_bar > 0.0:
            raise ValueError(f"need rho_bar >= c_bar > 0, got {self.rho_bar}, {self.c_bar}")
        if self.row_shift not in (0, 1):
            raise ValueError("row_shift must be 0 (beastpipe) or 1 (torchbeast)")


@dataclass(frozen=True)
class VtraceResult:
    """vtrace.py:36-40."""

    vs: object
    pg_advantages: object
    clipped_rhos: object


@dataclass(frozen=True)
class LossBundle:
    """vtrace.py:43-48 (sum-reduced scalars)."""

    pg_loss: float
    baseline_loss: float
    entropy_loss: float
    total: float


def action_log_rhos(behavior_logits, target_logits, actions):
    """log pi_target(a|x) - log pi_behavior(a|x) per (T, B) step (vtrace.py:51-69)."""
    if tuple(behavior_logits.shape) != tuple(target_logits.shape):
        raise SchemaError(f"logits shapes differ: {tuple(behavior_logits.shape)} vs "
                          f"{tuple(target_logits.shape)}")
    if tuple(actions.shape) != tuple(behavior_logits.shape[:-1]):
        raise SchemaError(f"actions shape {tuple(actions.shape)}, expected "
                          f"{tuple(behavior_logits.shape[:-1])}")
    as_np = not isinstance(behavior_logits, torch.Tensor)
    beh, _ = to_cuda(behavior_logits, torch.float32)
    squeeze = beh.dim() == 2
    tgt, _ = to_cuda(target_logits, torch.float32, beh.device)
    act, _ = to_cuda(actions, torch.int64, beh.device)
    if squeeze:  # (N, A) -> (1, N, A)
        beh, tgt, act = beh[None], tgt[None], act[None]
    T, B = act.shape
    z = torch.zeros((T, B), device=beh.device)
    r = from_logits(beh, tgt, act, z, z, z, torch.zeros(B, device=beh.device))
    status_word(beh.device).check("action_log_rhos")
    lr = r.log_rhos[0] if squeeze else r.log_rhos
    return out_like(lr, as_np)


def vtrace_targets(log_rhos, discounts, rewards, values, bootstrap_value, cfg: VtraceConfig):
    """Backward-recursion V-trace over (T, B) inputs (vtrace.py:94-128)."""
    shape = tuple(log_rhos.shape)
    if len(shape) != 2:
        raise SchemaError(f"log_rhos must be (T, B), got {shape}")
    for name, arr in (("discounts", discounts), ("rewards", rewards), ("values", values)):
        if tuple(arr.shape) != shape:
            raise SchemaError(f"{name} shape {tuple(arr.shape)}, expected {shape}")
    if tuple(bootstrap_value.shape) != (shape[1],):
        raise SchemaError(f"bootstrap_value shape {tuple(bootstrap_value.shape)}, "
                          f"expected ({shape[1]},)")
    as_np = not isinstance(log_rhos, torch.Tensor)
    pg_bar = cfg.rho_bar if cfg.pg_rho_bar is None else cfg.pg_rho_bar
    ret, cr = from_importance_weights(log_rhos, discounts, rewards, values, bootstrap_value,
                                      clip_rho_threshold=cfg.rho_bar,
                                      clip_pg_rho_threshold=pg_bar, clip_c_threshold=cfg.c_bar,
                                      check=True, return_clipped_rhos=True)
    return VtraceResult(vs=out_like(ret.vs, as_np), pg_advantages=out_like(ret.pg_advantages, as_np),
                        clipped_rhos=out_like(cr, as_np))


class LearnerLoss:
    """Reusable launcher of the fused learner-loss kernel (workspace cached per shape).

    forward(...) enqueues one kernel and returns device tensors; nothing syncs.
    """

    def __init__(self, device=None):
        self.device = torch.device(device or "cuda")
        self._ws = {}
        self.losses = torch.zeros(4, dtype=torch.float64, device=self.device)

    def workspace(self, T, B, A):
        key = (T, B, A)
        ws = self._ws.get(key)
        if ws is None:
            nbytes = N.lib().bp_learner_loss_workspace_bytes(T, B, A)
            ws = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
            self._ws[key] = ws
        return ws

    def __call__(self, learner_logits, learner_baseline, behavior_logits, actions, rewards, done,
                 cfg: VtraceConfig, d_logits=None, d_baseline=None, vs=None, pg_advantages=None,
                 losses=None, status=None, clipped_rhos=None):
        T, B, A = learner_logits.shape[-3], learner_logits.shape[-2], learner_logits.shape[-1]
        if d_logits is None:
            d_logits = torch.empty((T, B, A), dtype=torch.float32, device=self.device)
        if d_baseline is None:
            d_baseline = torch.empty((T + 1, B), dtype=torch.float32, device=self.device)
        if losses is None:
            losses = self.losses
        sw = status if status is not None else status_word(self.device)
        pg_bar = cfg.rho_bar if cfg.pg_rho_bar is None else cfg.pg_rho_bar
        N.check(N.lib().bp_learner_loss_f32(
            N.ptr(learner_logits), N.ptr(learner_baseline), N.ptr(behavior_logits), N.ptr(actions),
            N.ptr(rewards), N.ptr(done), T, B, A, float(cfg.discount), float(cfg.rho_bar),
            float(pg_bar), float(cfg.c_bar), float(cfg.pg_cost), float(cfg.baseline_cost),
            float(cfg.entropy_cost), int(bool(cfg.reward_clip)), N.ptr(d_logits),
            N.ptr(d_baseline), N.ptr(vs), N.ptr(pg_advantages), N.ptr(clipped_rhos), N.ptr(losses),
            N.ptr(self.workspace(T, B, A)), sw.ptr(), N.stream_handle(self.device)),
            "bp_learner_loss_f32")
        return d_logits, d_baseline, losses


_loss_launchers: dict = {}


def _launcher(device) -> LearnerLoss:
    key = device.index if device.index is not None else torch.cuda.current_device()
    ll = _loss_launchers.get(key)
    if ll is None:
        ll = LearnerLoss(torch.device("cuda", key))
        _loss_launchers[key] = ll
    return ll


def compute_losses(batch, learner_logits, learner_baseline, cfg: VtraceConfig):
    """Full learner loss for one batch in ONE kernel (vtrace.py:224-255).

    learner_logits (T, B, A), learner_baseline (T+1, B).  Rewards and done are
    read shifted by one row; actions / behaviour logits per `cfg.row_shift`.
    Returns (LossBundle, d_logits, d_baseline, VtraceResult) like the reference.
    """
    t_len = batch.observation.shape[0] - 1
    b = batch.observation.shape[1]
    a = batch.policy_logits.shape[-1]
    if tuple(learner_logits.shape) != (t_len, b, a):
        raise SchemaError(f"learner_logits shape {tuple(learner_logits.shape)}, expected "
                          f"({t_len}, {b}, {a})")
    if tuple(learner_baseline.shape) != (t_len + 1, b):
        raise SchemaError(f"baseline rows {learner_baseline.shape[0]}, expected {t_len + 1}")
    as_np = not isinstance(learner_logits, torch.Tensor)
    lg, _ = to_cuda(learner_logits, torch.float32)
    dev = lg.device
    bl, _ = to_cuda(learner_baseline, torch.float32, dev)
    beh_rows, _ = to_cuda(batch.policy_logits, torch.float32, dev)
    act_rows, _ = to_cuda(batch.action, torch.int64, dev)
    rew_rows, _ = to_cuda(batch.reward, torch.float32, dev)
    done_rows, _ = to_cuda(batch.done, torch.bool, dev)
    s = cfg.row_shift
    beh = beh_rows[s:s + t_len]
    act = act_rows[s:s + t_len]
    vs = torch.empty((t_len, b), device=dev)
    pg = torch.empty((t_len, b), device=dev)
    cr = torch.empty((t_len, b), device=dev)
    ll = _launcher(dev)
    losses = torch.empty(4, dtype=torch.float64, device=dev)
    d_logits, d_baseline, losses = ll(lg, bl, beh, act, rew_rows[1:], done_rows[1:], cfg,
                                      vs=vs, pg_advantages=pg, losses=losses, clipped_rhos=cr)
    status_word(dev).check("compute_losses")
    lv = losses.cpu().tolist()
    bundle = LossBundle(pg_loss=lv[0], baseline_loss=lv[1], entropy_loss=lv[2], total=lv[3])
    targets = VtraceResult(vs=out_like(vs, as_np), pg_advantages=out_like(pg, as_np),
                           clipped_rhos=out_like(cr, as_np))
    return bundle, out_like(d_logits, as_np), out_like(d_baseline, as_np), targets
