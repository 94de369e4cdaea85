"""Fused global-norm clip + RMSProp on flat fp32 buffers (two HBM-bound kernels).

Replaces SharedModel.apply_gradients (pipeline.py:247-251) =
clip_global_norm (model.py:224-233) + rmsprop_step (model.py:236-268), and
upstream learn()'s `clip_grad_norm_` + `torch.optim.RMSprop.step()`.

* `RMSprop` is a torch.optim.Optimizer with torch's signature (momentum=0,
  centered=False, weight_decay=0 only).  Its parameters, gradients and
  square_avg live in three flat buffers; the Parameters become views.
* `clip_global_norm` / `rmsprop_step` mirror the beastpipe functions on
  lists of arrays (numpy or CUDA tensors).
* clip modes: "beastpipe" (scale only when norm > max), "torch"
  (min(1, max/(norm+1e-6)), always applied), "none".
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from ._tensors import status_word, to_cuda
from .errors import NonFiniteError

CLIP_MODES = {"beastpipe": 0, "torch": 1, "none": 2}


class _Workspace:
    _cache: dict = {}

    @classmethod
    def get(cls, device, n):
        key = (device.index, "sumsq")
        ws = cls._cache.get(key)
        need = N.lib().bp_sumsq_workspace_bytes(n)
        if ws is None or ws.numel() < need:
            ws = torch.zeros(need, dtype=torch.uint8, device=device)
            cls._cache[key] = ws
        return ws


def sumsq_(flat: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """out[0] (f64, device) <- sum(flat**2); deterministic, no host sync."""
    N.check(N.lib().bp_sumsq_f32(N.ptr(flat), flat.numel(), N.ptr(out),
                                 N.ptr(_Workspace.get(flat.device, flat.numel())),
                                 N.stream_handle(flat.device)), "bp_sumsq_f32")
    return out


def rmsprop_clip_(params: torch.Tensor, grads: torch.Tensor, square_avg: torch.Tensor,
                  sumsq: torch.Tensor, *, lr: float, alpha: float, eps: float, max_norm: float,
                  clip_mode: str = "torch", lr_dev: torch.Tensor | None = None,
                  write_clipped_grads: bool = True, norm_out: torch.Tensor | None = None,
                  mirror: torch.Tensor | None = None, status=None,
                  reject_if_nonfinite: torch.Tensor | None = None) -> None:
    """In-place clip + RMSProp over flat buffers, norm read from `sumsq` on device.
    reject_if_nonfinite: a device f64 scalar (the step's total loss); non-finite -> the
    whole update is rejected on device, like a non-finite gradient norm.
    status: the StatusWord for BP_STATUS_NONFINITE_GRAD (None: the per-device word; False: none,
    e.g. when a concurrent stats pack derives the bit from `sumsq` itself)."""
    sw = None if status is False else status if status is not None else status_word(params.device)
    N.check(N.lib().bp_rmsprop_clip_f32(
        N.ptr(params), N.ptr(grads), N.ptr(square_avg), params.numel(), N.ptr(sumsq),
        float(max_norm), CLIP_MODES[clip_mode], float(lr), N.ptr(lr_dev), float(alpha),
        float(eps), int(write_clipped_grads), N.ptr(norm_out), N.ptr(mirror), sw.ptr() if sw else None,
        N.ptr(reject_if_nonfinite), N.stream_handle(params.device)), "bp_rmsprop_clip_f32")


def flatten_params_(params: list[torch.nn.Parameter], device) -> tuple[torch.Tensor, torch.Tensor]:
    """Re-home parameters (and their grads) as views of two flat fp32 buffers."""
    total = sum(p.numel() for p in params)
    flat = torch.empty(total, dtype=torch.float32, device=device)
    gflat = torch.zeros(total, dtype=torch.float32, device=device)
    off = 0
    for p in params:
        n = p.numel()
        flat[off:off + n].copy_(p.detach().reshape(-1))
        p.data = flat[off:off + n].view_as(p)
        p.grad = gflat[off:off + n].view_as(p)
        off += n
    return flat, gflat


def _is_flat(params, flat) -> bool:
    off = 0
    base = flat.data_ptr()
    for p in params:
        if p.data_ptr() != base + 4 * off or not p.is_contiguous():
            return False
        off += p.numel()
    return off == flat.numel()


def _flat_view(tensors):
    """If `tensors` are contiguous, in-order views of one f32 storage, return a flat view of them."""
    if not tensors or any(t is None or t.dtype != torch.float32 or not t.is_contiguous() for t in tensors):
        return None
    st = tensors[0].untyped_storage()
    off0 = tensors[0].storage_offset()
    off = off0
    for t in tensors:
        if t.untyped_storage().data_ptr() != st.data_ptr() or t.storage_offset() != off:
            return None
        off += t.numel()
    return tensors[0].detach().new_empty(0).set_(st, off0, (off - off0,))


class RMSprop(torch.optim.Optimizer):
    """torch.optim.RMSprop-compatible optimiser with a fused clip + update kernel.

    step(max_norm=None) applies clip_grad_norm_-style clipping (mode
    `clip_mode`) in the same two launches.  Flat buffers: `self.flat_params`,
    `self.flat_grads`, `self.square_avg`.
    """

    def __init__(self, params, lr=1e-2, alpha=0.99, eps=1e-8, weight_decay=0, momentum=0,
                 centered=False, clip_mode="torch", flat=None):
        if momentum != 0 or centered or weight_decay != 0:
            raise ValueError("fused RMSprop supports momentum=0, centered=False, weight_decay=0")
        defaults = dict(lr=lr, alpha=alpha, eps=eps, weight_decay=0, momentum=0, centered=False)
        super().__init__(params, defaults)
        plist = [p for g in self.param_groups for p in g["params"]]
        self.device = plist[0].device
        fp = _flat_view([p.data for p in plist])
        fg = _flat_view([p.grad for p in plist]) if fp is not None else None
        if flat is not None and _is_flat(plist, flat[0]):
            self.flat_params, self.flat_grads = flat
        elif fp is not None and fg is not None:  # e.g. AtariNet: params already flat
            self.flat_params, self.flat_grads = fp, fg
        else:
            self.flat_params, self.flat_grads = flatten_params_(plist, self.device)
        self.square_avg = torch.zeros_like(self.flat_params)
        self._sumsq = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.norm = torch.zeros(1, dtype=torch.float32, device=self.device)
        self.lr_dev = torch.full((1,), float(lr), dtype=torch.float32, device=self.device)
        self._lr_host = float(lr)
        self._sumsq_zero = False
        self.clip_mode = clip_mode
        off = 0
        for p in plist:  # expose torch-style state views
            n = p.numel()
            self.state[p]["square_avg"] = self.square_avg[off:off + n].view_as(p)
            self.state[p]["step"] = torch.zeros((), dtype=torch.float32)
            off += n

    @property
    def lr(self) -> float:
        return self.param_groups[0]["lr"]

    def zero_grad(self, set_to_none: bool = False):
        self.flat_grads.zero_()

    def sync_lr(self) -> None:
        """Mirror param_groups[0]["lr"] (edited by LR schedulers) into the device scalar
        the update kernel reads; called outside CUDA-graph replays."""
        lr = self.param_groups[0]["lr"]
        if lr != self._lr_host:
            self.lr_dev.fill_(lr)
            self._lr_host = lr

    @torch.no_grad()
    def step(self, closure=None, max_norm: float | None = None, mirror: torch.Tensor | None = None,
             status=None, reject_if_nonfinite: torch.Tensor | None = None, on_norm=None):
        """One fused clip + RMSProp update.  status: the StatusWord that receives
        BP_STATUS_NONFINITE_GRAD (default: the per-device word; False: none); reject_if_nonfinite:
        a device f64 scalar (the learner step's total loss) whose non-finite value rejects the
        update; on_norm(sumsq): called once the squared-norm reduction is enqueued, before the
        update (the learner forks its stats pack there)."""
        loss = closure() if closure is not None else None
        if not torch.cuda.is_current_stream_capturing():
            self.sync_lr()
        mode = self.clip_mode if max_norm is not None else "none"
        if mode != "none":
            sumsq_(self.flat_grads, self._sumsq)
        elif not self._sumsq_zero:
            self._sumsq.zero_()
        self._sumsq_zero = mode == "none"
        if on_norm is not None:
            on_norm(self._sumsq)
        g = self.param_groups[0]
        rmsprop_clip_(self.flat_params, self.flat_grads, self.square_avg, self._sumsq,
                      lr=g["lr"], alpha=g["alpha"], eps=g["eps"],
                      max_norm=float(max_norm or 0.0), clip_mode=mode, lr_dev=self.lr_dev,
                      norm_out=self.norm, mirror=mirror, status=status,
                      reject_if_nonfinite=reject_if_nonfinite)
        return loss


def clip_grad_norm_(parameters, max_norm: float) -> torch.Tensor:
    """Device-side global norm + torch-style in-place clip; returns the norm tensor."""
    params = [p for p in parameters if p.grad is not None]
    dev = params[0].grad.device
    flat = torch.cat([p.grad.reshape(-1) for p in params])
    ss = torch.zeros(1, dtype=torch.float64, device=dev)
    sumsq_(flat, ss)
    norm = ss.sqrt().to(torch.float32)[0]
    coef = torch.clamp(max_norm / (norm + 1e-6), max=1.0)
    for p in params:
        p.grad.mul_(coef)
    return norm


# --- beastpipe mirrors (model.py:224-268), lists of arrays in / out ------------

def clip_global_norm(grads, max_norm: float):
    """model.py:224-233 on a list of arrays; returns (clipped list, total norm float)."""
    as_np = not isinstance(grads[0], torch.Tensor)
    ts = [to_cuda(g, torch.float32)[0] for g in grads]
    flat = torch.cat([t.reshape(-1) for t in ts])
    ss = torch.zeros(1, dtype=torch.float64, device=flat.device)
    sumsq_(flat, ss)
    total = float(np.sqrt(ss.item()))
    if max_norm <= 0 or total <= max_norm:
        out = [t.clone() for t in ts]
    else:
        scale = max_norm / total
        out = [t * np.float32(scale) for t in ts]
    if as_np:
        out = [t.cpu().numpy() for t in out]
    return out, total


def rmsprop_step(params, grads, g2, learning_rate=0.005, decay=0.99, epsilon=0.01):
    """model.py:236-268 on lists of arrays; returns fresh (params, g2) lists."""
    as_np = not isinstance(params[0], torch.Tensor)
    ps = [to_cuda(p, torch.float32)[0] for p in params]
    dev = ps[0].device
    shapes = [p.shape for p in ps]
    fp = torch.cat([p.reshape(-1) for p in ps])
    fg = torch.cat([to_cuda(g, torch.float32, dev)[0].reshape(-1) for g in grads])
    fs = torch.cat([to_cuda(s, torch.float32, dev)[0].reshape(-1) for s in g2])
    if not bool(torch.isfinite(fg).all()):
        raise NonFiniteError("grad contains non-finite values")
    ss = torch.zeros(1, dtype=torch.float64, device=dev)
    rmsprop_clip_(fp, fg, fs, ss, lr=learning_rate, alpha=decay, eps=epsilon, max_norm=0.0,
                  clip_mode="none", write_clipped_grads=False)
    status_word(dev).check("rmsprop_step")
    outp, outs, off = [], [], 0
    for shp in shapes:
        n = int(np.prod(shp)) if len(shp) else 1
        outp.append(fp[off:off + n].view(shp))
        outs.append(fs[off:off + n].view(shp))
        off += n
    if as_np:
        outp = [t.cpu().numpy() for t in outp]
        outs = [t.cpu().numpy() for t in outs]
    return outp, outs
