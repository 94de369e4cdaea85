"""numpy restatement of the softmax family, global-norm clip and RMSProp.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.
Citations are into /root/reference/pkg/src/beastpipe/model.py.
"""
from __future__ import annotations

import numpy as np


class NonFiniteError(ValueError):
    """Mirror of model.py:21."""


def log_softmax(logits: np.ndarray) -> np.ndarray:
    """model.py:206-209: max-shifted log-softmax over the last axis."""
    shifted = logits - logits.max(axis=-1, keepdims=True)
    return shifted - np.log(np.exp(shifted).sum(axis=-1, keepdims=True))


def entropy(logits: np.ndarray) -> np.ndarray:
    """model.py:212-215: -sum pi log pi over the last axis."""
    logp = log_softmax(logits)
    return -(np.exp(logp) * logp).sum(axis=-1)


def global_norm(grads) -> float:
    """model.py:226-228: sqrt of the sum of squares over every gradient array (fp64)."""
    return float(np.sqrt(sum(float(np.sum(np.asarray(g, np.float64) ** 2)) for g in grads)))


def clip_global_norm(grads, max_norm: float, mode: str = "beastpipe"):
    """Clip a list of gradient arrays; returns (clipped list, total norm).

    mode="beastpipe": model.py:224-233 -- scale by max/total only if total > max
    (and max > 0).
    mode="torch": torch.nn.utils.clip_grad_norm_ -- coef = max/(total+1e-6),
    clamped to <= 1, always applied [upstream learn(), not vendored].
    """
    total = global_norm(grads)
    if mode == "beastpipe":
        if max_norm <= 0 or total <= max_norm:
            return [np.array(g, copy=True) for g in grads], total
        scale = max_norm / total
    elif mode == "torch":
        scale = min(1.0, max_norm / (total + 1e-6))
    else:
        raise ValueError(mode)
    return [g * g.dtype.type(scale) for g in grads], total


def rmsprop_step(params, grads, g2, lr: float, decay: float, eps: float):
    """model.py:236-268: g2 <- a g2 + (1-a) g^2; p <- p - lr g / (sqrt(g2) + eps).

    Epsilon outside the root, no momentum (== torch.optim.RMSprop defaults).
    Returns fresh (params, g2) lists; rejects non-finite gradients (model.py:251-252).
    """
    new_p, new_g2 = [], []
    for p, g, s in zip(params, grads, g2):
        if not np.all(np.isfinite(g)):
            raise NonFiniteError("non-finite gradient")
        s2 = decay * s + (1.0 - decay) * g * g
        denom = np.sqrt(s2) + eps
        step = np.divide(g, denom, out=np.zeros_like(g), where=denom != 0.0)
        new_p.append(p - lr * step)
        new_g2.append(s2)
    return new_p, new_g2
