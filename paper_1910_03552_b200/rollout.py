"""Learner input schema on the device (mirror of beastpipe rollout.py:67-192).

`TrainingBatch` holds B rollouts stacked time-major, leading dims (T+1, B),
as CUDA tensors (u8 frames stay u8 in HBM).  `validate_batch` performs the
reference's shape / dtype checks on the host (rollout.py:160-183); the
data-dependent scans (action range rollout.py:184-188, finiteness :189-192)
are folded into the fused loss kernel's device status word instead of
separate full-array passes, and raise the same SchemaError / NonFiniteError
when the status is checked.
"""
from __future__ import annotations

from dataclasses import dataclass, fields

import torch

from .errors import SchemaError


@dataclass
class TrainingBatch:
    """rollout.py:67-89 (device-resident).  done is torch.bool (1 byte / entry)."""

    observation: torch.Tensor      # (T+1, B, *obs) uint8 frames or float
    reward: torch.Tensor           # (T+1, B) f32
    done: torch.Tensor             # (T+1, B) bool
    policy_logits: torch.Tensor    # (T+1, B, A) f32 behaviour logits
    baseline: torch.Tensor         # (T+1, B) f32 behaviour baseline
    action: torch.Tensor           # (T+1, B) int64
    model_versions: torch.Tensor   # (B,) int64
    last_action: torch.Tensor | None = None  # (T+1, B) int64 (AtariNet input)

    @property
    def unroll_length(self) -> int:
        return self.observation.shape[0] - 1

    @property
    def batch_size(self) -> int:
        return self.observation.shape[1]

    @property
    def num_actions(self) -> int:
        return self.policy_logits.shape[-1]

    def to(self, device, non_blocking: bool = False) -> "TrainingBatch":
        kw = {}
        for f in fields(self):
            v = getattr(self, f.name)
            kw[f.name] = v.to(device, non_blocking=non_blocking) if v is not None else None
        return TrainingBatch(**kw)

    def shard(self, rank: int, world: int) -> "TrainingBatch":
        """Contiguous column block [rank*B/world, (rank+1)*B/world) of the batch axis."""
        b = self.batch_size
        if b % world:
            raise SchemaError(f"batch {b} not divisible by world size {world}")
        lo, hi = rank * b // world, (rank + 1) * b // world
        kw = {}
        for f in fields(self):
            v = getattr(self, f.name)
            if v is None:
                kw[f.name] = None
            elif f.name == "model_versions":
                kw[f.name] = v[lo:hi]
            else:
                kw[f.name] = v[:, lo:hi]
        return TrainingBatch(**kw)


def validate_batch(batch) -> None:
    """Shape / dtype checks of rollout.py:160-183 (raises SchemaError naming the field)."""
    obs = batch.observation
    if obs.ndim < 2:
        raise SchemaError(f"observation: dims {tuple(obs.shape)}, need at least (T+1, B)")
    t1, b = obs.shape[0], obs.shape[1]
    if t1 < 2:
        raise SchemaError(f"observation: dims {tuple(obs.shape)}, need T+1 >= 2 rows")
    for name in ("reward", "done", "baseline", "action"):
        arr = getattr(batch, name)
        if tuple(arr.shape) != (t1, b):
            raise SchemaError(f"{name}: dims {tuple(arr.shape)}, expected ({t1}, {b})")
    logits = batch.policy_logits
    if logits.ndim != 3 or tuple(logits.shape[:2]) != (t1, b):
        raise SchemaError(f"policy_logits: dims {tuple(logits.shape)}, expected ({t1}, {b}, A)")
    if tuple(batch.model_versions.shape) != (b,):
        raise SchemaError(f"model_versions: dims {tuple(batch.model_versions.shape)}, expected ({b},)")
    if batch.done.dtype not in (torch.bool,) and str(batch.done.dtype) != "bool":
        raise SchemaError(f"done: dtype {batch.done.dtype}, expected bool")


# ---------------------------------------------------------------------------
# Frame-stack dedup.  Upstream TorchBeast feeds AtariNet frames made by
# the FrameStack(k=4) wrapper: channel c of the frame at step t is the raw plane of
# step t-3+c, and on an episode reset (done[t]) the stack is k copies of the reset
# plane.  The reference ships (T+1)*B*4 planes per batch (np.stack at enqueue,
# rollout.py:116-144); a plane store ships each raw plane once, (T+4)*B planes: row j
# of the store is step j-3 (rows 0..2 are the 3 planes before the unroll).
# ---------------------------------------------------------------------------
HISTORY = 3


def frame_stack_index(done: torch.Tensor) -> torch.Tensor:
    """done (T+1, B) bool -> plane index (T+1, B, 4) int32 into a (T+4, B) plane store
    flattened as row * B + b (FrameStack semantics, resets replicate the reset plane)."""
    if done.dim() != 2:
        raise SchemaError(f"done: dims {tuple(done.shape)}, expected (T+1, B)")
    t1, b = done.shape
    d = done.to("cpu", torch.bool)
    t = torch.arange(t1).view(t1, 1)
    # plane row of the latest reset at or before t (or -1): running max of (t+3) * done
    start = torch.where(d, t + HISTORY, torch.full_like(t, -1).expand(t1, b))
    start = torch.cummax(start, dim=0).values
    rows = t.view(t1, 1, 1) + torch.arange(4).view(1, 1, 4)             # t + c
    rows = torch.maximum(rows.expand(t1, b, 4), start.view(t1, b, 1))
    return (rows * b + torch.arange(b).view(1, b, 1)).to(torch.int32).to(done.device)


def stack_frames(planes: torch.Tensor, index: torch.Tensor) -> torch.Tensor:
    """Plane store (P, 84, 84) or (T+4, B, 84, 84) + index (T+1, B, 4) -> frames (T+1, B, 4, 84, 84)."""
    flat = planes.reshape(-1, *planes.shape[-2:])
    return flat[index.reshape(-1).long()].reshape(*index.shape, *planes.shape[-2:])


def dedup_frames(frames: torch.Tensor, done: torch.Tensor, check: bool = True):
    """Stacked frames (T+1, B, 4, 84, 84) u8 + done (T+1, B) -> (planes (T+4, B, 84, 84),
    index (T+1, B, 4) int32).  check=True verifies the batch really is FrameStack data
    (stack_frames(planes, index) == frames) and raises SchemaError otherwise."""
    if frames.dim() != 5 or frames.shape[2] != 4:
        raise SchemaError(f"frame: dims {tuple(frames.shape)}, expected (T+1, B, 4, H, W)")
    t1, b = frames.shape[:2]
    planes = torch.empty((t1 + HISTORY, b, *frames.shape[-2:]), dtype=frames.dtype, device=frames.device)
    planes[:HISTORY] = frames[0, :, :HISTORY].transpose(0, 1)
    planes[HISTORY:] = frames[:, :, 3]
    index = frame_stack_index(done)
    if check and not torch.equal(stack_frames(planes, index.to(frames.device)), frames):
        raise SchemaError("frame: batch is not FrameStack(4) data; cannot deduplicate")
    return planes, index.to(frames.device)
