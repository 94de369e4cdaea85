"""AtariNet (upstream TorchBeast monobeast.AtariNet) on the sm_100a kernels.

Drop-in for `AtariNet(observation_shape, num_actions, use_lstm=False)`:
same submodule names / parameter shapes / state_dict keys as upstream
(conv1, conv2, conv3, fc, policy, baseline), same `forward(inputs,
core_state) -> (dict(policy_logits, baseline, action), core_state)` and
`initial_state(batch_size)`.  The reference network seam it replaces is
beastpipe mlp_forward / mlp_backward (model.py:126-203).

Every dense contraction runs on tcgen05 tensor cores through the C ABI
(bp_atari_forward / bp_atari_backward; bf16 operands, f32 accumulation).
Parameters are views into one flat f32 buffer (`flat_params`), gradients
into `flat_grads`, so the fused optimiser and the NCCL all-reduce see one
contiguous buffer each.

Autograd: `forward` is an autograd.Function whose backward calls the fused
backward kernels, so `total_loss.backward()` works as upstream.  `learn()`
bypasses autograd and drives the kernels directly.
"""
from __future__ import annotations

import ctypes as C

import torch
from torch import nn

from . import _native as N
from .errors import DimensionError

OBS_SHAPE = (4, 84, 84)


class _Buffers:
    """Caller-owned device buffers of the C ABI struct BpAtariNet, for n <= capacity."""

    def __init__(self, num_actions: int, capacity: int, device):
        self.capacity = capacity
        d = device
        bf = torch.bfloat16

        def z(*shape, dtype=bf):
            return torch.zeros(*shape, dtype=dtype, device=d)

        def e(*shape, dtype=bf):
            return torch.empty(*shape, dtype=dtype, device=d)

        n = capacity
        self.t = dict(
            w1f=e(32, 256), w2f=e(64, 512), w3f=e(64, 576), wfcf=e(512, 3136), whf=e(32, 512),
            w2d=e(128, 256), w3d=e(64, 576), wfcd=e(3136, 512), whd=e(512, 64),
            x0=e(n * 441, 64), x1=e(n * 100, 128), x2=e(n * 81, 64), x3=e(n, 3136), h=e(n, 512),
            g=e(n, 64), d_fc=e(n, 512),
            # grid padding rows of these are never written: zero once
            d_pre3=z(n * 81, 64), d_pre2=z(n * 100, 64), d_pre1=z(n * 441, 32),
        )
        ws_bytes = N.lib().bp_atari_workspace_bytes(num_actions, capacity)
        self.t["ws"] = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=d)
        self.struct = N.BpAtariNet(num_actions, capacity, *[self.t[k].data_ptr() for k in (
            "w1f", "w2f", "w3f", "wfcf", "whf", "w2d", "w3d", "wfcd", "whd", "x0", "x1", "x2",
            "x3", "h", "g", "d_fc", "d_pre3", "d_pre2", "d_pre1", "ws")], ws_bytes)
        self.ref = C.byref(self.struct)


class _AtariFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, net, frames, reward, last_action, *params):
        logits, baseline = net._forward_kernels(frames, reward, last_action)
        ctx.net = net
        ctx.save_for_backward(reward, last_action)
        return logits, baseline

    @staticmethod
    def backward(ctx, d_logits, d_baseline):
        net = ctx.net
        reward, last_action = ctx.saved_tensors
        grads = torch.empty_like(net.flat_params)
        net._backward_kernels(d_logits, d_baseline, reward, last_action, grads)
        views = net._split(grads)
        return (None, None, None, None, *views)


class AtariNet(nn.Module):
    def __init__(self, observation_shape=OBS_SHAPE, num_actions=6, use_lstm=False, device=None):
        super().__init__()
        if tuple(observation_shape) != OBS_SHAPE:
            raise DimensionError(f"AtariNet kernels take {OBS_SHAPE} u8 frames, got {observation_shape}")
        if use_lstm:
            raise NotImplementedError("LSTM core: see DESIGN.md (not in this build yet)")
        if not 1 <= num_actions <= 31:
            raise DimensionError("num_actions must be in [1, 31]")
        self.observation_shape = tuple(observation_shape)
        self.num_actions = num_actions
        self.use_lstm = use_lstm
        device = torch.device(device or "cuda")
        # upstream module structure (default torch init), then re-home into flat buffers
        self.conv1 = nn.Conv2d(observation_shape[0], 32, kernel_size=8, stride=4)
        self.conv2 = nn.Conv2d(32, 64, kernel_size=4, stride=2)
        self.conv3 = nn.Conv2d(64, 64, kernel_size=3, stride=1)
        self.fc = nn.Linear(3136, 512)
        core = self.fc.out_features + num_actions + 1
        self.policy = nn.Linear(core, num_actions)
        self.baseline = nn.Linear(core, 1)
        self.to(device)
        count = N.lib().bp_atari_param_count(num_actions, 0)
        params = list(self.parameters())
        assert sum(p.numel() for p in params) == count
        self.flat_params = torch.empty(count, dtype=torch.float32, device=device)
        self.flat_grads = torch.zeros(count, dtype=torch.float32, device=device)
        off = 0
        self._shapes = []
        for p in params:
            n = p.numel()
            self.flat_params[off:off + n].copy_(p.detach().reshape(-1))
            p.data = self.flat_params[off:off + n].view_as(p)
            p.grad = self.flat_grads[off:off + n].view_as(p)
            self._shapes.append((off, n, p.shape))
            off += n
        self._bufs: _Buffers | None = None
        self._logits = None
        self._baseline = None
        self.sample_seed = 0x5EED
        self._calls = 0

    # ------------------------------------------------------------------ helpers
    def _split(self, flat):
        return [flat[o:o + n].view(s) for o, n, s in self._shapes]

    def buffers_for(self, n: int) -> _Buffers:
        if self._bufs is None or self._bufs.capacity < n:
            self._bufs = _Buffers(self.num_actions, n, self.flat_params.device)
            self._logits = torch.empty(n, self.num_actions, device=self.flat_params.device)
            self._baseline = torch.empty(n, device=self.flat_params.device)
        return self._bufs

    def pack_weights(self) -> None:
        """bf16 GEMM operand copies of the current f32 parameters (one kernel)."""
        b = self.buffers_for(1)
        N.check(N.lib().bp_atari_pack_weights(b.ref, N.ptr(self.flat_params),
                                              N.stream_handle(self.flat_params.device)),
                "bp_atari_pack_weights")

    def _forward_kernels(self, frames, reward, last_action, logits=None, baseline=None):
        """frames u8 (n,4,84,84), reward f32 (n,), last_action i64 (n,) -> logits, baseline."""
        n = frames.shape[0]
        b = self.buffers_for(n)
        self.pack_weights()
        if logits is None:
            logits = torch.empty(n, self.num_actions, device=frames.device)
        if baseline is None:
            baseline = torch.empty(n, device=frames.device)
        N.check(N.lib().bp_atari_forward(b.ref, n, N.ptr(frames), N.ptr(reward), N.ptr(last_action),
                                         N.ptr(self.flat_params), N.ptr(logits), N.ptr(baseline),
                                         N.stream_handle(frames.device)), "bp_atari_forward")
        self._last_n = n
        return logits, baseline

    def _backward_kernels(self, d_logits, d_baseline, reward, last_action, grads):
        n = d_logits.shape[0]
        b = self.buffers_for(n)
        d_logits = d_logits.contiguous().float()
        d_baseline = d_baseline.contiguous().float()
        N.check(N.lib().bp_atari_backward(b.ref, n, N.ptr(d_logits), N.ptr(d_baseline), N.ptr(reward),
                                          N.ptr(last_action), N.ptr(grads),
                                          N.stream_handle(d_logits.device)), "bp_atari_backward")

    def sample(self, logits: torch.Tensor, greedy: bool) -> torch.Tensor:
        """Gumbel-max categorical sample (training) or argmax (eval), one kernel."""
        n = logits.shape[0]
        out = torch.empty(n, dtype=torch.int64, device=logits.device)
        self._calls += 1
        seed = (self.sample_seed * 0x9E3779B97F4A7C15 + self._calls) & 0xFFFFFFFFFFFFFFFF
        N.check(N.lib().bp_sample_actions_f32(N.ptr(logits), n, self.num_actions, seed, int(greedy),
                                              N.ptr(out), N.stream_handle(logits.device)),
                "bp_sample_actions_f32")
        return out

    # ------------------------------------------------------------------ upstream API
    def initial_state(self, batch_size):
        return tuple()

    def forward(self, inputs, core_state=()):
        x = inputs["frame"]
        T, B = x.shape[0], x.shape[1]
        if tuple(x.shape[2:]) != self.observation_shape:
            raise DimensionError(f"frame shape {tuple(x.shape)}, expected (T, B, *{self.observation_shape})")
        frames = x.reshape(T * B, *self.observation_shape)
        if frames.dtype != torch.uint8:
            raise DimensionError("frames must be uint8 (the kernels apply the /255 scale)")
        frames = frames.contiguous()
        reward = inputs["reward"].reshape(T * B).float().contiguous()
        last_action = inputs["last_action"].reshape(T * B).to(torch.int64).contiguous()
        if torch.is_grad_enabled():
            logits, baseline = _AtariFunction.apply(self, frames, reward, last_action,
                                                    *self.parameters())
        else:
            logits, baseline = self._forward_kernels(frames, reward, last_action)
        action = self.sample(logits.detach(), greedy=not self.training)
        return (dict(policy_logits=logits.view(T, B, self.num_actions), baseline=baseline.view(T, B),
                     action=action.view(T, B)), tuple())
