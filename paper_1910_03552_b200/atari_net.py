"""AtariNet (upstream TorchBeast monobeast.AtariNet) on the sm_100a kernels.

Drop-in for `AtariNet(observation_shape, num_actions, use_lstm=False)`:
same submodule names and state_dict keys / shapes / layouts as upstream
(conv1, conv2, conv3, fc, policy, baseline), same `forward(inputs,
core_state) -> (dict(policy_logits, baseline, action), core_state)` and
`initial_state(batch_size)`.  The reference network seam it replaces is
beastpipe mlp_forward / mlp_backward (model.py:126-203).

Every dense contraction runs on tcgen05 tensor cores through the C ABI
(bp_atari_forward / bp_atari_backward; bf16 operands, f32 accumulation).
Parameters are views into one flat f32 buffer (`flat_params`), gradients
into `flat_grads`, so the fused optimiser and the NCCL all-reduce see one
contiguous buffer each.  The conv / fc weight Parameters hold the kernels'
[Cout][K] GEMM layout (`torch_to_gemm`); `state_dict()` / `load_state_dict()`
convert to / from the upstream torch layouts, so checkpoints interoperate.

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


def torch_to_gemm(name: str, w: torch.Tensor) -> torch.Tensor:
    """Upstream torch weight layout -> the [Cout][K] GEMM layout of the kernels
    (K = (tap, input channel), include/beast_b200.h)."""
    if name == "conv1.weight":  # [32][4][8][8], ky = 4dy+ry, kx = 4dx+rx
        return w.reshape(32, 4, 2, 4, 2, 4).permute(0, 2, 4, 1, 3, 5).reshape(32, 256)
    if name == "conv2.weight":  # [64][32][4][4], ky = 2dy+py, kx = 2dx+px
        return w.reshape(64, 32, 2, 2, 2, 2).permute(0, 2, 4, 3, 5, 1).reshape(64, 512)
    if name == "conv3.weight":  # [64][64][3][3]
        return w.permute(0, 2, 3, 1).reshape(64, 576)
    if name == "fc.weight":  # [512][3136], torch feature c*49 + pos -> k = pos*64 + c
        return w.reshape(512, 64, 49).permute(0, 2, 1).reshape(512, 3136)
    return w


def gemm_to_torch(name: str, w: torch.Tensor) -> torch.Tensor:
    if name == "conv1.weight":
        return w.reshape(32, 2, 2, 4, 4, 4).permute(0, 3, 1, 4, 2, 5).reshape(32, 4, 8, 8)
    if name == "conv2.weight":
        return w.reshape(64, 2, 2, 2, 2, 32).permute(0, 5, 1, 3, 2, 4).reshape(64, 32, 4, 4)
    if name == "conv3.weight":
        return w.reshape(64, 3, 3, 64).permute(0, 3, 1, 2)
    if name == "fc.weight":
        return w.reshape(512, 49, 64).permute(0, 2, 1).reshape(512, 3136)
    return w


GEMM_WEIGHTS = ("conv1.weight", "conv2.weight", "conv3.weight", "fc.weight")


class _LstmBuffers:
    """Caller-owned device buffers of the C ABI struct BpLstmCore, for n <= capacity rows."""

    def __init__(self, num_actions: int, capacity: int, device):
        H = 513 + num_actions
        G4 = (4 * H + 127) // 128 * 128
        n, d, bf, f32 = capacity, device, torch.bfloat16, torch.float32
        self.hidden = H
        self.t = dict(
            wih=torch.empty(2, G4, 576, dtype=bf, device=d),
            gx=torch.empty(n, G4, dtype=f32, device=d),
            gates=torch.empty(2, n, 8 * H, dtype=f32, device=d),
            cseq=torch.empty(2, n, H, dtype=f32, device=d),
            # padding columns of these are never written: zero once
            hprev=torch.zeros(2, n, 576, dtype=bf, device=d),
            out=torch.zeros(2, n, 576, dtype=bf, device=d),
            hx=torch.empty(2, H, 32, dtype=f32, device=d),
            part=torch.empty(N.lib().bp_lstm_partial_floats(H), dtype=f32, device=d),
            dgates=torch.zeros(2, n, G4, dtype=bf, device=d),  # per layer
            dh=torch.empty(n, 576, dtype=f32, device=d),
            dx=torch.empty(n, 576, dtype=f32, device=d),
            wpart=torch.empty(2, 2, G4, 576, dtype=f32, device=d),  # W_ih / W_hh x split-K parts
        )
        names = ("wih", "gx", "gates", "cseq", "hprev", "out", "hx", "part", "dgates", "dh", "dx", "wpart")
        self.struct = N.BpLstmCore(H, capacity, *[self.t[k].data_ptr() for k in names])
        self.ref = C.byref(self.struct)


class _Buffers:
    """Caller-owned device buffers of the C ABI struct BpAtariNet, for n <= capacity."""

    def __init__(self, num_actions: int, capacity: int, nparams: int, device, use_lstm: bool = False):
        self.capacity = capacity
        d = device
        bf = torch.bfloat16

        def z(*shape, dtype=bf):
            return torch.zeros(*shape, dtype=dtype, device=d)

        def e(*shape, dtype=bf):
            return torch.empty(*shape, dtype=dtype, device=d)

        n = capacity
        self.t = dict(
            wbf=e(nparams), whf=e(32, 576),
            x0=e(n * 441, 64), x1=e(n * 100, 128), x2=e(n * 81, 64), x3=e(n, 3136), core=e(n, 576),
            m1=e(n * 400, dtype=torch.int32), m2=e(n * 162, dtype=torch.int32),
            m3=e(n * 98, dtype=torch.int32), mc=e(n * 18, dtype=torch.int32),
            g=e(n, 64), d_fc=e(n, 512),
            # grid padding rows of these are never written: zero once
            d_pre3=z(n * 81, 64), d_pre2=z(n * 100, 64), d_pre1=z(n * 441, 32),
        )
        ws_bytes = N.lib().bp_atari_workspace_bytes(num_actions, capacity)
        self.t["ws"] = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=d)
        names = ("wbf", "whf", "x0", "x1", "x2", "x3", "core", "m1", "m2", "m3", "mc", "g", "d_fc",
                 "d_pre3", "d_pre2", "d_pre1", "ws")
        # conv1's forward converts the u8 frames on chip and writes the bf16 X0 grid as a side
        # output for the weight gradient (flags=BP_NET_NO_X0 would convert again in the
        # backward instead; measured slower)
        self.struct = N.BpAtariNet(num_actions, capacity, int(use_lstm),
                                   *[self.t[k].data_ptr() for k in names], ws_bytes, 0)
        self.ref = C.byref(self.struct)
        self.lstm = _LstmBuffers(num_actions, capacity, device) if use_lstm else None


def _check_fwd_gen(ctx):
    if ctx.net._fwd_gen != ctx.fwd_gen:
        raise RuntimeError("AtariNet: backward after another forward on the same module; the fused "
                           "kernels keep only the last forward's activations -- call backward "
                           "before the next forward (or use a second AtariNet)")


class _AtariFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, net, frames, reward, last_action, *params):
        logits, baseline = net._forward_kernels(frames, reward, last_action, repack=True)
        ctx.net = net
        ctx.fwd_gen = net._fwd_gen
        ctx.save_for_backward(reward, last_action)
        return logits, baseline

    @staticmethod
    def backward(ctx, d_logits, d_baseline):
        net = ctx.net
        _check_fwd_gen(ctx)
        reward, last_action = ctx.saved_tensors
        grads = torch.empty_like(net.flat_params)
        net._backward_kernels(d_logits, d_baseline, reward, last_action, grads)
        views = net._split(grads)
        return (None, None, None, None, *views)


class _AtariLstmFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, net, frames, reward, last_action, done, h0, c0, T1, B, *params):
        lstm = dict(T1=T1, B=B, done=done, h0=h0, c0=c0)
        logits, baseline = net._forward_kernels(frames, reward, last_action, repack=True, lstm=lstm)
        ctx.net = net
        ctx.fwd_gen = net._fwd_gen
        ctx.dims = (T1, B)
        ctx.save_for_backward(reward, last_action, done, c0)
        ctx.mark_non_differentiable(lstm["hN"], lstm["cN"])
        return logits, baseline, lstm["hN"], lstm["cN"]

    @staticmethod
    def backward(ctx, d_logits, d_baseline, d_hN, d_cN):
        net = ctx.net
        _check_fwd_gen(ctx)
        reward, last_action, done, c0 = ctx.saved_tensors
        T1, B = ctx.dims
        grads = torch.empty_like(net.flat_params)
        net._backward_kernels(d_logits, d_baseline, reward, last_action, grads,
                              lstm=dict(T1=T1, B=B, done=done, c0=c0))
        views = net._split(grads)
        return (None,) * 9 + tuple(views)


class AtariNet(nn.Module):
    def __init__(self, observation_shape=OBS_SHAPE, num_actions=6, use_lstm=False, device=None):
        super().__init__()
        if tuple(observation_shape) != OBS_SHAPE:
            raise DimensionError(f"AtariNet kernels take {OBS_SHAPE} u8 frames, got {observation_shape}")
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
        if use_lstm:  # upstream: nn.LSTM(core_output_size, core_output_size, 2)
            self.core = nn.LSTM(core, core, 2)
        self.policy = nn.Linear(core, num_actions)
        self.baseline = nn.Linear(core, 1)
        self.to(device)
        # conv / fc weights live in the kernels' [Cout][K] GEMM layout; state_dict() and
        # load_state_dict() convert to / from the upstream torch layouts (hooks below)
        with torch.no_grad():
            for name in GEMM_WEIGHTS:
                mod = getattr(self, name.split(".")[0])
                mod.weight = nn.Parameter(torch_to_gemm(name, mod.weight.detach()).contiguous())
        count = N.lib().bp_atari_param_count(num_actions, int(use_lstm))
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
        self._register_state_dict_hook(AtariNet._to_torch_layout)
        self.register_load_state_dict_pre_hook(AtariNet._from_torch_layout)
        self._bufs: _Buffers | None = None
        # bumped whenever the activation / workspace buffers are reallocated: CUDA graphs that
        # captured the old addresses must be dropped (FusedLearner checks it)
        self.buffer_generation = 0
        # bumped by every forward: an autograd backward must follow ITS forward (the kernels
        # read the activations the forward left in the shared buffers)
        self._fwd_gen = 0
        self._logits = None
        self._baseline = None
        self.sample_seed = 0x5EED
        self._calls = 0
        self.mirror_fresh = False  # bf16 operand mirror (wbf) up to date with flat_params

    @staticmethod
    def _to_torch_layout(module, state_dict, prefix, local_metadata):
        for name in GEMM_WEIGHTS:
            k = prefix + name
            if k in state_dict:
                state_dict[k] = gemm_to_torch(name, state_dict[k]).contiguous()
        return state_dict

    @staticmethod
    def _from_torch_layout(module, state_dict, prefix, local_metadata, strict, missing_keys,
                           unexpected_keys, error_msgs):
        # state_dicts are always in the upstream torch layout (state_dict() emits it too)
        for name in GEMM_WEIGHTS:
            k = prefix + name
            if k in state_dict:
                state_dict[k] = torch_to_gemm(name, state_dict[k]).contiguous()
        module.mirror_fresh = False

    # ------------------------------------------------------------------ helpers
    def _split(self, flat):
        return [flat[o:o + n].view(s) for o, n, s in self._shapes]

    def torch_layout_grads(self, flat):
        """{name: gradient in the upstream torch layout} of a flat gradient buffer."""
        names = [k for k, _ in self.named_parameters()]
        return {k: gemm_to_torch(k, v) for k, v in zip(names, self._split(flat))}

    def buffers_for(self, n: int) -> _Buffers:
        if self._bufs is None or self._bufs.capacity < n:
            self._bufs = _Buffers(self.num_actions, n, self.flat_params.numel(), self.flat_params.device,
                                  self.use_lstm)
            self._logits = torch.empty(n, self.num_actions, device=self.flat_params.device)
            self._baseline = torch.empty(n, device=self.flat_params.device)
            self.mirror_fresh = False
            self.buffer_generation += 1
        return self._bufs

    @property
    def flat_bf16(self) -> torch.Tensor:
        """bf16 mirror of flat_params: the GEMM operand the kernels read."""
        return self.buffers_for(1).t["wbf"]

    def pack_weights(self) -> None:
        """Refresh the bf16 operand mirror from the f32 parameters (one cast kernel)."""
        b = self.buffers_for(1)
        N.check(N.lib().bp_atari_pack_weights(b.ref, N.ptr(self.flat_params),
                                              N.stream_handle(self.flat_params.device)),
                "bp_atari_pack_weights")
        self.mirror_fresh = True
        self._packed_version = self.flat_params._version

    def mirror_stale(self) -> bool:
        """True if the bf16 mirror may lag the f32 parameters: never packed, or the
        parameters were modified in place through torch since (version counter)."""
        return (not self.mirror_fresh or
                getattr(self, "_packed_version", None) != self.flat_params._version)

    def _forward_kernels(self, frames, reward, last_action, logits=None, baseline=None,
                         repack: bool | None = None, lstm: dict | None = None, plane_index=None,
                         keep_x0: bool = True, actions=None, seed: int = 0, greedy: bool = False,
                         seed_state=None):
        """frames u8 (n,4,84,84), reward f32 (n,), last_action i64 (n,) -> logits, baseline.

        Frame-stack dedup: with plane_index (n,4) int32, `frames` is a plane store
        (P,84,84) u8 and channel c of frame i is frames[plane_index[i, c]]
        (rollout.frame_stack_index builds the upstream FrameStack indexing).
        repack=None packs the bf16 mirror only when stale; False trusts its version (the fused
        optimiser step keeps it fresh) but still packs a never-packed buffer set; True always packs.  LSTM nets take
        lstm=dict(T1, B, done u8 (n,), h0, c0 (2,B,H) f32[, hN, cN]); the final state
        is returned in lstm["hN"], lstm["cN"].  keep_x0=False (inference without a backward)
        skips conv1's X0 side output.  actions (n,) int64: the heads epilogue also draws the
        actions (Gumbel-max with `seed`, or argmax when greedy; same draws as sample())."""
        if plane_index is not None:
            if plane_index.dtype != torch.int32 or plane_index.shape[-1] != 4:
                raise DimensionError("plane_index must be int32 (n, 4)")
            if frames.dim() < 3 or tuple(frames.shape[-2:]) != OBS_SHAPE[1:]:
                raise DimensionError(f"plane store must be (..., 84, 84), got {tuple(frames.shape)}")
            frames = frames.reshape(-1, *OBS_SHAPE[1:])
            plane_index = plane_index.reshape(-1, 4)
            n, num_planes = plane_index.shape[0], frames.shape[0]
        else:
            n = frames.shape[0]
        b = self.buffers_for(n)
        # (a freshly (re)allocated buffer set has no mirror yet: packed even with repack=False)
        if repack or not self.mirror_fresh or (repack is None and self.mirror_stale()):
            self.pack_weights()
        if logits is None:
            logits = torch.empty(n, self.num_actions, device=frames.device)
        if baseline is None:
            baseline = torch.empty(n, device=frames.device)
        stream = N.stream_handle(frames.device)
        b.struct.flags = 0 if (keep_x0 or self.use_lstm) else N.BP_NET_NO_X0
        if self.use_lstm:
            if lstm is None:
                raise DimensionError("LSTM AtariNet forward needs done / core_state (lstm=...)")
            T1, B = lstm["T1"], lstm["B"]
            if T1 * B != n:
                raise DimensionError(f"lstm dims {T1}x{B} != {n} frames")
            shape = (2, B, self.core_hidden)
            for k in ("hN", "cN"):
                if lstm.get(k) is None:
                    lstm[k] = torch.empty(shape, device=frames.device)
            tail = (N.ptr(reward), N.ptr(last_action), N.ptr(lstm["done"]), N.ptr(self.flat_params),
                    N.ptr(lstm["h0"]), N.ptr(lstm["c0"]), N.ptr(logits), N.ptr(baseline),
                    N.ptr(lstm["hN"]), N.ptr(lstm["cN"]), stream)
            if actions is not None:
                idx = N.ptr(plane_index) if plane_index is not None else None
                np_ = num_planes if plane_index is not None else 0
                N.check(N.lib().bp_atari_lstm_forward_sample(
                    b.ref, b.lstm.ref, T1, B, N.ptr(frames), idx, np_, N.ptr(reward), N.ptr(last_action),
                    N.ptr(lstm["done"]), N.ptr(self.flat_params), N.ptr(lstm["h0"]), N.ptr(lstm["c0"]),
                    seed, N.ptr(seed_state) if seed_state is not None else None, int(greedy), N.ptr(logits),
                    N.ptr(baseline), N.ptr(lstm["hN"]), N.ptr(lstm["cN"]),
                    N.ptr(actions), stream), "bp_atari_lstm_forward_sample")
            elif plane_index is not None:
                N.check(N.lib().bp_atari_lstm_forward_planes(
                    b.ref, b.lstm.ref, T1, B, N.ptr(frames), N.ptr(plane_index), num_planes, *tail),
                    "bp_atari_lstm_forward_planes")
            else:
                N.check(N.lib().bp_atari_lstm_forward(b.ref, b.lstm.ref, T1, B, N.ptr(frames), *tail),
                        "bp_atari_lstm_forward")
        else:
            tail = (N.ptr(reward), N.ptr(last_action), N.ptr(self.flat_params), N.ptr(logits),
                    N.ptr(baseline), stream)
            if actions is not None:
                idx = N.ptr(plane_index) if plane_index is not None else None
                np_ = num_planes if plane_index is not None else 0
                N.check(N.lib().bp_atari_forward_sample(
                    b.ref, n, N.ptr(frames), idx, np_, N.ptr(reward), N.ptr(last_action),
                    N.ptr(self.flat_params), seed, N.ptr(seed_state) if seed_state is not None else None,
                    int(greedy), N.ptr(logits), N.ptr(baseline),
                    N.ptr(actions), stream), "bp_atari_forward_sample")
            elif plane_index is not None:
                N.check(N.lib().bp_atari_forward_planes(b.ref, n, N.ptr(frames), N.ptr(plane_index),
                                                        num_planes, *tail), "bp_atari_forward_planes")
            else:
                N.check(N.lib().bp_atari_forward(b.ref, n, N.ptr(frames), *tail), "bp_atari_forward")
        self._last_n = n
        self._fwd_gen += 1
        # frame source of this forward, for the backward (kept alive until the next forward)
        self._frame_src = (frames, plane_index, num_planes if plane_index is not None else 0)
        return logits, baseline

    def _backward_kernels(self, d_logits, d_baseline, reward, last_action, grads, lstm: dict | None = None):
        n = d_logits.shape[0]
        b = self.buffers_for(n)
        d_logits = d_logits.contiguous().float()
        d_baseline = d_baseline.contiguous().float()
        stream = N.stream_handle(d_logits.device)
        if self.use_lstm:
            N.check(N.lib().bp_atari_lstm_backward(
                b.ref, b.lstm.ref, lstm["T1"], lstm["B"], N.ptr(d_logits), N.ptr(d_baseline),
                N.ptr(lstm["done"]), N.ptr(self.flat_params), N.ptr(lstm["c0"]), N.ptr(grads), stream),
                "bp_atari_lstm_backward")
            return
        src = getattr(self, "_frame_src", None)
        if src is None:
            raise DimensionError("backward without a preceding forward")
        frames, plane_index, num_planes = src
        N.check(N.lib().bp_atari_backward_frames(b.ref, n, N.ptr(frames), N.ptr(plane_index), num_planes,
                                                 N.ptr(d_logits), N.ptr(d_baseline), N.ptr(grads), stream),
                "bp_atari_backward_frames")

    def next_sample_seed(self) -> int:
        """Per-call 64-bit Philox key of the action sampler (sample_seed, call counter)."""
        self._calls += 1
        return (self.sample_seed * 0x9E3779B97F4A7C15 + self._calls) & 0xFFFFFFFFFFFFFFFF

    def sample(self, logits: torch.Tensor, greedy: bool, seed: int | None = None) -> torch.Tensor:
        """Gumbel-max categorical sample (training) or argmax (eval), one kernel."""
        n = logits.shape[0]
        out = torch.empty(n, dtype=torch.int64, device=logits.device)
        if seed is None:
            seed = self.next_sample_seed()
        N.check(N.lib().bp_sample_actions_f32(N.ptr(logits), n, self.num_actions, seed, int(greedy),
                                              N.ptr(out), N.stream_handle(logits.device)),
                "bp_sample_actions_f32")
        return out

    # ------------------------------------------------------------------ upstream API
    @property
    def core_hidden(self) -> int:
        return self.fc.out_features + self.num_actions + 1

    def initial_state(self, batch_size):
        if not self.use_lstm:
            return tuple()
        dev = self.flat_params.device
        return tuple(torch.zeros(2, batch_size, self.core_hidden, device=dev) for _ in range(2))

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
        state = tuple()
        if self.use_lstm:
            done = inputs["done"].reshape(T * B).contiguous()
            done = done.view(torch.uint8) if done.dtype == torch.bool else (done != 0).to(torch.uint8)
            if len(core_state) != 2:
                raise DimensionError("LSTM core_state must be (h, c), each (2, B, hidden)")
            h0, c0 = (s.detach().float().contiguous() for s in core_state)
            if tuple(h0.shape) != (2, B, self.core_hidden) or tuple(c0.shape) != (2, B, self.core_hidden):
                raise DimensionError(f"core_state shapes {tuple(h0.shape)}, expected (2, {B}, {self.core_hidden})")
            if torch.is_grad_enabled():
                logits, baseline, hN, cN = _AtariLstmFunction.apply(
                    self, frames, reward, last_action, done, h0, c0, T, B, *self.parameters())
            else:  # inference: the heads epilogue samples the actions
                lstm = dict(T1=T, B=B, done=done, h0=h0, c0=c0)
                action = torch.empty(T * B, dtype=torch.int64, device=frames.device)
                logits, baseline = self._forward_kernels(frames, reward, last_action, lstm=lstm, actions=action,
                                                         seed=self.next_sample_seed(), greedy=not self.training)
                hN, cN = lstm["hN"], lstm["cN"]
            state = (hN, cN)
        elif torch.is_grad_enabled():
            logits, baseline = _AtariFunction.apply(self, frames, reward, last_action,
                                                    *self.parameters())
        else:  # inference: no backward follows (conv1 skips the X0 side output), fused sampling
            action = torch.empty(T * B, dtype=torch.int64, device=frames.device)
            logits, baseline = self._forward_kernels(frames, reward, last_action, keep_x0=False, actions=action,
                                                     seed=self.next_sample_seed(), greedy=not self.training)
        if torch.is_grad_enabled():
            action = self.sample(logits.detach(), greedy=not self.training)
        return (dict(policy_logits=logits.view(T, B, self.num_actions), baseline=baseline.view(T, B),
                     action=action.view(T, B)), state)
