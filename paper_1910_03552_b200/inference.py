"""Actor inference: the dynamic-batching inference loop body on the fused kernels.

Replaces the body of beastpipe `LearnerContext._inference_loop` (pipeline.py:609-634:
`mlp_forward(params, obs)` + `sample_actions(logits, rng)` per dynamic batch of k
observations handed over by `DynamicBatcher` (queues.py:190-296)) and upstream
PolyBeast's `inference()` (`model(batch, core_state)` under no_grad).

One call is one AtariNet forward over the k observations whose heads-GEMM epilogue
also draws the actions (Gumbel-max, Philox keyed by (seed, row, column);
bp_atari_forward_sample / bp_atari_lstm_forward_sample).  Two modes:

  eager   any k: the forward is enqueued directly (one C call, ~6 kernels);
  graphs  k is rounded up to a captured bucket (e.g. 1, 32, 256, 1024): the inputs are
          copied into the bucket's static buffers and the captured forward replays.
          The sampling key is device-resident and advances on every replay, so
          replays draw fresh actions without host involvement.

Outputs follow the reference's inference handle: action (1, k) int64,
policy_logits (1, k, A) f32, baseline (1, k) f32, model_version (1, k) int64; with
an LSTM core the new core_state is returned as well (T = 1 actor step).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as N

from .errors import DimensionError
from ._tensors import graph_capture


class ActorInference:
    def __init__(self, model, graph_buckets=(), greedy: bool = False, seed: int = 0x5EED):
        self.model = model
        self.greedy = greedy
        self.version = 0
        dev = model.flat_params.device
        self.device = dev
        self.buckets = tuple(sorted(int(b) for b in graph_buckets))
        # device-resident sampling key of the graph replays (advanced by every replay)
        self.seed_state = torch.tensor([seed & 0x7FFFFFFFFFFFFFFF], dtype=torch.int64, device=dev)
        self._graphs: dict[int, tuple] = {}
        self._mv: dict[int, tuple] = {}  # k -> (version, model_version tensor (1, k))
        if self.buckets:
            model.buffers_for(self.buckets[-1])

    # ------------------------------------------------------------------ eager path
    def _run(self, frames, reward, last_action, done, h0, c0, actions, logits, baseline, seed_state=None,
             lstm_out=None):
        m = self.model
        n = frames.shape[0]
        seed = 0 if seed_state is not None else m.next_sample_seed()
        if m.use_lstm:
            lstm = dict(T1=1, B=n, done=done, h0=h0, c0=c0)
            if lstm_out is not None:
                lstm["hN"], lstm["cN"] = lstm_out
            m._forward_kernels(frames, reward, last_action, logits=logits, baseline=baseline, lstm=lstm,
                               actions=actions, seed=seed, greedy=self.greedy, seed_state=seed_state,
                               repack=False)
            return lstm["hN"], lstm["cN"]
        m._forward_kernels(frames, reward, last_action, logits=logits, baseline=baseline, keep_x0=False,
                           actions=actions, seed=seed, greedy=self.greedy, seed_state=seed_state, repack=False)
        return None

    def _inputs(self, inputs):
        x = inputs["frame"] if "frame" in inputs else inputs["observation"]
        if x.dim() == 5:  # (1, k, 4, 84, 84) as the reference's inference handle
            if x.shape[0] != 1:
                raise DimensionError(f"inference batch must be (1, k, ...), got {tuple(x.shape)}")
            x = x[0]
        if x.dtype != torch.uint8 or tuple(x.shape[1:]) != self.model.observation_shape:
            raise DimensionError(f"frames must be uint8 (k, {self.model.observation_shape}), got "
                                 f"{x.dtype} {tuple(x.shape)}")
        k = x.shape[0]
        reward = inputs["reward"].reshape(k).float()
        last_action = inputs["last_action"].reshape(k).to(torch.int64)
        done = None
        if self.model.use_lstm:
            d = inputs["done"].reshape(k)
            done = d.view(torch.uint8) if d.dtype == torch.bool else (d != 0).to(torch.uint8)
        return x.contiguous(), reward.contiguous(), last_action.contiguous(), done

    def _state(self, core_state, k):
        if not self.model.use_lstm:
            return None, None
        H = self.model.core_hidden
        if len(core_state) != 2:
            raise DimensionError("LSTM core_state must be (h, c), each (2, k, hidden)")
        h0, c0 = (s.float().contiguous() for s in core_state)
        if tuple(h0.shape) != (2, k, H) or tuple(c0.shape) != (2, k, H):
            raise DimensionError(f"core_state shapes {tuple(h0.shape)}, expected (2, {k}, {H})")
        return h0, c0

    @torch.no_grad()
    def __call__(self, inputs, core_state=()):
        frames, reward, last_action, done = self._inputs(inputs)
        k = frames.shape[0]
        h0, c0 = self._state(core_state, k)
        self.model.buffers_for(max(k, self.buckets[-1] if self.buckets else 0))
        if self.model.mirror_stale():
            self.model.pack_weights()
        bucket = next((b for b in self.buckets if b >= k), None)
        if bucket is None:
            A = self.model.num_actions
            actions = torch.empty(k, dtype=torch.int64, device=self.device)
            logits = torch.empty(k, A, device=self.device)
            baseline = torch.empty(k, device=self.device)
            state = self._run(frames, reward, last_action, done, h0, c0, actions, logits, baseline)
        else:
            actions, logits, baseline, state = self._replay(bucket, k, frames, reward, last_action, done, h0, c0)
        mv = self._mv.get(k)
        if mv is None or mv[0] != self.version:  # (cached per k: one fill when the version moves)
            mv = self._mv[k] = (self.version, torch.full((1, k), self.version, dtype=torch.int64, device=self.device))
        out = dict(action=actions.view(1, k), policy_logits=logits.view(1, k, -1), baseline=baseline.view(1, k),
                   model_version=mv[1])
        return (out, tuple(state) if state is not None else tuple())

    # ------------------------------------------------------------------ graph path
    def _capture(self, b):
        m, dev, A = self.model, self.device, self.model.num_actions
        # outputs packed in one buffer [actions b x i64 | logits b x A f32 | baseline b f32]: one
        # clone per call returns them
        outbuf = torch.empty(b * (8 + 4 * A + 4), dtype=torch.uint8, device=dev)
        st = dict(frames=torch.zeros(b, *m.observation_shape, dtype=torch.uint8, device=dev),
                  reward=torch.zeros(b, device=dev), last_action=torch.zeros(b, dtype=torch.int64, device=dev),
                  done=torch.zeros(b, dtype=torch.uint8, device=dev), outbuf=outbuf,
                  actions=outbuf[:8 * b].view(torch.int64), logits=outbuf[8 * b:8 * b + 4 * A * b].view(torch.float32).view(b, A),
                  baseline=outbuf[8 * b + 4 * A * b:].view(torch.float32))
        if m.use_lstm:
            shape = (2, b, m.core_hidden)
            st.update(h0=torch.zeros(shape, device=dev), c0=torch.zeros(shape, device=dev),
                      hN=torch.empty(shape, device=dev), cN=torch.empty(shape, device=dev))

        def body():
            self._run(st["frames"], st["reward"], st["last_action"], st["done"], st.get("h0"), st.get("c0"),
                      st["actions"], st["logits"], st["baseline"], seed_state=self.seed_state,
                      lstm_out=(st["hN"], st["cN"]) if m.use_lstm else None)

        saved = self.seed_state.clone()
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            body()  # warm-up: lazy init (tensor maps, function attributes) outside the capture
        torch.cuda.current_stream(dev).wait_stream(s)
        graph = torch.cuda.CUDAGraph()
        with graph_capture(graph):
            body()
        self.seed_state.copy_(saved)
        self._graphs[b] = (graph, st, m.buffer_generation)
        return self._graphs[b]

    def _replay(self, b, k, frames, reward, last_action, done, h0, c0):
        m = self.model
        ent = self._graphs.get(b)
        if ent is None or ent[2] != m.buffer_generation:
            ent = self._capture(b)
        graph, st, _ = ent
        # the inputs into the bucket's static buffers: one native call, one copy kernel (the
        # ctypes argument arrays are kept per bucket; only sources and sizes change)
        srcs_t = (frames, reward, last_action, done) if m.use_lstm else (frames, reward, last_action)
        arrs = st.get("_copy_args")
        if arrs is None:
            n = len(srcs_t)
            dst_t = (st["frames"], st["reward"], st["last_action"], st["done"])[:n]
            arrs = st["_copy_args"] = ((C.c_void_p * n)(*[d.data_ptr() for d in dst_t]), (C.c_void_p * n)(),
                                       (C.c_size_t * n)(), n, N.lib().bp_copy_many)
        dsts, srcs, nbytes, n, fn = arrs
        for i, src in enumerate(srcs_t):
            srcs[i] = src.data_ptr()
            nbytes[i] = src.numel() * src.element_size()
        N.check(fn(dsts, srcs, nbytes, n, torch.cuda.current_stream(self.device).cuda_stream), "bp_copy_many")
        if m.use_lstm:  # (strided (2, k, H) slices: torch copies)
            st["h0"][:, :k].copy_(h0)
            st["c0"][:, :k].copy_(c0)
        graph.replay()
        state = None
        if m.use_lstm:
            state = (st["hN"][:, :k].clone(), st["cN"][:, :k].clone())
        A, out = m.num_actions, st["outbuf"].clone()
        return (out[:8 * b].view(torch.int64)[:k], out[8 * b:8 * b + 4 * A * b].view(torch.float32).view(b, A)[:k],
                out[8 * b + 4 * A * b:].view(torch.float32)[:k], state)
