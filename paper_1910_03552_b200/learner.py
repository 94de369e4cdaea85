"""The IMPALA learner step: upstream TorchBeast `learn()` as a fused device pipeline.

Replaces LearnerContext.train_batch (pipeline.py:297-373) +
SharedModel.apply_gradients (pipeline.py:247-251) -- and upstream
`monobeast.learn(flags, actor_model, model, batch, initial_agent_state,
optimizer, scheduler, lock)` [upstream, not vendored] with the same signature.

One step = (all on the current CUDA stream, no host sync until stats are read)
  1. AtariNet forward on (T+1)*B frames          bp_atari_forward   (tcgen05)
     (LSTM core: bp_atari_lstm_forward -- persistent recurrent kernels)
  2. fused V-trace + 3 losses + d_logits/d_base  bp_learner_loss_f32
  3. AtariNet backward -> flat f32 gradients     bp_atari_backward  (tcgen05)
  4. [DP] NCCL all-reduce(SUM) of the flat gradient buffer (torch.distributed)
  5. global-norm clip + RMSProp                  bp_sumsq_f32 + bp_rmsprop_clip_f32

Row alignment follows upstream (`batch[1:]` for actions / behaviour logits /
rewards / done, learner outputs rows [:-1], bootstrap = baseline[-1]).
"""
from __future__ import annotations

import collections
import os
import threading

import numpy as np
import torch

from . import _native as N  # noqa: F401  (fail loudly if the library is missing)
from .errors import NONFINITE_GRAD, NONFINITE_IN, NONFINITE_LOSS, SchemaError, StatusWord, raise_for_bits
from .learner_ops import LearnerLoss, VtraceConfig
from ._tensors import graph_capture
from .optim import RMSprop, sumsq_

# learner-input fields and their dtypes (upstream learn() batch; validate_batch rollout.py:160-192)
_BATCH_DTYPES = {"reward": (torch.float32,), "done": (torch.bool,),
                 "policy_logits": (torch.float32,), "action": (torch.int64,),
                 "last_action": (torch.int64,), "frame": (torch.uint8,),
                 "frame_planes": (torch.uint8,), "frame_index": (torch.int32,),
                 "episode_return": (torch.float32,)}
# max captured step graphs per learner (each pins its own memory pool); least recently used
# graphs are evicted beyond this
MAX_GRAPHS = int(os.environ.get("BP_MAX_GRAPHS", "4"))


def _flag(flags, name, default=None):
    if isinstance(flags, dict):
        return flags.get(name, default)
    return getattr(flags, name, default)


class FusedLearner:
    """Preallocated learner step for one (model, T, B); `step()` enqueues only."""

    def __init__(self, model, flags, unroll_length: int, batch_size: int, process_group=None):
        self.model = model
        self.T = unroll_length
        self.B = batch_size
        self.n = (unroll_length + 1) * batch_size
        dev = model.flat_params.device
        A = model.num_actions
        self.cfg = VtraceConfig(
            discount=float(_flag(flags, "discounting", 0.99)),
            baseline_cost=float(_flag(flags, "baseline_cost", 0.5)),
            entropy_cost=float(_flag(flags, "entropy_cost", 0.0006)),
            reward_clip=_flag(flags, "reward_clipping", "abs_one") == "abs_one",
            row_shift=1)
        self.max_norm = float(_flag(flags, "grad_norm_clipping", 40.0))
        self.loss = LearnerLoss(dev)
        self.logits = torch.empty(self.n, A, device=dev)
        self.baseline = torch.empty(self.n, device=dev)
        self.d_logits = torch.zeros(self.n, A, device=dev)  # row T stays zero
        self.d_baseline = torch.zeros(self.n, device=dev)
        self.losses = torch.zeros(4, dtype=torch.float64, device=dev)
        # stats read-back: losses + done[1:] + episode_return[1:], written by one kernel straight
        # into pinned (device-mapped) host memory: one device->host transfer per step, no copy node
        self._stats_host = torch.empty(40 + unroll_length * batch_size * 5, dtype=torch.uint8,
                                       pin_memory=True)
        self._stats_event = torch.cuda.Event()
        # numpy views of the pinned read-back buffer (no per-step tensor/numpy conversions)
        tb = unroll_length * batch_size
        hnp = self._stats_host.numpy()
        self._np_losses = hnp[:32].view(np.float64)
        self._np_status = hnp[32:36].view(np.uint32)
        # completion sequence number, published by the pack kernel after its other writes
        # (bp_pack_stats seq_state): stats() spins on it instead of an event round trip
        self._np_seq = hnp[36:40].view(np.uint32)
        self._np_seq[0] = 0
        self._seq_state = torch.zeros(2, dtype=torch.int32, device=dev)
        self._pack_stream = torch.cuda.Stream(device=dev)  # the stats pack beside the update
        self._state_zero = False  # LSTM: h0 / c0 staged buffers hold zeros
        self._packs = 0  # packs enqueued (graph replays included)
        self._seq_addr = self._stats_host.data_ptr() + 36
        self._c_wait = N.lib().bp_host_wait_seq
        self._np_done = hnp[40:40 + tb].view(np.bool_)
        self._np_ret = hnp[40 + tb:].view(np.float32)
        # this learner's device status word: the fused loss ORs violation bits into it, the
        # optimiser rejects a step whose (all-reduced) total loss is non-finite, and the stats
        # pack reads it back with the losses and clears it (include/beast_b200.h BP_STATUS_*)
        self.status = StatusWord(dev)
        self.pg = process_group
        # where a non-finite step dumps its batch (pipeline.py:254-268 _dump_batch)
        self.logdir = _flag(flags, "logdir", None) or _flag(flags, "savedir", None)
        model.buffers_for(self.n)
        # LSTM core: the initial agent state is staged into fixed buffers (graph inputs)
        self.lstm = None
        if getattr(model, "use_lstm", False):
            shape = (2, batch_size, model.core_hidden)
            self.lstm = dict(T1=unroll_length + 1, B=batch_size,
                             h0=torch.zeros(shape, device=dev), c0=torch.zeros(shape, device=dev),
                             hN=torch.empty(shape, device=dev), cN=torch.empty(shape, device=dev))
        # CUDA graphs: one captured step per (batch buffer set, optimizer); see step()
        self.use_graphs = True
        self.kernels_per_step = 0
        self._graphs: collections.OrderedDict = collections.OrderedDict()  # LRU, <= MAX_GRAPHS
        self._seen: collections.OrderedDict = collections.OrderedDict()
        self._validated: set = set()  # graph keys whose batch schema was checked
        self._key_memo: dict = {}     # id(batch) -> (tensors, versions, addresses, optimiser, gen, key, batch)
        self._buf_gen = model.buffer_generation
        # data parallel: the fc weight gradient (95% of the no-LSTM parameters) is all-reduced on
        # a side stream as soon as the backward has written it (BpAtariNet.fc_grad_ready), while
        # the conv data / weight gradients still run; the small remainder after the backward
        self.bucketed = process_group is not None and not getattr(model, "use_lstm", False)
        if self.bucketed:
            names = [k for k, _ in model.named_parameters()]
            off, cnt, _ = model._shapes[names.index("fc.weight")]
            g = model.flat_grads
            self._buckets = (g[off:off + cnt], g[:off], g[off + cnt:])
            self._fc_ready = torch.cuda.Event()
            self._fc_ready.record()  # materialise the CUDA event handle
            self._dp_stream = torch.cuda.Stream(device=dev)

    def _pg_is_nccl(self) -> bool:
        """NCCL collectives can be captured in a CUDA graph; gloo ones cannot."""
        grp = None if self.pg is True else self.pg
        return torch.distributed.get_backend(grp) == "nccl"

    def _fields(self, batch):
        return (("frame_planes", "frame_index") if "frame_planes" in batch else ("frame",)) + (
            "reward", "done", "policy_logits", "action", "last_action")

    def _graph_key(self, batch, optimizer):
        """A captured step reads raw device addresses: key it on every batch tensor's address,
        dtype, shape and strides, the optimiser, and the model's activation-buffer generation.
        Memoised per batch dict (e.g. the DeviceInfeed slots): a hit needs the same tensor
        objects (held by the memo, so their ids cannot be recycled) at the same version counters
        and addresses -- in-place reshapes / set_() bump the version or move the data."""
        ep = batch.get("episode_return") if isinstance(batch, dict) else None
        ts = [batch[k] for k in self._fields(batch)] + ([ep] if ep is not None else [])
        m = self._key_memo.get(id(batch))
        if (m is not None and m[3] is optimizer and m[4] == self.model.buffer_generation and len(m[0]) == len(ts)
                and all(a is b and a._version == v and a.data_ptr() == p
                        for a, b, v, p in zip(ts, m[0], m[1], m[2]))):
            return m[5]
        key = tuple((t.data_ptr(), t.dtype, tuple(t.shape), t.stride()) for t in ts) + (
            ep is not None, id(optimizer), self.model.buffer_generation)
        self._key_memo[id(batch)] = (tuple(ts), tuple(t._version for t in ts), tuple(t.data_ptr() for t in ts),
                                     optimizer, self.model.buffer_generation, key, batch)
        while len(self._key_memo) > 2 * MAX_GRAPHS:
            self._key_memo.pop(next(iter(self._key_memo)))
        return key

    def validate(self, batch):
        """Host-side schema checks of validate_batch (rollout.py:160-192): shapes and dtypes
        (done must be bool).  The data-dependent checks (action range, finite reward / logits)
        run inside the fused loss kernel and are raised by stats()."""
        T, B, A = self.T, self.B, self.model.num_actions
        for k in self._fields(batch):
            if k not in batch:
                raise SchemaError(f"batch has no {k!r}")
            v = batch[k]
            if not isinstance(v, torch.Tensor) or not v.is_cuda:
                raise SchemaError(f"{k}: expected a CUDA tensor")
            if v.dtype not in _BATCH_DTYPES[k]:
                raise SchemaError(f"{k}: dtype {v.dtype}, expected {_BATCH_DTYPES[k][0]}")
            if not v.is_contiguous():
                raise SchemaError(f"{k}: must be contiguous (time-major (T+1, B, ...))")
        want = {"reward": (T + 1, B), "done": (T + 1, B), "action": (T + 1, B), "last_action": (T + 1, B),
                "policy_logits": (T + 1, B, A)}
        if "frame_planes" in batch:
            want["frame_index"] = (T + 1, B, 4)
        else:
            want["frame"] = (T + 1, B) + tuple(self.model.observation_shape)
        for k, shape in want.items():
            if tuple(batch[k].shape) != shape:
                raise SchemaError(f"{k}: dims {tuple(batch[k].shape)}, expected {shape}")
        ep = batch.get("episode_return")
        if ep is not None and tuple(ep.shape) != (T + 1, B):
            raise SchemaError(f"episode_return: dims {tuple(ep.shape)}, expected ({T + 1}, {B})")

    def _drop_graphs(self):
        self._graphs.clear()
        self._key_memo.clear()
        self._seen.clear()
        self._validated.clear()

    def step(self, batch, optimizer=None, scheduler=None, initial_agent_state=()):
        """Enqueue one learner step on the current stream; returns the device loss vector.

        With `use_graphs` (default) the whole step -- forward, fused loss,
        backward, all-reduce, clip + RMSProp: ~23 kernels -- is captured once per
        set of batch buffers (e.g. the two DeviceInfeed slots) as a CUDA graph and
        replayed, so host launch overhead leaves the critical path.  The first
        call per buffer set runs eagerly (warm-up), the second captures.
        LSTM nets copy `initial_agent_state` (h, c) into the staged state buffers first.
        """
        if self.lstm is not None:
            if len(initial_agent_state) == 2:
                self.lstm["h0"].copy_(initial_agent_state[0])
                self.lstm["c0"].copy_(initial_agent_state[1])
                self._state_zero = False
            elif not self._state_zero:  # (the step only reads h0 / c0: zero stays zero)
                self.lstm["h0"].zero_()
                self.lstm["c0"].zero_()
                self._state_zero = True
        if self._buf_gen != self.model.buffer_generation:
            # the model reallocated its activation buffers (e.g. a larger forward): every
            # captured graph points at freed memory
            self._drop_graphs()
            self._buf_gen = self.model.buffer_generation
        key = self._graph_key(batch, optimizer)
        if key not in self._validated:
            self.validate(batch)
            self._validated.add(key)
        graphable = (self.use_graphs and (self.pg is None or self._pg_is_nccl()) and
                     (optimizer is None or (isinstance(optimizer, RMSprop) and
                                            optimizer.flat_params.data_ptr() ==
                                            self.model.flat_params.data_ptr())))
        if graphable:
            g = self._graphs.get(key)
            if g is None and key in self._seen:
                optimizer and optimizer.sync_lr()
                if self.model.mirror_stale():  # the captured step must not contain the pack
                    self.model.pack_weights()
                g = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream()
                side.wait_stream(torch.cuda.current_stream())
                c0 = N.lib().bp_launch_count()
                try:
                    with graph_capture(g, stream=side):
                        self._step_eager(batch, optimizer)
                except (RuntimeError, torch.cuda.CudaError) as exc:
                    if self.pg is None:
                        raise
                    # a process group whose collectives cannot be captured (NCCL without graph
                    # support): run this learner's steps eagerly instead of failing the job
                    torch.cuda.synchronize()
                    self.use_graphs = False
                    self.capture_error = repr(exc)
                    self._step_eager(batch, optimizer)
                    if scheduler is not None:
                        scheduler.step()
                    return self.losses
                self.kernels_per_step = int(N.lib().bp_launch_count() - c0)
                torch.cuda.current_stream().wait_stream(side)
                self._graphs[key] = g
                while len(self._graphs) > MAX_GRAPHS:
                    self._graphs.popitem(last=False)
            if g is not None:
                self._graphs.move_to_end(key)
                if optimizer is not None:
                    optimizer.sync_lr()
                if self.model.mirror_stale():  # e.g. load_state_dict between steps
                    self.model.pack_weights()
                g.replay()
                self._packs += 1  # the replayed step packs its stats
                if scheduler is not None:
                    scheduler.step()
                return self.losses
            self._seen[key] = True
            while len(self._seen) > 4 * MAX_GRAPHS:
                self._seen.popitem(last=False)
        self._step_eager(batch, optimizer)
        if scheduler is not None:
            scheduler.step()
        return self.losses

    def _step_eager(self, batch, optimizer=None):
        m, T, B, n = self.model, self.T, self.B, self.n
        plane_index = None
        if "frame_planes" in batch:  # frame-stack dedup (rollout.frame_stack_index)
            frames, plane_index = batch["frame_planes"], batch["frame_index"]
            if tuple(plane_index.shape) != (T + 1, B, 4):
                raise SchemaError(f"frame_index dims {tuple(plane_index.shape)}, expected ({T + 1}, {B}, 4)")
            frames = frames.reshape(-1, *m.observation_shape[1:])
        else:
            frames = batch["frame"]
            if tuple(frames.shape[:2]) != (T + 1, B):
                raise SchemaError(f"frame dims {tuple(frames.shape)}, expected ({T + 1}, {B}, ...)")
            frames = frames.reshape(n, *m.observation_shape)
        A = m.num_actions
        reward = batch["reward"]
        last_action = batch["last_action"]
        lstm = None
        if self.lstm is not None:
            done = batch["done"].reshape(n)
            lstm = dict(self.lstm, done=done.view(torch.uint8) if done.dtype == torch.bool else done)
        # 1. forward (the bf16 operand mirror is refreshed by the fused optimiser below)
        m._forward_kernels(frames, reward.reshape(n), last_action.reshape(n), logits=self.logits,
                           baseline=self.baseline,
                           repack=None,  # packs only if stale (first step, load_state_dict, ...)
                           lstm=lstm, plane_index=plane_index)
        # 2. fused V-trace + losses + gradients w.r.t. logits / baseline
        self.loss(self.logits[:T * B].view(T, B, A), self.baseline.view(T + 1, B),
                  batch["policy_logits"][1:], batch["action"][1:], reward[1:], batch["done"][1:],
                  self.cfg, d_logits=self.d_logits[:T * B].view(T, B, A),
                  d_baseline=self.d_baseline.view(T + 1, B), losses=self.losses, status=self.status)
        # 3. backward into the flat gradient buffer
        if self.bucketed:
            m._bufs.struct.fc_grad_ready = self._fc_ready.cuda_event
        try:
            m._backward_kernels(self.d_logits, self.d_baseline, reward.reshape(n), last_action.reshape(n),
                                m.flat_grads, lstm=lstm)
        finally:
            if self.bucketed:
                m._bufs.struct.fc_grad_ready = None
        # 4. data-parallel over B: the losses are sums over (T, B) (vtrace.py:194-196), so
        #    the full-batch gradient is the SUM of the shard gradients (all-reduce of the flat
        #    f32 buffer); the loss scalars are summed too, for the stats and the reject check
        if self.pg is not None:
            grp = self.pg if self.pg is not True else None
            SUM = torch.distributed.ReduceOp.SUM
            if self.bucketed:
                fc_w, head, tail = self._buckets
                side = self._dp_stream
                side.wait_event(self._fc_ready)  # recorded by the backward after the fc wgrad
                with torch.cuda.stream(side):
                    torch.distributed.all_reduce(fc_w, op=SUM, group=grp)
                torch.distributed.all_reduce(head, op=SUM, group=grp)
                torch.distributed.all_reduce(tail, op=SUM, group=grp)
                torch.distributed.all_reduce(self.losses, op=SUM, group=grp)
                torch.cuda.current_stream().wait_stream(side)
            else:
                torch.distributed.all_reduce(m.flat_grads, op=SUM, group=grp)
                torch.distributed.all_reduce(self.losses, op=SUM, group=grp)
        # 5. clip + RMSProp.  A step whose (all-reduced) total loss is non-finite -- a NaN loss,
        #    or a batch violation, which the loss kernel turns into a NaN total -- is rejected on
        #    the device (model.py:251-252: parameters untouched); stats() then raises
        if optimizer is not None:
            if isinstance(optimizer, RMSprop) and optimizer.flat_params.data_ptr() == m.flat_params.data_ptr():
                # the stats pack forks off once the gradient norm is reduced and runs beside the
                # update: it derives the update's reject verdict from the same norm + loss, so
                # the host's read-back (and its turnaround to the next step) overlaps the
                # RMSProp pass instead of trailing it.  (Measured alternatives: the pack beside
                # the backward delays a persistent GEMM's CTA; copy-engine copies of the stats
                # as graph memcpy nodes cost ~10 us per step.)
                cur = torch.cuda.current_stream()
                side = self._pack_stream

                def fork_pack(sumsq):
                    side.wait_stream(cur)
                    with torch.cuda.stream(side):
                        self._pack_stats(batch, self.losses, sumsq=sumsq)

                optimizer.step(max_norm=self.max_norm, mirror=m.flat_bf16,  # params + bf16 mirror
                               status=False, reject_if_nonfinite=self.losses[3:], on_norm=fork_pack)
                cur.wait_stream(side)
                m.mirror_fresh = True
                m._packed_version = m.flat_params._version
                return self.losses
            else:  # any torch optimiser: check the step first (one sync), then clip + its own step
                bits = self.status.bits()
                if bits or not bool(torch.isfinite(self.losses[3])):
                    self.status.clear()
                    self._raise(batch, bits | NONFINITE_LOSS)
                ss = torch.zeros(1, dtype=torch.float64, device=m.flat_grads.device)
                sumsq_(m.flat_grads, ss)
                coef = torch.clamp(self.max_norm / (ss.sqrt().float() + 1e-6), max=1.0)
                m.flat_grads.mul_(coef)
                optimizer.step()
                m.mirror_fresh = False
        self._pack_stats(batch, self.losses)
        return self.losses

    def _pack_stats(self, batch, losses, sumsq=None):
        """Loss vector, done[1:] and episode_return[1:] -> the pinned read-back buffer, written
        by one kernel through the device mapping of the pinned host memory (unified virtual
        addressing).  Part of the step (and of its CUDA graph)."""
        T, B = self.T, self.B
        tb = T * B
        host = self._stats_host
        done = batch["done"][1:].reshape(tb)
        done = done.view(torch.uint8) if done.dtype == torch.bool else done.to(torch.uint8)
        ep = batch.get("episode_return") if isinstance(batch, dict) else None
        if ep is not None:
            ep = ep[1:].reshape(tb)
            if ep.dtype != torch.float32 or not ep.is_contiguous():
                ep = ep.float().contiguous()
        losses = losses if losses.dtype == torch.float64 and losses.is_contiguous() else losses.double().contiguous()
        if not torch.cuda.is_current_stream_capturing():  # (a capture runs nothing; replays count)
            self._packs += 1
        N.check(N.lib().bp_pack_stats(losses.data_ptr(), done.data_ptr(), ep.data_ptr() if ep is not None else None,
                                      tb, self.status.ptr(), sumsq.data_ptr() if sumsq is not None else None,
                                      self._seq_state.data_ptr(), host.data_ptr(),
                                      N.stream_handle(losses.device)),
                "bp_pack_stats")

    def _wait_pack(self):
        """Wait for the latest enqueued stats pack: spin on its completion word in the pinned
        buffer (sub-microsecond wake-up, no driver call); after ~50 ms of spinning fall back to
        a stream synchronise, which also surfaces device errors."""
        want = self._packs & 0xFFFFFFFF
        flag = self._np_seq
        # done once the published sequence number reached `want` (wrap-around safe; packs
        # replayed outside step() only move it further ahead)
        if ((int(flag[0]) - want) & 0xFFFFFFFF) < 0x80000000:
            return
        # the spin runs in C without the GIL (other Python threads keep running)
        if self._c_wait(self._seq_addr, want, 50_000):
            torch.cuda.current_stream(self.model.flat_params.device).synchronize()
            if ((int(flag[0]) - want) & 0xFFFFFFFF) >= 0x80000000:
                raise RuntimeError(f"learner stats pack {want} never completed (seq {int(flag[0])})")

    def stats(self, batch, losses=None):
        """Upstream learn() stats dict from the step's packed read-back (one sync)."""
        if losses is not None:  # an explicit loss vector: pack it now
            self._pack_stats(batch, losses)
        ep = batch.get("episode_return") if isinstance(batch, dict) else None
        self._wait_pack()
        bits = int(self._np_status[0])
        pg, base, ent, total = self._np_losses.tolist()
        if bits or not np.isfinite(total):
            # a rank whose own batch is fine still sees its peers' violations as a NaN total
            self._raise(batch, bits if bits else NONFINITE_LOSS)
        cfg = self.cfg
        returns = self._np_ret[self._np_done].tolist() if ep is not None else []
        return {
            "episode_returns": tuple(returns),
            # (a Python sum over the few finished episodes: cheaper than numpy's mean on a small
            # array; same value up to summation order)
            "mean_episode_return": sum(returns) / len(returns) if returns else float("nan"),
            "total_loss": total,
            "pg_loss": pg * cfg.pg_cost,
            "baseline_loss": base * cfg.baseline_cost,
            "entropy_loss": ent * cfg.entropy_cost,
        }


    def _raise(self, batch, bits):
        """The reference's error contract for a learner step: batch schema violations raise
        SchemaError (validate_batch, rollout.py:160-192); a non-finite loss or gradient dumps the
        batch to <logdir>/diagnostic_batch.npz and raises NonFiniteError (pipeline.py:333-338,
        vtrace.py:202-205, model.py:251-252).  The device already rejected the update."""
        dumped = None
        if bits & (NONFINITE_IN | NONFINITE_LOSS | NONFINITE_GRAD) and not bits & ~(
                NONFINITE_IN | NONFINITE_LOSS | NONFINITE_GRAD) and self.logdir:
            dumped = dump_batch(batch, self.logdir)
        try:
            raise_for_bits(bits, "learner step", learner=True)
        except Exception as e:
            if dumped:
                e.add_note(f"offending batch dumped to {dumped}")
            raise


def dump_batch(batch, logdir) -> str:
    """pipeline.py:254-268 `_dump_batch`: the offending learner batch as diagnostic_batch.npz."""
    os.makedirs(logdir, exist_ok=True)
    path = os.path.join(logdir, "diagnostic_batch.npz")
    np.savez(path, **{k: v.detach().cpu().numpy() for k, v in batch.items() if isinstance(v, torch.Tensor)})
    return path


def learn(flags, actor_model, model, batch, initial_agent_state, optimizer, scheduler,
          lock=threading.Lock(), process_group=None):
    """Upstream `learn()` signature; performs the fused step and returns the stats dict.

    `batch` is the upstream learner dict (frame (T+1,B,4,84,84) u8, reward, done,
    policy_logits, action, last_action[, episode_return]).  With frame-stack dedup it
    carries `frame_planes` (P,84,84) u8 + `frame_index` (T+1,B,4) int32 instead of
    `frame` (rollout.dedup_frames / frame_stack_index): a quarter of the H2D bytes,
    bit-identical results."""
    with lock:
        T1, B = (batch["frame_index"] if "frame_planes" in batch else batch["frame"]).shape[:2]
        key = (T1 - 1, B)
        fl = getattr(model, "_fused_learners", None)
        if fl is None:
            fl = model._fused_learners = {}
        L = fl.get(key)
        if L is None:
            L = fl[key] = FusedLearner(model, flags, T1 - 1, B, process_group)
        L.step(batch, optimizer, scheduler, initial_agent_state)
        stats = L.stats(batch)
        if actor_model is not None and actor_model is not model:
            actor_model.load_state_dict(model.state_dict())
        return stats


class DeviceInfeed:
    """Double-buffered pinned-host -> HBM batch infeed on a side stream.

    Next-row item of SURVEY 8f-2 (the reference stacks host rollouts with
    np.stack, rollout.py:116-144, and the learner reads them from host memory):
    `put(host_batch)` enqueues the H2D copies of the NEXT batch on a copy
    stream while the current learner step runs; `get()` makes the compute
    stream wait for that copy and returns the device batch.
    """

    def __init__(self, like: dict, device=None, depth: int = 2):
        self.device = torch.device(device or "cuda")
        self.depth = depth
        # packed layout: every field at a 256-byte aligned offset of one flat buffer, so a
        # host batch in the same layout (alloc_host) moves with ONE H2D copy per step
        self.layout = {}
        off = 0
        for k, v in like.items():
            self.layout[k] = (off, tuple(v.shape), v.dtype)
            off += (v.numel() * v.element_size() + 255) & ~255
        self.packed_bytes = off
        self.flat = [torch.empty(off, dtype=torch.uint8, device=self.device) for _ in range(depth)]
        self.slots = [self._views(f) for f in self.flat]
        self.events = [torch.cuda.Event() for _ in range(depth)]
        self.freed = [torch.cuda.Event() for _ in range(depth)]
        self.stream = torch.cuda.Stream(device=self.device)
        # raw handles for the one-call refill (bp_infeed_put); torch creates an event's
        # CUDA handle at its first record
        for ev in self.events + self.freed:
            ev.record(self.stream)
        self._stream_h = self.stream.cuda_stream
        self.state = [self._FREE] * depth
        self.head = 0  # next slot to fill
        self.tail = 0  # next slot to consume
        self.bytes_per_batch = sum(v.numel() * v.element_size() for v in like.values())

    def _views(self, flat: torch.Tensor) -> dict:
        out = {}
        for k, (off, shape, dtype) in self.layout.items():
            nbytes = torch.Size(shape).numel() * torch.empty(0, dtype=dtype).element_size()
            out[k] = flat[off:off + nbytes].view(dtype).view(shape)
        return out

    def alloc_host(self) -> dict:
        """A pinned host batch in the infeed's packed layout (what an actor writes its
        rollouts into); put() moves it with a single H2D copy."""
        flat = torch.empty(self.packed_bytes, dtype=torch.uint8, pin_memory=True)
        views = self._views(flat)
        views["__flat__"] = flat
        return views

    # slot life cycle (host-side bookkeeping; the device ordering is by events):
    #   free -> filled (put: H2D copy enqueued) -> consumed (get: the compute stream waits for
    #   the copy; steps enqueued after get() read it) -> released (freed event recorded on the
    #   compute stream after those steps) -> filled ...
    _FREE, _FILLED, _CONSUMED, _RELEASED = range(4)

    def _release_slot(self, slot: int) -> None:
        self.freed[slot].record(torch.cuda.current_stream(self.device))
        self.state[slot] = self._RELEASED

    def _claim_for_put(self) -> tuple[int, bool]:
        """The slot the next put() fills, and whether its copy must wait for a release.
        Raises if the producer ran a full ring ahead of the consumer (the slot still holds a
        batch nobody consumed).  A consumed slot that was never release()d is released HERE, on
        the current stream: the steps that read it were enqueued before this put (get(); step;
        put() order), so the copy cannot overwrite a batch an in-flight step still reads."""
        slot = self.head % self.depth
        st = self.state[slot]
        if st == self._FILLED:
            raise RuntimeError("DeviceInfeed.put(): ring full -- every slot holds a batch that was "
                               "not yet consumed by get()")
        if st == self._CONSUMED:
            self._release_slot(slot)
        return slot, self.state[slot] == self._RELEASED

    def put(self, host_batch: dict) -> None:
        slot, wait = self._claim_for_put()
        flat = host_batch.get("__flat__")
        if flat is not None and flat.numel() == self.packed_bytes and flat.is_pinned():
            # packed pinned batch: wait-for-release + one H2D copy + ready event in one C call
            N.check(N.lib().bp_infeed_put(self.flat[slot].data_ptr(), flat.data_ptr(), self.packed_bytes,
                                          self._stream_h, self.freed[slot].cuda_event if wait else None,
                                          self.events[slot].cuda_event), "bp_infeed_put")
        else:
            with torch.cuda.stream(self.stream):
                if wait:
                    self.stream.wait_event(self.freed[slot])  # consumer done with this slot
                if flat is not None and flat.numel() == self.packed_bytes:
                    self.flat[slot].copy_(flat, non_blocking=True)
                else:
                    for k, v in host_batch.items():
                        self.slots[slot][k].copy_(v, non_blocking=True)
                self.events[slot].record(self.stream)
        self.state[slot] = self._FILLED
        self.head += 1

    def get(self) -> dict:
        """The next filled slot; the current stream waits for its copy.  Every other slot that
        was consumed and not yet release()d is released first (at this point of the stream, i.e.
        after the steps enqueued on it so far)."""
        if self.tail >= self.head:
            raise RuntimeError("DeviceInfeed.get() without a pending put()")
        slot = self.tail % self.depth
        assert self.state[slot] == self._FILLED
        rel = None
        for other in range(self.depth):
            if other != slot and self.state[other] == self._CONSUMED:
                if rel is None:  # one release rides in the C call, any further ones here
                    rel = other
                else:
                    self._release_slot(other)
        N.check(N.lib().bp_infeed_get(torch.cuda.current_stream(self.device).cuda_stream,
                                      self.freed[rel].cuda_event if rel is not None else None,
                                      self.events[slot].cuda_event), "bp_infeed_get")
        if rel is not None:
            self.state[rel] = self._RELEASED
        self.state[slot] = self._CONSUMED
        self.tail += 1
        return self.slots[slot]

    def release(self) -> None:
        """Mark the most recently consumed slot reusable (after its step was enqueued on the
        current stream).  Optional: get() and put() release consumed slots themselves."""
        slot = (self.tail - 1) % self.depth
        if self.tail > 0 and self.state[slot] == self._CONSUMED:
            self._release_slot(slot)
