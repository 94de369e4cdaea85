"""torch-CPU fp32 restatement of upstream TorchBeast AtariNet and learn().

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

The reference mount has no conv / LSTM network (SPEC.md:108 non-goal); the
north-star names upstream torchbeast `monobeast.AtariNet` and `learn()`
(github facebookresearch/torchbeast, not vendored, no pinned version).  This
is a restatement of that public algorithm, PARITY UNPINNED by the reference's
own tests; it is pinned instead by autograd + finite differences
(tests/test_oracle_network.py), following the reference's gradient-check
methodology (pkg/tests/conftest.py:5-26).
"""
from __future__ import annotations

import torch
import torch.nn.functional as F
from torch import nn


class AtariNetRef(nn.Module):
    """Upstream AtariNet (no-LSTM and LSTM paths), fp32, any device."""

    def __init__(self, observation_shape=(4, 84, 84), num_actions=6, use_lstm=False):
        super().__init__()
        self.observation_shape = observation_shape
        self.num_actions = num_actions
        self.conv1 = nn.Conv2d(observation_shape[0], 32, kernel_size=8, stride=4)
        self.conv2 = nn.Conv2d(32, 64, kernel_size=4, stride=2)
        self.conv3 = nn.Conv2d(64, 64, kernel_size=3, stride=1)
        self.fc = nn.Linear(3136, 512)
        core_output_size = self.fc.out_features + num_actions + 1
        self.use_lstm = use_lstm
        if use_lstm:
            self.core = nn.LSTM(core_output_size, core_output_size, 2)
        self.policy = nn.Linear(core_output_size, num_actions)
        self.baseline = nn.Linear(core_output_size, 1)

    def initial_state(self, batch_size):
        if not self.use_lstm:
            return tuple()
        return tuple(torch.zeros(self.core.num_layers, batch_size, self.core.hidden_size)
                     for _ in range(2))

    def torso(self, inputs):
        x = inputs["frame"]
        T, B, *_ = x.shape
        dt = self.conv1.weight.dtype
        x = torch.flatten(x, 0, 1).to(dt) / 255.0
        x = F.relu(self.conv1(x))
        x = F.relu(self.conv2(x))
        x = F.relu(self.conv3(x))
        x = x.view(T * B, -1)
        x = F.relu(self.fc(x))
        one_hot = F.one_hot(inputs["last_action"].view(T * B), self.num_actions).to(dt)
        clipped_reward = torch.clamp(inputs["reward"], -1, 1).view(T * B, 1).to(dt)
        return torch.cat([x, clipped_reward, one_hot], dim=-1)

    def forward(self, inputs, core_state=()):
        T, B = inputs["frame"].shape[:2]
        core_input = self.torso(inputs)
        if self.use_lstm:
            core_input = core_input.view(T, B, -1)
            outs = []
            notdone = (~inputs["done"]).float()
            for inp, nd in zip(core_input.unbind(), notdone.unbind()):
                nd = nd.view(1, -1, 1)
                core_state = tuple(nd * s for s in core_state)
                out, core_state = self.core(inp.unsqueeze(0), core_state)
                outs.append(out)
            core_output = torch.flatten(torch.cat(outs), 0, 1)
        else:
            core_output = core_input
            core_state = tuple()
        policy_logits = self.policy(core_output)
        baseline = self.baseline(core_output)
        action = torch.argmax(policy_logits, dim=1)
        return (dict(policy_logits=policy_logits.view(T, B, self.num_actions),
                     baseline=baseline.view(T, B), action=action.view(T, B)), core_state)


# ---------------------------------------------------------------------------------------------
# bf16-operand emulation of the GPU network (parity oracle for the tcgen05 kernels)
#
# The kernels (paper_1910_03552_b200/csrc/network.cu) round to bf16 at fixed storage points and
# accumulate in f32.  Restating those roundings on top of the fp32 upstream graph turns the
# comparison from "bf16 vs fp32" (ReLU sign flips of near-zero pre-activations dominate, ~10%
# torso gradient noise) into "f32 vs f64 accumulation order" (~1e-6), so gradients can be pinned
# tightly.  Storage points restated here (network.cu torso_forward / heads_backward /
# torso_backward, lstm_cluster.cu):
#   forward   every GEMM operand: weights (flat bf16 mirror), activations X1, X2, X3, core
#             (relu(fc) | clip(r) | onehot(a) | 1), heads operand [W | b] (so the head BIASES are
#             bf16 too); LSTM: [W_ih | b_ih + b_hh] (one bf16 bias), layer outputs, and in the
#             cluster recurrence W_hh and h_{t-1}
#   backward  G = [d_logits | d_baseline] bf16 (heads weight / bias / data gradients); every
#             conv data gradient d_pre1/2/3 (= the gradient at the pre-activation, also the
#             operand of the weight gradient and the summand of the bias gradient); d_fc for
#             Wfc and X3 (but d bfc is the epilogue's f32 column sum); LSTM gate gradients
#             dgates (all LSTM weight / input gradients and, cluster mode, the recurrent dz)
# Not emulated: the cluster recurrence's MUFU tanh (~2^-11 relative).
# ---------------------------------------------------------------------------------------------


def bf16_round(t):
    return t.to(torch.bfloat16).to(t.dtype)


def st_bf16(t):
    """Straight-through bf16 rounding: rounded forward, identity gradient."""
    return t + (bf16_round(t) - t).detach()


class _RoundGrad(torch.autograd.Function):
    """Identity forward; the incoming gradient is rounded to bf16 (a bf16-stored dY)."""

    @staticmethod
    def forward(ctx, x):
        return x.view_as(x)

    @staticmethod
    def backward(ctx, g):
        return bf16_round(g)


def rg_bf16(t):
    return _RoundGrad.apply(t)


def _relu(z, zabs, mask, band, stats, name):
    """ReLU whose decision adopts the kernel's mask ONLY inside the accumulation-ambiguity band
    |z| <= band * sum|terms| (the tensor cores' accumulation error, ~1e-5 relative to sum|terms|,
    can legitimately flip the sign there); everywhere else the oracle's own sign decides, and
    `stats[name]` counts kernel masks that disagree OUTSIDE the band (must be 0) and adoptions."""
    own = z > 0
    if mask is None:
        return z * own.to(z.dtype)
    mask = mask.to(own.device)
    amb = z.abs() <= band * zabs
    if stats is not None:
        stats[name] = dict(disagree=int(((mask != own) & ~amb).sum()),
                           adopted=int(((mask != own) & amb).sum()), total=int(z.numel()))
    return z * torch.where(amb, mask, own).to(z.dtype)


def emulated_core_input(model, inputs, masks=None, band=1e-4, mask_stats=None):
    """The GPU `core` buffer (n, 513+A): [relu(fc) | clip(r) | onehot(last_a)], bf16 values,
    with the kernels' storage roundings (see the block comment above).
    masks: optional kernel ReLU decisions (conv1 (n,32,20,20), conv2 (n,64,9,9), conv3
    (n,64,7,7), fc (n,512) bool), adopted only inside the ambiguity band (_relu)."""
    x = inputs["frame"]
    T, B = x.shape[:2]
    n = T * B
    dt = model.conv1.weight.dtype
    x = torch.flatten(x, 0, 1).to(dt)  # u8 values are exact in bf16; the 1/255 is the epilogue's alpha
    w = st_bf16
    m = masks or (None,) * 4

    def sab(fn, xin, wt, b):  # sum |terms| of a pre-activation (ambiguity-band scale)
        if masks is None:
            return None
        with torch.no_grad():
            return fn(xin.abs(), wt.abs()) + b.abs()

    conv1 = lambda xx, ww: F.conv2d(xx, ww, None, stride=4) * (1.0 / 255.0)  # noqa: E731
    z1 = rg_bf16(conv1(x, w(model.conv1.weight)) + model.conv1.bias[:, None, None])
    a1 = st_bf16(_relu(z1, sab(conv1, x, w(model.conv1.weight), model.conv1.bias[:, None, None]), m[0], band,
                       mask_stats, "conv1"))
    conv2 = lambda xx, ww: F.conv2d(xx, ww, None, stride=2)  # noqa: E731
    z2 = rg_bf16(conv2(a1, w(model.conv2.weight)) + model.conv2.bias[:, None, None])
    a2 = st_bf16(_relu(z2, sab(conv2, a1, w(model.conv2.weight), model.conv2.bias[:, None, None]), m[1], band,
                       mask_stats, "conv2"))
    conv3 = lambda xx, ww: F.conv2d(xx, ww, None)  # noqa: E731
    z3 = rg_bf16(conv3(a2, w(model.conv3.weight)) + model.conv3.bias[:, None, None])
    a3 = st_bf16(_relu(z3, sab(conv3, a2, w(model.conv3.weight), model.conv3.bias[:, None, None]), m[2], band,
                       mask_stats, "conv3"))
    fc = lambda xx, ww: xx @ ww.t()  # noqa: E731
    x3 = a3.reshape(n, -1)
    zf = rg_bf16(fc(x3, w(model.fc.weight))) + model.fc.bias  # d bfc: f32 column sum
    h = st_bf16(_relu(zf, sab(fc, x3, w(model.fc.weight), model.fc.bias), m[3], band, mask_stats, "fc"))
    one_hot = F.one_hot(inputs["last_action"].reshape(n), model.num_actions).to(dt)
    clipped_reward = st_bf16(torch.clamp(inputs["reward"], -1, 1).reshape(n, 1).to(dt))
    return torch.cat([h, clipped_reward, one_hot], dim=-1)


def emulated_lstm(model, core_input, done, core_state, recurrence_bf16=True):
    """Upstream 2-layer nn.LSTM stepped with done resets, with the GPU's roundings.
    core_input (T1*B, H); done (T1, B) bool; core_state (h, c) each (2, B, H).
    recurrence_bf16: the cluster recurrence (bf16 W_hh, h_{t-1} and dz mma.sync operands);
    False: the cooperative f32 recurrence (only the GEMM operands are bf16).
    Returns (layer outputs [(T1, B, H)] * 2, (h_N, c_N))."""
    T1, B = done.shape
    H = core_input.shape[-1]
    dt = core_input.dtype
    inp = core_input.reshape(T1, B, H)
    outs, hs, cs = [], [], []
    for layer in range(2):
        wih = getattr(model.core, f"weight_ih_l{layer}")
        whh = getattr(model.core, f"weight_hh_l{layer}")
        bias = getattr(model.core, f"bias_ih_l{layer}") + getattr(model.core, f"bias_hh_l{layer}")
        gx = inp @ st_bf16(wih).t() + st_bf16(bias)
        whh_op = st_bf16(whh) if recurrence_bf16 else whh
        h, c = core_state[0][layer].to(dt), core_state[1][layer].to(dt)
        seq = []
        for t in range(T1):
            nd = (~done[t]).to(dt)[:, None]
            h, c = h * nd, c * nd
            if recurrence_bf16:
                z = rg_bf16(gx[t] + st_bf16(h) @ whh_op.t())
            else:  # f32 recurrence; the weight-gradient GEMMs still see bf16 dgates / h_{t-1}
                z = rg_bf16(gx[t]) + h @ whh.t()
            i, f, g, o = z.chunk(4, -1)
            c = torch.sigmoid(f) * c + torch.sigmoid(i) * torch.tanh(g)
            h = torch.sigmoid(o) * torch.tanh(c)
            seq.append(h)
        out = torch.stack(seq)
        outs.append(out)
        hs.append(h)
        cs.append(c)
        inp = st_bf16(out)  # the next layer / the heads read the bf16 output sequence
    return outs, (torch.stack(hs), torch.stack(cs))


def emulated_forward(model, inputs, core_state=(), recurrence_bf16=True, masks=None, band=1e-4,
                     mask_stats=None):
    """AtariNetRef.forward restated with the GPU kernels' bf16 storage points; same outputs.
    Run it on an fp64 copy of the model (any device) so the remaining difference to the
    kernels is their accumulation (the tensor cores' f32 accumulation truncates: ~1e-5 of
    sum|terms| at K = 3136, measured by tools/parity_diag.py).  masks / band / mask_stats: see
    emulated_core_input and _relu."""
    T, B = inputs["frame"].shape[:2]
    n = T * B
    core = emulated_core_input(model, inputs, masks, band, mask_stats)
    state = tuple()
    if model.use_lstm:
        outs, state = emulated_lstm(model, core, inputs["done"], core_state, recurrence_bf16)
        core = outs[1].reshape(n, -1)
    core = st_bf16(core)
    logits = rg_bf16(core @ st_bf16(model.policy.weight).t() + st_bf16(model.policy.bias))
    baseline = rg_bf16(core @ st_bf16(model.baseline.weight).t() + st_bf16(model.baseline.bias))
    action = torch.argmax(logits, dim=1)
    return (dict(policy_logits=logits.view(T, B, model.num_actions), baseline=baseline.view(T, B),
                 action=action.view(T, B)), state)


def vtrace_from_logits(behavior_policy_logits, target_policy_logits, actions, discounts, rewards,
                       values, bootstrap_value, clip_rho_threshold=1.0, clip_pg_rho_threshold=1.0):
    """Upstream vtrace.from_logits (torch restatement; targets under no_grad)."""
    def alp(logits, a):
        return -F.nll_loss(F.log_softmax(torch.flatten(logits, 0, -2), dim=-1), torch.flatten(a),
                           reduction="none").view_as(a)

    tlp = alp(target_policy_logits, actions)
    blp = alp(behavior_policy_logits, actions)
    log_rhos = tlp - blp
    with torch.no_grad():
        rhos = torch.exp(log_rhos)
        clipped = torch.clamp(rhos, max=clip_rho_threshold)
        cs = torch.clamp(rhos, max=1.0)
        v1 = torch.cat([values[1:], bootstrap_value.unsqueeze(0)], dim=0)
        deltas = clipped * (rewards + discounts * v1 - values)
        acc = torch.zeros_like(bootstrap_value)
        res = []
        for t in range(discounts.shape[0] - 1, -1, -1):
            acc = deltas[t] + discounts[t] * cs[t] * acc
            res.append(acc)
        res.reverse()
        vs = torch.stack(res) + values
        vs1 = torch.cat([vs[1:], bootstrap_value.unsqueeze(0)], dim=0)
        pg_adv = torch.clamp(rhos, max=clip_pg_rho_threshold) * (rewards + discounts * vs1 - values)
    return vs, pg_adv


def learn_losses(model, batch, flags, core_state=(), forward=None, scales=None):
    """Upstream learn() up to total_loss (no optimiser); returns (total, parts, outputs).
    forward: the network forward (default `model(batch, core_state)`; emulated_forward for the
    bf16-operand oracle).  scales: an optional dict that receives sum|term| of each loss (the
    tolerance basis for loss sums with cancellation)."""
    out, _ = (forward or model)(batch, core_state)
    bootstrap_value = out["baseline"][-1]
    b = {k: v[1:] for k, v in batch.items()}
    o = {k: v[:-1] for k, v in out.items()}
    rewards = b["reward"]
    clipped = torch.clamp(rewards, -1, 1) if flags["reward_clipping"] == "abs_one" else rewards
    discounts = (~b["done"]).to(rewards.dtype) * flags["discounting"]
    vs, pg_adv = vtrace_from_logits(b["policy_logits"], o["policy_logits"], b["action"], discounts,
                                    clipped, o["baseline"], bootstrap_value)
    ce = F.nll_loss(F.log_softmax(torch.flatten(o["policy_logits"], 0, 1), dim=-1),
                    target=torch.flatten(b["action"], 0, 1), reduction="none").view_as(pg_adv)
    pg_loss = torch.sum(ce * pg_adv.detach())
    baseline_loss = flags["baseline_cost"] * 0.5 * torch.sum((vs - o["baseline"]) ** 2)
    pol = F.softmax(o["policy_logits"], dim=-1)
    entropy_loss = flags["entropy_cost"] * torch.sum(pol * F.log_softmax(o["policy_logits"], dim=-1))
    total = pg_loss + baseline_loss + entropy_loss
    if scales is not None:
        with torch.no_grad():
            scales["pg_loss"] = float(torch.sum(torch.abs(ce * pg_adv)))
            scales["baseline_loss"] = float(baseline_loss)
            scales["entropy_loss"] = float(torch.abs(entropy_loss))
            scales["total_loss"] = scales["pg_loss"] + scales["baseline_loss"] + scales["entropy_loss"]
    return total, (pg_loss, baseline_loss, entropy_loss), out


def learn_grads(model, batch, flags, core_state=(), forward=None):
    """Upstream learn() up to the pre-optimiser gradients: (grads {name: tensor}, parts, scales).
    With forward=emulated_forward (on an fp64 model) this is the bf16-operand parity oracle of
    the fused learner step's flat gradients."""
    scales = {}
    total, parts, _ = learn_losses(model, batch, flags, core_state, forward=forward, scales=scales)
    for p in model.parameters():
        p.grad = None
    total.backward()
    grads = {k: p.grad.detach().clone() for k, p in model.named_parameters()}
    return grads, dict(total_loss=float(total.detach()), pg_loss=float(parts[0].detach()),
                       baseline_loss=float(parts[1].detach()), entropy_loss=float(parts[2].detach())), scales


def rmsprop_first_update(grads, flags):
    """clip_grad_norm_ (max/(norm+1e-6), clamped to 1) then the first torch RMSprop step from a
    zero square_avg: the parameter update -lr g / (sqrt((1-alpha) g^2) + eps), per tensor."""
    norm = torch.sqrt(sum(torch.sum(g.double() ** 2) for g in grads.values()))
    coef = torch.clamp(flags["grad_norm_clipping"] / (norm + 1e-6), max=1.0)
    out = {}
    for k, g in grads.items():
        g = g.double() * coef
        sq = (1.0 - flags["alpha"]) * g * g
        out[k] = -flags["learning_rate"] * g / (torch.sqrt(sq) + flags["epsilon"])
    return out, float(norm)


def learn_step(model, optimizer, batch, flags, core_state=()):
    """Upstream learn(): losses, backward, clip_grad_norm_, RMSprop step."""
    total, parts, out = learn_losses(model, batch, flags, core_state)
    optimizer.zero_grad()
    total.backward()
    norm = nn.utils.clip_grad_norm_(model.parameters(), flags["grad_norm_clipping"])
    optimizer.step()
    return total.item(), [p.item() for p in parts], float(norm)


DEFAULT_FLAGS = dict(discounting=0.99, baseline_cost=0.5, entropy_cost=0.0006,
                     reward_clipping="abs_one", grad_norm_clipping=40.0, learning_rate=0.00048,
                     alpha=0.99, epsilon=0.01, momentum=0.0)


def synthetic_batch(T, B, A, seed=0, device="cpu", frame_seed=None):
    """Synthetic learner batch with upstream keys, time-major (T+1, B)."""
    g = torch.Generator().manual_seed(seed)
    t1 = T + 1
    frames = torch.randint(0, 256, (t1, B, 4, 84, 84), dtype=torch.uint8, generator=g)
    batch = dict(
        frame=frames,
        reward=torch.rand(t1, B, generator=g) * 2 - 1,
        done=torch.rand(t1, B, generator=g) < 0.05,
        episode_return=torch.randn(t1, B, generator=g),
        episode_step=torch.randint(0, 1000, (t1, B), generator=g),
        policy_logits=torch.randn(t1, B, A, generator=g),
        baseline=torch.randn(t1, B, generator=g),
        last_action=torch.randint(0, A, (t1, B), generator=g),
        action=torch.randint(0, A, (t1, B), generator=g),
    )
    return {k: v.to(device) for k, v in batch.items()}
