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


def learn_losses(model, batch, flags, core_state=()):
    """Upstream learn() up to total_loss (no optimiser); returns (total, parts, outputs)."""
    out, _ = model(batch, core_state)
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
    return total, (pg_loss, baseline_loss, entropy_loss), out


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
