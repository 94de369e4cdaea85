"""The whole fused learner step `learn()` vs the torch-CPU upstream restatement
(oracle/atari_ref.learn_step: autograd + clip_grad_norm_ + torch RMSprop).

bf16 network: the first step's losses (forward only) within 1e-2 relative;
the gradient norm within 5e-2; the parameter updates (RMSProp's first steps are
nearly sign(g)-like, so ReLU-flip noise in small gradients shows up in full)
compared by cosine similarity >= 0.9 per tensor."""
import pytest
import torch

from oracle import atari_ref

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    a = a.double().cpu()
    b = b.double().cpu()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


@pytest.mark.parametrize("T,B,A", [(4, 6, 6), (20, 8, 18)])
def test_learn_step_matches_upstream_restatement(T, B, A):
    from paper_1910_03552_b200 import learner, optim
    from paper_1910_03552_b200.atari_net import AtariNet

    flags = dict(atari_ref.DEFAULT_FLAGS)
    torch.manual_seed(0)
    ref = atari_ref.AtariNetRef(num_actions=A)
    with torch.no_grad():
        for p in ref.parameters():
            p.add_(0.05 * torch.randn_like(p))
    net = AtariNet(num_actions=A)
    net.load_state_dict(ref.state_dict())
    p0 = {k: v.detach().clone() for k, v in ref.named_parameters()}
    ropt = torch.optim.RMSprop(ref.parameters(), lr=flags["learning_rate"], alpha=flags["alpha"],
                               eps=flags["epsilon"])
    opt = optim.RMSprop(net.parameters(), lr=flags["learning_rate"], alpha=flags["alpha"],
                        eps=flags["epsilon"])
    for step in range(2):
        batch = atari_ref.synthetic_batch(T, B, A, seed=10 + step)
        total_ref, parts_ref, norm_ref = atari_ref.learn_step(ref, ropt, batch, flags)
        stats = learner.learn(flags, None, net, {k: v.cuda() for k, v in batch.items()}, (), opt,
                              None)
        if step == 0:
            assert abs(stats["total_loss"] - total_ref) <= 1e-2 * max(1.0, abs(total_ref))
            assert abs(stats["baseline_loss"] - parts_ref[1]) <= 1e-2 * abs(parts_ref[1])
        assert float(opt.norm) == pytest.approx(norm_ref, rel=5e-2)
    got = net.state_dict()  # upstream torch layout
    for k, v in ref.named_parameters():
        upd_ref = (v.detach() - p0[k]).double().reshape(1, -1)
        upd = (got[k].detach().cpu() - p0[k]).double().reshape(1, -1)
        cos = float(torch.nn.functional.cosine_similarity(upd, upd_ref))
        assert cos > 0.9, (k, cos)


def test_learn_is_repeatable_and_finite():
    from paper_1910_03552_b200 import learner, optim
    from paper_1910_03552_b200.atari_net import AtariNet

    flags = dict(atari_ref.DEFAULT_FLAGS)
    outs = []
    for _ in range(2):
        torch.manual_seed(1)
        net = AtariNet(num_actions=6)
        opt = optim.RMSprop(net.parameters(), lr=flags["learning_rate"], alpha=0.99, eps=0.01)
        batch = {k: v.cuda() for k, v in atari_ref.synthetic_batch(80, 32, 6, seed=3).items()}
        for _ in range(3):
            stats = learner.learn(flags, None, net, batch, (), opt, None)
        assert all(map(lambda x: x == x, [stats["total_loss"], stats["pg_loss"]]))
        outs.append(net.flat_params.clone())
    assert torch.equal(outs[0], outs[1]), "fused learner step must be deterministic"


def test_learn_after_load_state_dict_uses_new_weights():
    """The bf16 operand mirror must follow load_state_dict, also on graph replays."""
    from paper_1910_03552_b200 import learner, optim
    from paper_1910_03552_b200.atari_net import AtariNet

    flags = dict(atari_ref.DEFAULT_FLAGS)
    torch.manual_seed(2)
    net = AtariNet(num_actions=6)
    opt = optim.RMSprop(net.parameters(), lr=flags["learning_rate"], alpha=0.99, eps=0.01)
    batch = {k: v.cuda() for k, v in atari_ref.synthetic_batch(4, 4, 6, seed=1).items()}
    for _ in range(3):  # eager, capture, replay
        learner.learn(flags, None, net, batch, (), opt, None)
    ref = atari_ref.AtariNetRef(num_actions=6)
    net.load_state_dict(ref.state_dict())
    ropt = torch.optim.RMSprop(ref.parameters(), lr=flags["learning_rate"], alpha=0.99, eps=0.01)
    total_ref, _, _ = atari_ref.learn_step(ref, ropt, {k: v.cpu() for k, v in batch.items()}, flags)
    stats = learner.learn(flags, None, net, batch, (), opt, None)  # graph replay path
    assert abs(stats["total_loss"] - total_ref) <= 1e-2 * max(1.0, abs(total_ref))
