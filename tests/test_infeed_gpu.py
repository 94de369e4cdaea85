"""DeviceInfeed (SURVEY 8f-2 rollout infeed): packed single-copy and per-field puts deliver
the host batch bit-exactly; learn() stats read back the episode returns of done rows."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_infeed_packed_and_per_field_puts():
    from oracle import atari_ref
    from paper_1910_03552_b200.learner import DeviceInfeed

    src = [atari_ref.synthetic_batch(6, 4, 6, seed=s) for s in range(3)]
    inf = DeviceInfeed(src[0], "cuda")
    packed = inf.alloc_host()
    assert packed["__flat__"].is_pinned()
    for k, v in src[0].items():
        packed[k].copy_(v)
    inf.put(packed)                                   # one H2D copy
    inf.put({k: v.pin_memory() for k, v in src[1].items()})  # per-field copies
    for want in src[:2]:
        got = inf.get()
        for k, v in want.items():
            assert torch.equal(got[k].cpu(), v), k
        inf.release()
    for k, v in src[2].items():
        packed[k].copy_(v)
    inf.put(packed)                                   # reuses slot 0 after release
    got = inf.get()
    assert all(torch.equal(got[k].cpu(), v) for k, v in src[2].items())


def test_learn_stats_episode_returns():
    from oracle import atari_ref
    from paper_1910_03552_b200 import learner, optim
    from paper_1910_03552_b200.atari_net import AtariNet

    flags = dict(atari_ref.DEFAULT_FLAGS)
    torch.manual_seed(0)
    net = AtariNet(num_actions=6)
    opt = optim.RMSprop(net.parameters(), lr=flags["learning_rate"], alpha=0.99, eps=0.01)
    batch = atari_ref.synthetic_batch(10, 4, 6, seed=2)
    batch["done"][3, 1] = True
    want = batch["episode_return"][1:][batch["done"][1:]]
    stats = learner.learn(flags, None, net, {k: v.cuda() for k, v in batch.items()}, (), opt, None)
    assert len(stats["episode_returns"]) == want.numel() >= 1
    assert torch.allclose(torch.tensor(stats["episode_returns"]), want)
    assert stats["mean_episode_return"] == pytest.approx(float(want.mean()), rel=1e-6)
