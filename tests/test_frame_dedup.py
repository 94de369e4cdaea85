"""Frame-stack dedup: the learner batch ships each raw 84x84 plane once
(a (T+4, B) plane store + a (T+1, B, 4) int32 plane index) instead of (T+1)*B*4 stacked
planes (np.stack at enqueue, rollout.py:116-144).  The index follows upstream
TorchBeast FrameStack(4): channel c of frame t is the plane of step t-3+c, and a reset
(done[t]) replicates the reset plane.  The GPU path must be bit-identical to the
stacked-frame path (same u8 bytes reach the same GEMMs)."""
import pytest
import torch

from paper_1910_03552_b200 import rollout
from paper_1910_03552_b200.errors import SchemaError


def framestack_batch(T, B, A, seed=0, p_done=0.1):
    """Synthetic batch whose frames really are FrameStack(4) data built from random planes."""
    from oracle import atari_ref

    batch = atari_ref.synthetic_batch(T, B, A, seed=seed)
    g = torch.Generator().manual_seed(seed + 1000)
    done = torch.rand(T + 1, B, generator=g) < p_done
    planes = torch.randint(0, 256, (T + 4, B, 84, 84), dtype=torch.uint8, generator=g)
    index = rollout.frame_stack_index(done)
    batch["done"] = done
    batch["frame"] = rollout.stack_frames(planes, index)
    return batch, planes, index


def test_frame_stack_index_semantics():
    T, B = 5, 2
    done = torch.zeros(T + 1, B, dtype=torch.bool)
    done[2, 0] = True
    idx = rollout.frame_stack_index(done)
    assert idx.dtype == torch.int32 and tuple(idx.shape) == (T + 1, B, 4)
    rows = (idx // B).tolist()
    assert rows[0][1] == [0, 1, 2, 3]            # no reset: planes t .. t+3 (step t-3 .. t)
    assert rows[5][1] == [5, 6, 7, 8]
    assert rows[2][0] == [5, 5, 5, 5]            # reset at t=2: 4 copies of the reset plane
    assert rows[3][0] == [5, 5, 5, 6]
    assert rows[5][0] == [5, 6, 7, 8]            # history no longer reaches before the reset
    assert ((idx % B) == torch.arange(B).view(1, B, 1)).all()


def test_dedup_round_trip_and_bytes():
    batch, planes, index = framestack_batch(20, 4, 6, seed=3)
    p2, i2 = rollout.dedup_frames(batch["frame"], batch["done"])
    assert torch.equal(i2, index)
    assert torch.equal(rollout.stack_frames(p2, i2), batch["frame"])
    full = batch["frame"].numel()
    assert p2.numel() * 4 <= full * (24 / 21) + 1  # (T+4)/(T+1) / 4 of the stacked bytes


def test_dedup_rejects_non_framestack_batches():
    from oracle import atari_ref

    batch = atari_ref.synthetic_batch(4, 2, 6, seed=1)  # independent random planes
    with pytest.raises(SchemaError):
        rollout.dedup_frames(batch["frame"], batch["done"])


@pytest.mark.gpu
@pytest.mark.parametrize("use_lstm", [False, True])
def test_forward_planes_bit_identical(use_lstm):
    from paper_1910_03552_b200.atari_net import AtariNet

    T, B, A = 6, 4, 6
    batch, planes, index = framestack_batch(T, B, A, seed=5)
    torch.manual_seed(0)
    net = AtariNet(num_actions=A, use_lstm=use_lstm)
    n = (T + 1) * B
    frames = batch["frame"].cuda().reshape(n, 4, 84, 84)
    reward = batch["reward"].cuda().reshape(n)
    la = batch["last_action"].cuda().reshape(n)
    lstm = None
    if use_lstm:
        st = net.initial_state(B)
        lstm = dict(T1=T + 1, B=B, done=batch["done"].cuda().reshape(n).view(torch.uint8), h0=st[0], c0=st[1])
    l0, b0 = net._forward_kernels(frames, reward, la, repack=True, lstm=dict(lstm) if lstm else None)
    l0, b0 = l0.clone(), b0.clone()
    l1, b1 = net._forward_kernels(planes.cuda(), reward, la, repack=False, lstm=dict(lstm) if lstm else None,
                                  plane_index=index.cuda().reshape(n, 4))
    assert torch.equal(l0, l1) and torch.equal(b0, b1)


@pytest.mark.gpu
def test_learn_with_plane_store_matches_stacked_frames():
    from oracle import atari_ref
    from paper_1910_03552_b200 import learner, optim
    from paper_1910_03552_b200.atari_net import AtariNet

    flags = dict(atari_ref.DEFAULT_FLAGS)
    T, B, A = 20, 8, 6
    batch, planes, index = framestack_batch(T, B, A, seed=7)
    dev = {k: v.cuda() for k, v in batch.items()}
    ded = {k: v for k, v in dev.items() if k != "frame"}
    ded["frame_planes"], ded["frame_index"] = planes.cuda(), index.cuda()
    outs = []
    for b in (dev, ded):
        torch.manual_seed(4)
        net = AtariNet(num_actions=A)
        opt = optim.RMSprop(net.parameters(), lr=flags["learning_rate"], alpha=0.99, eps=0.01)
        for _ in range(3):  # eager, graph capture, graph replay
            stats = learner.learn(flags, None, net, b, (), opt, None)
        outs.append((stats["total_loss"], net.flat_params.clone()))
    assert outs[0][0] == outs[1][0]
    assert torch.equal(outs[0][1], outs[1][1])
