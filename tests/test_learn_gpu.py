"""learn() determinism and weight-mirror bookkeeping.  Gradient / loss / update parity of
learn() against the bf16-emulating oracle is in test_learn_parity_gpu.py."""
import pytest
import torch

from oracle import atari_ref

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    a = a.double().cpu()
    b = b.double().cpu()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


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


def test_stats_after_several_unread_steps_and_in_place_batch_edit():
    """stats() waits for the LATEST step's pack (completion word), also when several steps ran
    without a stats read; an in-place edit of a batch tensor misses the memoised graph key
    (version counter) and still replays the right graph (same addresses) with the new data."""
    from paper_1910_03552_b200 import learner, optim
    from paper_1910_03552_b200.atari_net import AtariNet

    flags = dict(atari_ref.DEFAULT_FLAGS)
    torch.manual_seed(4)
    net = AtariNet(num_actions=6)
    opt = optim.RMSprop(net.parameters(), lr=flags["learning_rate"], alpha=0.99, eps=0.01)
    batch = {k: v.cuda() for k, v in atari_ref.synthetic_batch(8, 4, 6, seed=5).items()}
    L = learner.FusedLearner(net, flags, 8, 4)
    for _ in range(4):  # eager, capture + replay, replays; no stats read in between
        L.step(batch, opt)
    s1 = L.stats(batch)
    torch.cuda.synchronize()
    assert s1["total_loss"] == float(L.losses[3])
    key = L._graph_key(batch, opt)
    assert L._graph_key(batch, opt) is key  # memo hit
    batch["reward"].mul_(0.5)  # in place: bumps the version counter, same address
    key2 = L._graph_key(batch, opt)
    assert key2 == key and key2 is not key
    L.step(batch, opt)
    s2 = L.stats(batch)
    torch.cuda.synchronize()
    assert s2["total_loss"] == float(L.losses[3])
    assert len(L._graphs) == 1


def test_graph_capture_pauses_the_cyclic_collector():
    """A CUDA graph that only a reference cycle keeps alive is destroyed whenever the cyclic
    garbage collector runs; destroying a graph executable during a global-mode stream capture
    invalidates that capture.  The learner's and the actor-inference captures therefore run in
    _tensors.graph_capture, which pauses the automatic collector.  Here a graph becomes cyclic
    garbage in the middle of a capture while the collector would run at every allocation."""
    import gc

    from paper_1910_03552_b200._tensors import graph_capture

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    x = torch.zeros(4, device="cuda")
    dead = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(dead):
            x.add_(1.0)
    keep = [dead]
    del dead

    class Cycle:
        pass

    g = torch.cuda.CUDAGraph()
    thresholds = gc.get_threshold()
    gc.set_threshold(1, 1, 1)
    try:
        with torch.cuda.stream(s):
            with graph_capture(g):
                x.mul_(2.0)
                c = Cycle()
                c.graph, c.self = keep.pop(), c
                del c
                junk = [[i] for i in range(2000)]  # the automatic collector would run here
                del junk
                x.add_(3.0)
    finally:
        gc.set_threshold(*thresholds)
    torch.cuda.current_stream().wait_stream(s)
    x.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(x.cpu(), torch.full((4,), 3.0))
