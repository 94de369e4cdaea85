"""learn()'s error contract (the reference's train_batch): a batch that violates the schema
raises SchemaError (validate_batch, rollout.py:160-192: action outside [0, A), non-finite
reward / policy_logits, done not bool); a non-finite loss dumps the batch to
<logdir>/diagnostic_batch.npz and raises NonFiniteError (pipeline.py:333-338, vtrace.py:202-205).
In every case the parameters and the optimiser state are left untouched (model.py:251-252), on
the eager path and on CUDA-graph replays, and the next clean step trains normally."""
import os

import numpy as np
import pytest
import torch

from oracle import atari_ref

pytestmark = pytest.mark.gpu


def _setup(T=6, B=4, A=6, seed=0):
    from paper_1910_03552_b200 import optim
    from paper_1910_03552_b200.atari_net import AtariNet

    torch.manual_seed(seed)
    net = AtariNet(num_actions=A)
    opt = optim.RMSprop(net.parameters(), lr=4.8e-4, alpha=0.99, eps=0.01)
    batch = {k: v.cuda() for k, v in atari_ref.synthetic_batch(T, B, A, seed=seed + 1).items()}
    return net, opt, batch


def _corrupt(batch, kind):
    if kind == "nan_reward":
        batch["reward"][3, 1] = float("nan")
    elif kind == "inf_logit":
        batch["policy_logits"][2, 0, 1] = float("inf")
    elif kind == "action_range":
        batch["action"][4, 2] = batch["policy_logits"].shape[-1]
    elif kind == "negative_action":
        batch["action"][1, 3] = -1
    else:
        raise ValueError(kind)


@pytest.mark.parametrize("kind", ["nan_reward", "inf_logit", "action_range", "negative_action"])
@pytest.mark.parametrize("replay", [False, True], ids=["eager", "graph"])
def test_schema_violation_raises_and_leaves_params(kind, replay):
    from paper_1910_03552_b200 import learner
    from paper_1910_03552_b200.errors import SchemaError

    flags = dict(atari_ref.DEFAULT_FLAGS)
    net, opt, batch = _setup()
    clean = {k: v.clone() for k, v in batch.items()}
    if replay:  # eager + capture on these very buffers, so the bad step is a graph replay
        for _ in range(2):
            learner.learn(flags, None, net, batch, (), opt, None)
    p0, s0 = net.flat_params.clone(), opt.square_avg.clone()
    _corrupt(batch, kind)
    with pytest.raises(SchemaError):
        learner.learn(flags, None, net, batch, (), opt, None)
    torch.cuda.synchronize()
    assert torch.equal(net.flat_params, p0), "parameters changed by a rejected step"
    assert torch.equal(opt.square_avg, s0), "square_avg changed by a rejected step"
    if replay:
        L = next(iter(net._fused_learners.values()))
        assert len(L._graphs) == 1, "the bad step must have run the captured graph"
    # the status word was cleared: the next clean step trains
    for k, v in clean.items():
        batch[k].copy_(v)
    stats = learner.learn(flags, None, net, batch, (), opt, None)
    assert np.isfinite(stats["total_loss"])
    assert not torch.equal(net.flat_params, p0)


def test_nonfinite_loss_dumps_batch_and_raises(tmp_path):
    from paper_1910_03552_b200 import learner
    from paper_1910_03552_b200.errors import NonFiniteError

    flags = dict(atari_ref.DEFAULT_FLAGS, logdir=str(tmp_path))
    net, opt, batch = _setup(seed=3)
    with torch.no_grad():
        net.fc.bias[7] = float("inf")  # the network's own outputs turn non-finite
    p0 = net.flat_params.clone()
    with pytest.raises(NonFiniteError) as ei:
        learner.learn(flags, None, net, batch, (), opt, None)
    torch.cuda.synchronize()
    path = os.path.join(str(tmp_path), "diagnostic_batch.npz")
    assert os.path.exists(path)
    assert any("diagnostic_batch.npz" in n for n in getattr(ei.value, "__notes__", []))
    dumped = np.load(path)
    assert np.array_equal(dumped["action"], batch["action"].cpu().numpy())
    assert torch.equal(net.flat_params, p0), "parameters changed by a rejected step"


def test_done_must_be_bool():
    from paper_1910_03552_b200 import learner
    from paper_1910_03552_b200.errors import SchemaError

    flags = dict(atari_ref.DEFAULT_FLAGS)
    net, opt, batch = _setup(seed=5)
    batch["done"] = batch["done"].to(torch.uint8)
    with pytest.raises(SchemaError, match="done"):
        learner.learn(flags, None, net, batch, (), opt, None)


def test_graph_cache_keys_on_dtype_and_is_bounded():
    """A batch at the same addresses but another layout is validated again (not replayed);
    the number of captured graphs stays bounded with fresh batches every step."""
    from paper_1910_03552_b200 import learner

    flags = dict(atari_ref.DEFAULT_FLAGS)
    net, opt, _ = _setup(seed=6)
    for i in range(3 * learner.MAX_GRAPHS):
        batch = {k: v.cuda() for k, v in atari_ref.synthetic_batch(6, 4, 6, seed=100 + (i // 2)).items()}
        learner.learn(flags, None, net, batch, (), opt, None)
    L = next(iter(net._fused_learners.values()))
    assert len(L._graphs) <= learner.MAX_GRAPHS


def test_buffer_reallocation_drops_captured_graphs():
    """A forward over more frames reallocates the activation buffers; a learner's graphs that
    captured the old addresses must not replay (use-after-free)."""
    from paper_1910_03552_b200 import learner

    flags = dict(atari_ref.DEFAULT_FLAGS)
    net, opt, batch = _setup(seed=7)
    for _ in range(3):
        learner.learn(flags, None, net, batch, (), opt, None)
    L = next(iter(net._fused_learners.values()))
    assert len(L._graphs) == 1
    gen = net.buffer_generation
    big = {k: v.cuda() for k, v in atari_ref.synthetic_batch(20, 8, 6, seed=9).items()}
    with torch.no_grad():
        net(big)
    assert net.buffer_generation > gen
    p_before = net.flat_params.clone()
    stats = learner.learn(flags, None, net, batch, (), opt, None)
    assert len(L._graphs) == 0 and np.isfinite(stats["total_loss"])
    assert not torch.equal(net.flat_params, p_before)


@pytest.mark.parametrize("sumsq,total,want", [(float("inf"), 1.0, 16), (float("nan"), 1.0, 16),
                                              (4.0, 1.0, 0), (float("inf"), float("nan"), 0)])
def test_stats_pack_derives_the_update_verdict(sumsq, total, want):
    """The pack beside the RMSProp update reports BP_STATUS_NONFINITE_GRAD exactly when the
    update rejects for a non-finite norm (rmsprop_kernel: non-finite norm, finite total loss;
    a non-finite total is reported by the loss kernel's own bit instead)."""
    from paper_1910_03552_b200 import _native as N

    tb = 8
    losses = torch.tensor([0.5, 0.25, -0.1, total], dtype=torch.float64, device="cuda")
    done = torch.zeros(tb, dtype=torch.uint8, device="cuda")
    ss = torch.tensor([sumsq], dtype=torch.float64, device="cuda")
    status = torch.tensor([4], dtype=torch.int32, device="cuda")  # a bit the loss kernel set
    seq = torch.zeros(2, dtype=torch.int32, device="cuda")
    out = torch.zeros(40 + 5 * tb, dtype=torch.uint8).pin_memory()
    N.check(N.lib().bp_pack_stats(losses.data_ptr(), done.data_ptr(), None, tb, status.data_ptr(), ss.data_ptr(),
                                  seq.data_ptr(), out.data_ptr(), N.stream_handle()), "bp_pack_stats")
    torch.cuda.synchronize()
    words = out[:40].numpy().view(np.uint32)
    assert words[8] == 4 | want and words[9] == 1
    assert int(status.item()) == 0  # read, then cleared for the next step
