"""Actor inference (§8f-1): the fused heads-epilogue sampler and the variable-k / graph paths.

Pins:
  * the fused sampler (bp_atari_forward_sample) draws exactly the standalone sampler's
    actions (bp_sample_actions_f32) for the same seed, and both follow the numpy Philox
    restatement (oracle/sample_np.py, itself pinned to the Philox known-answer vectors);
  * greedy = argmax of the returned logits, bit-exact;
  * a dynamic batch of k observations gives, row for row, the same logits / baseline as the
    full batch (rows are independent: bit-identical), on the eager path and on graph replays;
  * graph replays draw fresh actions (device-resident key advances) with the right law;
  * the LSTM actor step (T = 1, core_state carried) equals one T-step forward and the
    bf16-emulating oracle.
The reference loop: pipeline.py:609-634 (mlp_forward + sample_actions, model.py:218-221)."""
import numpy as np
import pytest
import torch

from oracle import atari_ref, sample_np

pytestmark = pytest.mark.gpu


def _net(A, use_lstm=False, seed=0):
    from paper_1910_03552_b200.atari_net import AtariNet

    torch.manual_seed(seed)
    ref = atari_ref.AtariNetRef(num_actions=A, use_lstm=use_lstm)
    with torch.no_grad():
        for p in ref.parameters():
            p.add_(0.05 * torch.randn_like(p))
    net = AtariNet(num_actions=A, use_lstm=use_lstm)
    net.load_state_dict(ref.state_dict())
    return net, ref


def _obs(k, A, seed):
    b = atari_ref.synthetic_batch(0, k, A, seed=seed)
    return {key: v[0].cuda() for key, v in b.items()}


@pytest.mark.parametrize("k,A", [(1, 6), (100, 6), (1024, 18), (333, 31)])
def test_fused_sampler_matches_standalone_and_oracle(k, A):
    net, _ = _net(A)
    net.eval()
    o = _obs(k, A, seed=k)
    actions = torch.empty(k, dtype=torch.int64, device="cuda")
    seed = 0x1234_5678_9ABC_DEF0 + k
    logits, _ = net._forward_kernels(o["frame"], o["reward"], o["last_action"], keep_x0=False,
                                     actions=actions, seed=seed, repack=True)
    standalone = net.sample(logits, greedy=False, seed=seed)
    assert torch.equal(actions, standalone)
    ref = sample_np.sample_actions(logits.cpu().numpy(), seed)
    assert (actions.cpu().numpy() == ref).mean() >= 0.999  # f32 vs f64 log rounding near ties only
    greedy = torch.empty_like(actions)
    net._forward_kernels(o["frame"], o["reward"], o["last_action"], keep_x0=False, actions=greedy, seed=seed,
                         greedy=True)
    assert torch.equal(greedy, logits.argmax(1))


def test_fused_sampler_law():
    """Gumbel-max law through the fused path: 4096 identical observations, 8 calls."""
    net, _ = _net(6)
    o = _obs(1, 6, seed=2)
    k = 4096
    frames = o["frame"].expand(k, 4, 84, 84).contiguous()
    reward, last = o["reward"].expand(k).contiguous(), o["last_action"].expand(k).contiguous()
    counts = np.zeros(6)
    logits = None
    for _ in range(8):
        actions = torch.empty(k, dtype=torch.int64, device="cuda")
        logits, _ = net._forward_kernels(frames, reward, last, keep_x0=False, actions=actions,
                                         seed=net.next_sample_seed(), repack=True)
        counts += np.bincount(actions.cpu().numpy(), minlength=6)
    p = torch.softmax(logits[0].double(), 0).cpu().numpy()
    assert np.abs(counts / counts.sum() - p).max() < 1.2e-2


@pytest.mark.parametrize("use_lstm", [False, True], ids=["ff", "lstm"])
def test_variable_k_eager_and_graphs_match_full_batch(use_lstm):
    from paper_1910_03552_b200.inference import ActorInference

    A = 18
    net, _ = _net(A, use_lstm=use_lstm, seed=3)
    net.eval()
    K = 256
    o = _obs(K, A, seed=5)
    H = net.core_hidden
    g = torch.Generator().manual_seed(1)
    state = tuple((0.5 * torch.randn(2, K, H, generator=g)).cuda() for _ in range(2)) if use_lstm else ()
    full = ActorInference(net)
    out_full, st_full = full({k: v[None] for k, v in o.items()}, state)
    eager = ActorInference(net)
    graphs = ActorInference(net, graph_buckets=(1, 32, 256))
    for lo, hi in [(0, 1), (1, 33), (40, 47), (0, 256)]:
        sub = {k: v[None, lo:hi] for k, v in o.items()}
        sst = tuple(s[:, lo:hi] for s in state)
        for inf in (eager, graphs):
            out, st = inf(sub, sst)
            kk = hi - lo
            assert out["action"].shape == (1, kk) and out["policy_logits"].shape == (1, kk, A)
            assert out["model_version"].shape == (1, kk)
            assert torch.equal(out["policy_logits"][0], out_full["policy_logits"][0, lo:hi])
            assert torch.equal(out["baseline"][0], out_full["baseline"][0, lo:hi])
            assert out["action"].min() >= 0 and out["action"].max() < A
            if use_lstm:
                for a, b in zip(st, st_full):
                    assert torch.equal(a, b[:, lo:hi])


def test_graph_replays_draw_fresh_actions():
    from paper_1910_03552_b200.inference import ActorInference

    net, _ = _net(6, seed=4)
    inf = ActorInference(net, graph_buckets=(1024,))
    o = _obs(1, 6, seed=9)
    k = 1000
    obs = {"frame": o["frame"].expand(k, 4, 84, 84)[None], "reward": o["reward"].expand(k)[None],
           "last_action": o["last_action"].expand(k)[None]}
    draws = [inf(obs)[0] for _ in range(6)]
    acts = torch.stack([d["action"][0] for d in draws])
    assert not torch.equal(acts[0], acts[1])
    p = torch.softmax(draws[0]["policy_logits"][0, 0].double(), 0).cpu().numpy()
    freq = np.bincount(acts.flatten().cpu().numpy(), minlength=6) / acts.numel()
    assert np.abs(freq - p).max() < 2.5e-2


def test_lstm_actor_steps_equal_one_unroll_and_oracle():
    """T = 1 actor steps carrying core_state == one T-step forward (bitwise) == oracle."""
    from paper_1910_03552_b200.inference import ActorInference

    A, B, T = 6, 16, 5
    net, ref = _net(A, use_lstm=True, seed=6)
    net.eval()
    H = net.core_hidden
    batch = atari_ref.synthetic_batch(T - 1, B, A, seed=11)
    batch["done"][2, :4] = True
    g = torch.Generator().manual_seed(2)
    state0 = tuple(0.5 * torch.randn(2, B, H, generator=g) for _ in range(2))
    cb = {k: v.cuda() for k, v in batch.items()}
    with torch.no_grad():
        unroll, st_unroll = net(cb, tuple(s.cuda() for s in state0))
    inf = ActorInference(net, graph_buckets=(16,))
    state = tuple(s.cuda() for s in state0)
    for t in range(T):
        out, state = inf({k: v[t:t + 1] for k, v in cb.items()}, state)
        assert torch.equal(out["policy_logits"][0], unroll["policy_logits"][t])
        assert torch.equal(out["baseline"][0], unroll["baseline"][t])
    for a, b in zip(state, st_unroll):
        assert torch.equal(a, b)
    refd = ref.double()
    with torch.no_grad():
        emu, st_emu = atari_ref.emulated_forward(refd, {k: (v.double() if v.is_floating_point() else v)
                                                        for k, v in batch.items()},
                                                 tuple(s.double() for s in state0))
    got = unroll["policy_logits"].double().cpu()
    want = emu["policy_logits"]
    assert float((got - want).norm() / want.norm()) < 4e-3
    assert float((state[0].double().cpu() - st_emu[0]).norm() / st_emu[0].norm()) < 4e-3


@pytest.mark.parametrize("k,A", [(1, 6), (100, 18), (256, 31)])
def test_small_batch_inference_tail_matches_gemm_path(k, A):
    """k <= 256: the split-K fc + CUDA-core heads tail (bp_atari_forward_sample) against the
    tcgen05 fc epilogue + heads GEMM of the plain forward (same bf16 operands, different f32
    summation order): logits / baseline within 1e-3 relative L2; against the bf16-emulating
    oracle without adopting the kernel's near-zero ReLU decisions: 2e-3; greedy actions =
    argmax of the returned logits."""
    net, ref = _net(A, seed=8)
    batch = atari_ref.synthetic_batch(0, k, A, seed=k + 3)
    o = {key: v[0].cuda() for key, v in batch.items()}
    actions = torch.empty(k, dtype=torch.int64, device="cuda")
    small, sb = net._forward_kernels(o["frame"], o["reward"], o["last_action"], keep_x0=False,
                                     actions=actions, seed=7, greedy=True, repack=True)
    small, sb = small.clone(), sb.clone()
    gemm, gb = net._forward_kernels(o["frame"], o["reward"], o["last_action"], keep_x0=True, repack=True)
    rel = lambda a, b: float((a.double().cpu() - b.double().cpu()).norm() / b.double().cpu().norm())  # noqa: E731
    assert rel(small, gemm) <= 1e-3 and rel(sb, gb) <= 1e-3
    assert torch.equal(actions, small.argmax(1))
    with torch.no_grad():
        emu, _ = atari_ref.emulated_forward(ref.double(), {key: (v.double() if v.is_floating_point() else v)
                                                           for key, v in batch.items()})
    assert rel(small, emu["policy_logits"][0]) <= 2e-3
    assert rel(sb, emu["baseline"][0]) <= 2e-3
