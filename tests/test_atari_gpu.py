"""AtariNet on tcgen05 vs the torch-CPU fp32 oracle (oracle/atari_ref.py) with
identical weights.  The network runs bf16 operands / f32 accumulation, so the
stated bounds are relative L2 <= 1e-2 on logits / baseline and
<= 2e-2 on every parameter gradient."""
import numpy as np
import pytest
import torch

from oracle import atari_ref

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    a = a.double().cpu()
    b = b.double().cpu()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def _models(A, seed=0):
    from paper_1910_03552_b200.atari_net import AtariNet

    torch.manual_seed(seed)
    ref = atari_ref.AtariNetRef(num_actions=A)
    # non-zero heads / biases so every path carries signal
    with torch.no_grad():
        for p in ref.parameters():
            p.add_(0.05 * torch.randn_like(p))
    net = AtariNet(num_actions=A)
    net.load_state_dict(ref.state_dict())
    return net, ref


@pytest.mark.parametrize("T,B,A", [(2, 3, 6), (5, 8, 18), (80, 32, 6)])
def test_forward_matches_oracle(T, B, A):
    net, ref = _models(A)
    batch = atari_ref.synthetic_batch(T, B, A, seed=1)
    with torch.no_grad():
        want, _ = ref(batch)
        got, _ = net({k: v.cuda() for k, v in batch.items()})
    assert rel_l2(got["policy_logits"], want["policy_logits"]) < 1e-2
    assert rel_l2(got["baseline"], want["baseline"]) < 1e-2


@pytest.mark.parametrize("T,B,A", [(2, 3, 6), (7, 16, 18), (80, 32, 6)])
def test_backward_matches_oracle(T, B, A):
    net, ref = _models(A, seed=3)
    batch = atari_ref.synthetic_batch(T, B, A, seed=2)
    n = (T + 1) * B
    g = torch.Generator().manual_seed(5)
    dl = torch.randn(n, A, generator=g)
    db = torch.randn(n, generator=g)
    out, _ = ref(batch)
    torch.autograd.backward([out["policy_logits"].reshape(n, A), out["baseline"].reshape(n)],
                            [dl, db])
    want = {k: p.grad for k, p in ref.named_parameters()}
    cb = {k: v.cuda() for k, v in batch.items()}
    frames = cb["frame"].reshape(n, 4, 84, 84)
    net._forward_kernels(frames, cb["reward"].reshape(n), cb["last_action"].reshape(n))
    grads = torch.full_like(net.flat_params, float("nan"))
    net._backward_kernels(dl.cuda(), db.cuda(), cb["reward"].reshape(n), cb["last_action"].reshape(n),
                          grads)
    views = dict(zip([k for k, _ in net.named_parameters()], net._split(grads)))
    for k, w in want.items():
        assert torch.isfinite(views[k]).all(), k
        assert rel_l2(views[k], w) < 2e-2, (k, rel_l2(views[k], w))


def test_autograd_path_matches_kernels():
    net, ref = _models(6, seed=4)
    batch = {k: v.cuda() for k, v in atari_ref.synthetic_batch(3, 4, 6, seed=9).items()}
    out, _ = net(batch)
    loss = (out["policy_logits"] ** 2).sum() + out["baseline"].sum()
    net.flat_grads.zero_()
    loss.backward()
    auto = net.flat_grads.clone()
    n = 16
    dl = (2 * out["policy_logits"].detach()).reshape(n, 6)
    db = torch.ones(n, device="cuda")
    grads = torch.empty_like(net.flat_params)
    net._backward_kernels(dl, db, batch["reward"].reshape(n), batch["last_action"].reshape(n), grads)
    torch.testing.assert_close(auto, grads, rtol=1e-5, atol=1e-6)


def test_state_dict_roundtrip_is_upstream_compatible():
    net, ref = _models(18)
    sd = net.state_dict()
    assert set(sd) == set(ref.state_dict())
    for k, v in ref.state_dict().items():
        assert tuple(sd[k].shape) == tuple(v.shape)
        torch.testing.assert_close(sd[k].cpu(), v)


def test_sampling_kernel_distribution_and_greedy():
    net, _ = _models(6)
    logits = torch.tensor([[2.0, 0.0, -1.0, 0.5, -3.0, 1.0]], device="cuda").repeat(200_000, 1)
    acts = net.sample(logits, greedy=False).cpu().numpy()
    freq = np.bincount(acts, minlength=6) / len(acts)
    p = torch.softmax(logits[0], 0).cpu().numpy()
    assert np.abs(freq - p).max() < 5e-3
    greedy = net.sample(torch.randn(1000, 6, device="cuda"), greedy=True)
    assert (greedy.cpu() == 0).sum() < 1000  # not degenerate
    x = torch.randn(1000, 6, device="cuda")
    assert torch.equal(net.sample(x, greedy=True), x.argmax(1))
