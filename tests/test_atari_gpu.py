"""AtariNet on tcgen05 vs the torch-CPU fp32 oracle (oracle/atari_ref.py) with
identical weights.  The network runs bf16 operands / f32 accumulation; stated
bounds: against the fp32 upstream graph, logits / baseline relative L2 <= 1e-2 and
parameter gradients <= 2e-2 through the GPU's ReLU masks; against the bf16-emulating
oracle (oracle/atari_ref.emulated_forward), logits / baseline <= 1e-3 and every
parameter gradient <= 5e-3 end to end."""
import numpy as np
import pytest
import torch

from conftest import gpu_relu_masks, parity_log
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


def _oracle_grads(ref, batch, dl, db, masks=None):
    """Autograd gradients of sum(dl*logits + db*baseline); masks replace the ReLUs."""
    import torch.nn.functional as F

    n, A = dl.shape
    for p in ref.parameters():
        p.grad = None
    relu = [F.relu] * 4 if masks is None else [lambda z, m=m: z * m.to(z.dtype) for m in masks]
    x = batch["frame"].reshape(n, 4, 84, 84).float() / 255.0
    a1 = relu[0](ref.conv1(x))
    a2 = relu[1](ref.conv2(a1))
    a3 = relu[2](ref.conv3(a2))
    h = relu[3](ref.fc(a3.reshape(n, -1)))
    core = torch.cat([h, torch.clamp(batch["reward"].reshape(n, 1), -1, 1),
                      F.one_hot(batch["last_action"].reshape(n), A).float()], -1)
    torch.autograd.backward([ref.policy(core), ref.baseline(core).reshape(n)], [dl, db])
    return {k: p.grad.clone() for k, p in ref.named_parameters()}


def _gpu_grads(net, batch, dl, db):
    n = dl.shape[0]
    cb = {k: v.cuda() for k, v in batch.items()}
    net._forward_kernels(cb["frame"].reshape(n, 4, 84, 84), cb["reward"].reshape(n),
                         cb["last_action"].reshape(n))
    grads = torch.full_like(net.flat_params, float("nan"))
    net._backward_kernels(dl.cuda(), db.cuda(), cb["reward"].reshape(n), cb["last_action"].reshape(n),
                          grads)
    torch.cuda.synchronize()
    return net.torch_layout_grads(grads)


@pytest.mark.parametrize("T,B,A", [(2, 3, 6), (7, 16, 18), (80, 32, 6)])
def test_backward_matches_masked_oracle(T, B, A):
    """Kernel correctness: oracle backward through the GPU forward's own ReLU masks.
    Only bf16 operand rounding remains: every gradient within 2e-2 relative L2."""
    net, ref = _models(A, seed=3)
    batch = atari_ref.synthetic_batch(T, B, A, seed=2)
    n = (T + 1) * B
    g = torch.Generator().manual_seed(5)
    dl = torch.randn(n, A, generator=g)
    db = torch.randn(n, generator=g)
    got = _gpu_grads(net, batch, dl, db)
    want = _oracle_grads(ref, batch, dl, db, masks=gpu_relu_masks(net, n))
    errs = {k: rel_l2(got[k], w) for k, w in want.items()}
    assert all(torch.isfinite(v).all() for v in got.values())
    assert max(errs.values()) < 2e-2, errs


@pytest.mark.parametrize("T,B,A", [(7, 16, 18), (80, 32, 6)])
def test_forward_backward_match_bf16_emulating_oracle(T, B, A):
    """End to end against oracle/atari_ref.emulated_forward (fp64, the kernels' bf16 storage
    points restated; ReLU decisions adopted only inside the accumulation-ambiguity band):
    logits / baseline relative L2 <= 1e-3, every parameter gradient <= 5e-3."""
    import copy

    net, ref = _models(A, seed=3)
    batch = atari_ref.synthetic_batch(T, B, A, seed=2)
    n = (T + 1) * B
    g = torch.Generator().manual_seed(5)
    dl = torch.randn(n, A, generator=g)
    db = torch.randn(n, generator=g)
    cb = {k: v.cuda() for k, v in batch.items()}
    logits, base = net._forward_kernels(cb["frame"].reshape(n, 4, 84, 84), cb["reward"].reshape(n),
                                        cb["last_action"].reshape(n))
    logits, base = logits.clone(), base.clone()
    grads = torch.full_like(net.flat_params, float("nan"))
    net._backward_kernels(dl.cuda(), db.cuda(), cb["reward"].reshape(n), cb["last_action"].reshape(n), grads)
    torch.cuda.synchronize()
    got = net.torch_layout_grads(grads)
    ref64 = copy.deepcopy(ref).double().cuda()
    stats = {}
    out, _ = atari_ref.emulated_forward(ref64, cb, masks=gpu_relu_masks(net, n), mask_stats=stats)
    assert rel_l2(logits, out["policy_logits"].reshape(n, A)) < 1e-3
    assert rel_l2(base, out["baseline"].reshape(n)) < 1e-3
    torch.autograd.backward([out["policy_logits"].reshape(n, A), out["baseline"].reshape(n)],
                            [dl.double().cuda(), db.double().cuda()])
    errs = {k: rel_l2(got[k], p.grad) for k, p in ref64.named_parameters()}
    parity_log(f"atari bwd T={T} B={B} A={A}", dict(grad_rel_l2=errs, masks=stats))
    assert max(errs.values()) < 5e-3, errs
    assert all(s["disagree"] <= 1e-6 * s["total"] for s in stats.values()), stats


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
