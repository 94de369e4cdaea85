"""Pin the torch-CPU network oracle (oracle/atari_ref.py), CPU only.

The AtariNet itself has no reference counterpart (parity unpinned by the
reference); its loss path is tied here to the golden-pinned numpy oracle
(oracle/vtrace_np.compute_losses with TorchBeast row alignment) and its
gradients to finite differences (reference methodology, conftest.py:5-26)."""
import numpy as np
import torch

from conftest import assert_grads_close
from oracle import atari_ref
from oracle import vtrace_np as ov


def test_learn_losses_equal_numpy_oracle():
    torch.manual_seed(0)
    T, B, A = 5, 3, 6
    model = atari_ref.AtariNetRef(num_actions=A).double()
    batch = atari_ref.synthetic_batch(T, B, A, seed=4)
    batch = {k: (v.double() if v.dtype == torch.float32 else v) for k, v in batch.items()}
    flags = dict(atari_ref.DEFAULT_FLAGS)
    total, (pg, base, ent), out = atari_ref.learn_losses(model, batch, flags)
    cfg = ov.VtraceConfig(discount=flags["discounting"], baseline_cost=flags["baseline_cost"],
                          entropy_cost=flags["entropy_cost"])
    logits = out["policy_logits"].detach().numpy()
    baseline = out["baseline"].detach().numpy()
    bundle, d_logits, d_baseline, _, _ = ov.compute_losses(
        batch["reward"].numpy(), batch["done"].numpy(), batch["policy_logits"].numpy(),
        batch["action"].numpy(), logits[:-1], baseline, cfg, shift=1, reward_clip=True)
    np.testing.assert_allclose(float(pg), bundle.pg_loss, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(float(base), cfg.baseline_cost * bundle.baseline_loss, rtol=1e-9)
    np.testing.assert_allclose(float(ent), cfg.entropy_cost * bundle.entropy_loss, rtol=1e-9)
    np.testing.assert_allclose(float(total), bundle.total, rtol=1e-9)
    # gradient of the torch restatement w.r.t. its logits / baseline == numpy oracle's
    lg = out["policy_logits"]
    bl = out["baseline"]
    lg.retain_grad()
    bl.retain_grad()
    total.backward()
    np.testing.assert_allclose(lg.grad.numpy()[:-1], d_logits, rtol=1e-9, atol=1e-12)
    np.testing.assert_array_equal(lg.grad.numpy()[-1], 0.0)
    np.testing.assert_allclose(bl.grad.numpy(), d_baseline, rtol=1e-9, atol=1e-12)


def test_network_gradient_finite_differences():
    torch.manual_seed(1)
    model = atari_ref.AtariNetRef(num_actions=4).double()
    batch = atari_ref.synthetic_batch(1, 2, 4, seed=5)
    g = torch.Generator().manual_seed(2)
    up_l = torch.randn(4, 4, generator=g, dtype=torch.float64)
    up_b = torch.randn(4, generator=g, dtype=torch.float64)

    def objective():
        out, _ = model(batch)
        return float((out["policy_logits"].reshape(4, 4) * up_l).sum()
                     + (out["baseline"].reshape(4) * up_b).sum())

    out, _ = model(batch)
    ((out["policy_logits"].reshape(4, 4) * up_l).sum() + (out["baseline"].reshape(4) * up_b).sum()).backward()
    for name in ("policy.weight", "baseline.bias", "fc.bias"):
        p = dict(model.named_parameters())[name]
        idx = [0, p.numel() // 2, p.numel() - 1]
        flat = p.data.view(-1)
        for i in idx:
            orig = float(flat[i])
            flat[i] = orig + 1e-6
            up = objective()
            flat[i] = orig - 1e-6
            dn = objective()
            flat[i] = orig
            fd = (up - dn) / 2e-6
            assert_grads_close(np.array([float(p.grad.view(-1)[i])]), np.array([fd]), rtol=1e-4)
