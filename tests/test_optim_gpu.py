"""GPU parity of the fused clip + RMSProp kernels.

Against (1) the reference's own outputs (golden: beastpipe clip_global_norm +
rmsprop_step), (2) torch.optim.RMSprop + clip_grad_norm_ (upstream learn()).
Elementwise tolerance 1e-6 relative (fp32), SURVEY 8c.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_mirrors_match_reference_golden(golden):
    from paper_1910_03552_b200 import optim

    fields = [str(f) for f in golden["opt/_fields"]]
    for i in range(int(golden["opt/_n"])):
        g = {k.split("/", 2)[2]: v for k, v in golden.items() if k.startswith(f"opt/{i}/")}
        max_norm, lr, decay, eps = [float(x) for x in g["hyper"]]
        clipped, norm = optim.clip_global_norm([g[f"g_{f}"] for f in fields], max_norm)
        assert norm == pytest.approx(float(g["norm"]), rel=1e-6)
        newp, news = optim.rmsprop_step([g[f"p_{f}"] for f in fields], clipped,
                                        [g[f"s_{f}"] for f in fields], lr, decay, eps)
        for f, p, s in zip(fields, newp, news):
            np.testing.assert_allclose(p, g[f"np_{f}"], rtol=1e-6, atol=1e-6)
            np.testing.assert_allclose(s, g[f"ns_{f}"], rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("n_params,max_norm", [([1000, 33, 7], 40.0), ([1_694_000, 512, 3], 0.5),
                                               ([6_214_001], 1e6)])
def test_fused_rmsprop_matches_torch(n_params, max_norm):
    from paper_1910_03552_b200 import optim

    g = torch.Generator(device="cuda").manual_seed(1)
    ps = [torch.nn.Parameter(torch.randn(n, device="cuda", generator=g)) for n in n_params]
    ref = [torch.nn.Parameter(p.detach().clone()) for p in ps]
    opt = optim.RMSprop(ps, lr=0.00048, alpha=0.99, eps=0.01)
    topt = torch.optim.RMSprop(ref, lr=0.00048, alpha=0.99, eps=0.01)
    for step in range(3):
        grads = [torch.randn(n, device="cuda", generator=g) * 3 for n in n_params]
        for p, r, gr in zip(ps, ref, grads):
            p.grad.copy_(gr)
            r.grad = gr.clone()
        opt.step(max_norm=max_norm)
        tn = torch.nn.utils.clip_grad_norm_(ref, max_norm)
        topt.step()
        assert opt.norm.item() == pytest.approx(tn.item(), rel=1e-5)
        for p, r in zip(ps, ref):
            torch.testing.assert_close(p.detach(), r.detach(), rtol=1e-6, atol=1e-6)
            torch.testing.assert_close(p.grad, r.grad, rtol=1e-6, atol=1e-7)
        for p, r in zip(ps, ref):
            # torch's addcmul_ rounds alpha*s + (1-alpha)*g*g differently: 1e-5 relative
            torch.testing.assert_close(opt.state[p]["square_avg"], topt.state[r]["square_avg"],
                                       rtol=1e-5, atol=1e-9)


def test_nonfinite_gradient_rejects_step():
    from paper_1910_03552_b200 import optim
    from paper_1910_03552_b200._tensors import status_word
    from paper_1910_03552_b200.errors import NonFiniteError

    p = torch.nn.Parameter(torch.ones(100, device="cuda"))
    opt = optim.RMSprop([p], lr=0.1, alpha=0.99, eps=0.01)
    p.grad.fill_(1.0)
    p.grad[5] = float("nan")
    before = p.detach().clone()
    opt.step(max_norm=40.0)
    with pytest.raises(NonFiniteError):
        status_word(p.device).check()
    assert torch.equal(p.detach(), before)


def test_sumsq_deterministic_and_exact_enough():
    from paper_1910_03552_b200 import optim

    x = torch.randn(10_000_019, device="cuda")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    vals = [optim.sumsq_(x, out).item() for _ in range(3)]
    assert vals[0] == vals[1] == vals[2]
    ref = float((x.double() ** 2).sum())
    assert vals[0] == pytest.approx(ref, rel=1e-6)
    # misaligned view takes the scalar path
    optim.sumsq_(x[1:], out)
    assert out.item() == pytest.approx(float((x[1:].double() ** 2).sum()), rel=1e-6)
