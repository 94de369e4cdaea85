"""The north-star loss helpers (losses.compute_policy_gradient_loss / compute_baseline_loss /
compute_entropy_loss, upstream monobeast signatures) on their fused kernels, pinned to the
golden vectors produced by running beastpipe itself (tests/golden/make_golden.py:
losses_from_targets vtrace.py:169-221 -> pg :194, baseline :195, entropy :196, d_logits
:208-214).  Bounds: each loss within 1e-5 of sum|terms| (pg terms cancel); gradients within
1e-5 of max|ref| (fp32 kernels vs the reference's own outputs; the fp64 cases set the scale)."""
import numpy as np
import pytest
import torch

from conftest import rel_err

pytestmark = pytest.mark.gpu

LOSS_TOL = 1e-5
GRAD_TOL = 1e-5


def _case(golden, idx):
    name = str(golden["loss/_names"][idx])
    g = {k.split("/", 2)[2]: v for k, v in golden.items() if k.startswith(f"loss/{name}/")}
    d, rho, c, bc, ec, pc = [float(x) for x in g["cfg"]]
    return name, g, dict(baseline_cost=bc, entropy_cost=ec, pg_cost=pc)


def _t(x, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


@pytest.mark.parametrize("idx", range(7))
def test_loss_helpers_match_reference_golden(golden, idx):
    from paper_1910_03552_b200 import losses

    name, g, costs = _case(golden, idx)
    T = int(g["T"])
    logits = _t(g["learner_logits"]).requires_grad_(True)
    actions = _t(g["action"][:T], torch.int64)  # beastpipe alignment: rows 0..T-1 (vtrace.py:243)
    adv = _t(g["pg_advantages"])
    vs = _t(g["vs"])
    values = _t(g["learner_baseline"][:-1]).requires_grad_(True)
    pg = losses.compute_policy_gradient_loss(logits, actions, adv, check=True)
    base = losses.compute_baseline_loss(vs - values)
    ent = losses.compute_entropy_loss(logits, check=True)
    assert pg.shape == () and pg.dtype == torch.float32
    # scales: sum |terms| (the pg terms cancel; baseline / entropy terms share a sign)
    lp = torch.log_softmax(torch.from_numpy(g["learner_logits"]).double(), -1)
    a = torch.from_numpy(g["action"][:T])
    pg_scale = float((lp.gather(-1, a[..., None])[..., 0] * torch.from_numpy(g["pg_advantages"]).double())
                     .abs().sum())
    ref = g["losses"]
    assert abs(float(pg) - ref[0]) <= LOSS_TOL * max(pg_scale, 1e-30), (name, float(pg), ref[0])
    assert abs(float(base) - ref[1]) <= LOSS_TOL * abs(ref[1]), (name, float(base), ref[1])
    assert abs(float(ent) - ref[2]) <= LOSS_TOL * max(abs(ref[2]), 1e-30), (name, float(ent), ref[2])
    # the reference total's gradients: pg_cost * pg + baseline_cost * base + entropy_cost * ent
    total = costs["pg_cost"] * pg + costs["baseline_cost"] * base + costs["entropy_cost"] * ent
    total.backward()
    assert rel_err(logits.grad.cpu().numpy(), g["d_logits"]) < GRAD_TOL, name
    d_base = np.zeros_like(g["d_baseline"])
    d_base[:-1] = values.grad.cpu().numpy()
    assert rel_err(d_base, g["d_baseline"]) < GRAD_TOL, name


@pytest.mark.parametrize("T,B,A", [(80, 32, 6), (80, 4096, 18), (3, 5, 1), (7, 3, 37)])
def test_loss_helpers_match_torch_fp64(T, B, A):
    """The upstream torch formulas in fp64 at the cfg sizes (incl. cfg4 T=80 B=4096 A=18)."""
    import torch.nn.functional as F

    from paper_1910_03552_b200 import losses

    g = torch.Generator().manual_seed(T * 1000 + B + A)
    x = torch.randn(T, B, A, generator=g) * 2
    act = torch.randint(0, A, (T, B), generator=g)
    adv = torch.randn(T, B, generator=g)
    x64 = x.double().requires_grad_(True)
    ce = F.nll_loss(F.log_softmax(x64.flatten(0, 1), -1), act.flatten(), reduction="none").view_as(adv)
    pg_ref = torch.sum(ce * adv.double())
    p = F.softmax(x64, -1)
    ent_ref = torch.sum(p * F.log_softmax(x64, -1))
    base_ref = 0.5 * torch.sum(adv.double() ** 2)
    (pg_ref + 0.01 * ent_ref).backward()
    xc = x.cuda().requires_grad_(True)
    advc = adv.cuda().requires_grad_(True)
    pg = losses.compute_policy_gradient_loss(xc, act.cuda(), advc, check=True)
    ent = losses.compute_entropy_loss(xc)
    base = losses.compute_baseline_loss(advc)
    (pg + 0.01 * ent).backward()
    base.backward()
    assert abs(float(pg) - float(pg_ref)) <= LOSS_TOL * float((ce * adv.double()).abs().sum())
    assert abs(float(ent) - float(ent_ref)) <= LOSS_TOL * abs(float(ent_ref))
    assert abs(float(base) - float(base_ref)) <= LOSS_TOL * float(base_ref)
    assert rel_err(xc.grad.cpu().numpy(), x64.grad.numpy()) < GRAD_TOL
    torch.testing.assert_close(advc.grad.cpu(), adv, rtol=1e-6, atol=1e-7)
    assert advc.grad is not None  # baseline grad only: the pg loss detaches advantages


def test_pg_loss_detaches_advantages_and_is_deterministic():
    from paper_1910_03552_b200 import losses

    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(80, 512, 18, device="cuda", generator=g)
    act = torch.randint(0, 18, (80, 512), device="cuda", generator=g)
    adv = torch.randn(80, 512, device="cuda", generator=g).requires_grad_(True)
    out = [losses.compute_policy_gradient_loss(x, act, adv) for _ in range(3)]
    assert all(torch.equal(o, out[0]) for o in out)
    out[0].backward()
    assert adv.grad is None


def test_pg_loss_action_out_of_range_raises():
    from paper_1910_03552_b200 import losses
    from paper_1910_03552_b200.errors import SchemaError

    x = torch.randn(4, 3, 6, device="cuda")
    act = torch.zeros(4, 3, dtype=torch.int64, device="cuda")
    act[2, 1] = 6
    with pytest.raises(SchemaError):
        losses.compute_policy_gradient_loss(x, act, torch.ones(4, 3, device="cuda"), check=True)
