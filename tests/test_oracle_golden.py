"""Pin the CPU oracle (oracle/) against the reference: golden vectors produced by
running beastpipe itself (tests/golden/make_golden.py) plus the hand-derived
known answers of the reference's own tests.  CPU only."""
import numpy as np
import pytest

from conftest import assert_grads_close, central_difference
from oracle import model_np as om
from oracle import vtrace_np as ov


def _cfg(arr):
    d, rho, c, bc, ec, pc = [float(x) for x in arr]
    return ov.VtraceConfig(discount=d, rho_bar=rho, c_bar=c, baseline_cost=bc, entropy_cost=ec,
                           pg_cost=pc)


@pytest.mark.parametrize("idx", range(7))
def test_compute_losses_matches_reference_golden(golden, idx):
    name = str(golden["loss/_names"][idx])
    g = {k.split("/", 2)[2]: v for k, v in golden.items() if k.startswith(f"loss/{name}/")}
    cfg = _cfg(g["cfg"])
    bundle, d_logits, d_baseline, targets, _ = ov.compute_losses(
        g["reward"], g["done"], g["policy_logits"], g["action"], g["learner_logits"],
        g["learner_baseline"], cfg, shift=0)
    # identical arithmetic order -> identical up to summation order
    tol = 1e-12 if g["learner_logits"].dtype == np.float64 else 1e-5
    np.testing.assert_allclose(targets.vs, g["vs"], rtol=tol, atol=tol)
    np.testing.assert_allclose(targets.pg_advantages, g["pg_advantages"], rtol=tol, atol=tol)
    np.testing.assert_allclose(d_logits, g["d_logits"], rtol=tol, atol=tol)
    np.testing.assert_array_equal(d_baseline[-1], 0.0)
    np.testing.assert_allclose(d_baseline, g["d_baseline"], rtol=tol, atol=tol)
    got = [bundle.pg_loss, bundle.baseline_loss, bundle.entropy_loss, bundle.total]
    np.testing.assert_allclose(got, g["losses"], rtol=1e-5, atol=1e-5)


def test_vtrace_matches_reference_golden(golden):
    cfg = ov.VtraceConfig(discount=1.0)
    for i in range(int(golden["vt/_n"])):
        g = {k.split("/", 2)[2]: v for k, v in golden.items() if k.startswith(f"vt/{i}/")}
        r = ov.vtrace_targets(g["log_rhos"], g["discounts"], g["rewards"], g["values"],
                              g["bootstrap"], cfg)
        np.testing.assert_allclose(r.vs, g["vs"], atol=1e-12)
        np.testing.assert_allclose(r.pg_advantages, g["pg"], atol=1e-12)
        d = ov.vtrace_definitional(g["log_rhos"], g["discounts"], g["rewards"], g["values"],
                                   g["bootstrap"], cfg)
        np.testing.assert_allclose(d.vs, g["vs_oracle"], atol=1e-12)


def test_optimizer_matches_reference_golden(golden):
    fields = [str(f) for f in golden["opt/_fields"]]
    for i in range(int(golden["opt/_n"])):
        g = {k.split("/", 2)[2]: v for k, v in golden.items() if k.startswith(f"opt/{i}/")}
        max_norm, lr, decay, eps = [float(x) for x in g["hyper"]]
        grads = [g[f"g_{f}"] for f in fields]
        clipped, norm = om.clip_global_norm(grads, max_norm, mode="beastpipe")
        assert norm == pytest.approx(float(g["norm"]), rel=1e-6)
        newp, news = om.rmsprop_step([g[f"p_{f}"] for f in fields], clipped,
                                     [g[f"s_{f}"] for f in fields], lr, decay, eps)
        for f, p, s in zip(fields, newp, news):
            np.testing.assert_allclose(p, g[f"np_{f}"], rtol=1e-6, atol=1e-7)
            np.testing.assert_allclose(s, g[f"ns_{f}"], rtol=1e-6, atol=1e-7)


# --- hand-derived known answers from the reference's tests -------------------------

def test_action_log_rhos_derived_value():
    # test_vtrace.py:54-59
    out = ov.action_log_rhos(np.array([[[0.0, 0.0]]]), np.array([[[1.0, 0.0]]]),
                             np.zeros((1, 1), np.int64))
    assert out[0, 0] == pytest.approx(0.3798854930417224, abs=1e-9)


def test_hand_backward_recursion():
    # test_vtrace.py:78-87
    cfg = ov.VtraceConfig(discount=0.9)
    r = ov.vtrace_targets(np.zeros((2, 1)), np.full((2, 1), 0.9), np.ones((2, 1)),
                          np.zeros((2, 1)), np.zeros(1), cfg)
    np.testing.assert_allclose(r.vs[:, 0], [1.9, 1.0], atol=1e-12)
    np.testing.assert_allclose(r.pg_advantages[:, 0], [1.9, 1.0], atol=1e-12)


def test_log_softmax_entropy_known_values():
    # test_model.py:144-146, :157-159
    np.testing.assert_allclose(om.log_softmax(np.array([1.0, 0.0])), [-0.31326169, -1.31326169],
                               atol=1e-7)
    for a in (2, 3, 5, 11):
        assert om.entropy(np.zeros(a)) == pytest.approx(np.log(a), abs=1e-12)


def test_rmsprop_hand_value_and_clip_345():
    # test_model.py:181-201 and :261-275
    p, s = om.rmsprop_step([np.array([[1.0]])], [np.array([[1.0]])], [np.zeros((1, 1))],
                           lr=0.1, decay=0.99, eps=0.0)
    assert s[0][0, 0] == pytest.approx(0.01)
    assert p[0][0, 0] == pytest.approx(0.0, abs=1e-12)
    clipped, norm = om.clip_global_norm([np.array([[3.0]]), np.array([4.0])], 1.0)
    assert norm == pytest.approx(5.0)
    assert np.sqrt(clipped[0][0, 0] ** 2 + clipped[1][0] ** 2) == pytest.approx(1.0)
    same, _ = om.clip_global_norm([np.array([[3.0]]), np.array([4.0])], 10.0)
    np.testing.assert_array_equal(same[0], [[3.0]])


def _random_instance(rng, t_max=10, b_max=4):
    # test_vtrace.py:18-28
    t_len = int(rng.integers(1, t_max + 1))
    b_len = int(rng.integers(1, b_max + 1))
    log_rhos = rng.uniform(-2.0, 2.0, size=(t_len, b_len))
    gamma = float(rng.uniform(0.5, 1.0))
    done = rng.random((t_len, b_len)) < 0.2
    return (log_rhos, gamma * ~done, rng.uniform(-5, 5, size=(t_len, b_len)),
            rng.uniform(-5, 5, size=(t_len, b_len)), rng.uniform(-5, 5, size=b_len))


def test_recursion_equals_definitional_sum(rng):
    # test_acceptance.py:58-74 (criterion 1), 200 instances here
    cfg = ov.VtraceConfig(discount=1.0)
    worst = 0.0
    for _ in range(200):
        inst = _random_instance(rng)
        a = ov.vtrace_targets(*inst, cfg)
        b = ov.vtrace_definitional(*inst, cfg)
        worst = max(worst, np.max(np.abs(a.vs - b.vs)), np.max(np.abs(a.pg_advantages - b.pg_advantages)))
    assert worst < 1e-6


def test_torchbeast_semantics_equal_beastpipe_on_shared_subset(rng):
    # upstream from_importance_weights == beastpipe vtrace_targets when c_bar=1 and pg clip == rho clip
    cfg = ov.VtraceConfig(discount=0.99, rho_bar=1.0, c_bar=1.0)
    for _ in range(20):
        inst = _random_instance(rng)
        a = ov.vtrace_targets(*inst, cfg)
        vs, pg = ov.tb_from_importance_weights(*inst, 1.0, 1.0)
        np.testing.assert_allclose(vs, a.vs, atol=1e-12)
        np.testing.assert_allclose(pg, a.pg_advantages, atol=1e-12)


def test_loss_gradients_match_finite_differences(rng):
    # test_vtrace.py:206-221 methodology
    cfg = ov.VtraceConfig(discount=0.9, baseline_cost=0.5, entropy_cost=0.01)
    t, b, a = 3, 2, 3
    reward = rng.normal(size=(t + 1, b))
    done = rng.random((t + 1, b)) < 0.2
    beh = rng.normal(size=(t + 1, b, a))
    act = rng.integers(0, a, size=(t + 1, b))
    logits = rng.normal(size=(t, b, a))
    baseline = rng.normal(size=(t + 1, b))
    _, d_logits, d_baseline, targets, _ = ov.compute_losses(reward, done, beh, act, logits,
                                                             baseline, cfg)

    def objective():
        bundle, _, _ = ov.losses_from_targets(logits, baseline, act[:t], targets, cfg)
        return bundle.total

    assert_grads_close(d_logits, central_difference(objective, logits))
    assert_grads_close(d_baseline, central_difference(objective, baseline))
    np.testing.assert_array_equal(d_baseline[-1], 0.0)
