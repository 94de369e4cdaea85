"""GPU parity of the fused V-trace kernels against the CPU oracle (fp64).

Tolerance (DESIGN.md / SURVEY 8c): max|gpu - oracle| <= 1e-5 * max|oracle| for
vs / pg_advantages / log-probs; the action gather and done-masking are exact.
"""
import numpy as np
import pytest
import torch

from conftest import rel_err
from oracle import vtrace_np as ov

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _inputs(seed, T, B, A, done_p=0.05, gamma=0.99):
    rng = np.random.default_rng(seed)
    beh = rng.normal(size=(T, B, A)).astype(np.float32)
    tgt = rng.normal(size=(T, B, A)).astype(np.float32)
    act = rng.integers(0, A, size=(T, B)).astype(np.int64)
    done = rng.random((T, B)) < done_p
    disc = (np.float32(gamma) * ~done).astype(np.float32)
    rew = rng.uniform(-1, 1, size=(T, B)).astype(np.float32)
    val = rng.normal(size=(T, B)).astype(np.float32)
    boot = rng.normal(size=B).astype(np.float32)
    return beh, tgt, act, disc, rew, val, boot


def _cuda(*arrs):
    return [torch.from_numpy(a).cuda() for a in arrs]


SHAPES = [(20, 32, 6), (80, 32, 18), (80, 4096, 18), (7, 3, 5), (1, 1, 1), (33, 4097, 18),
          (5, 300, 48), (80, 512, 6), (300, 20, 3), (2048, 2, 4), (80, 514, 18), (248, 64, 6),
          (249, 64, 18), (80, 16384, 18)]


@pytest.mark.parametrize("T,B,A", SHAPES)
@pytest.mark.parametrize("seed", [0, 1])
def test_from_logits_matches_oracle(T, B, A, seed):
    from paper_1910_03552_b200 import vtrace

    arrs = _inputs(seed, T, B, A)
    f64 = [a.astype(np.float64) if a.dtype == np.float32 else a for a in arrs]
    vs, pg, lr, blp, tlp = ov.tb_from_logits(*f64)
    r = vtrace.from_logits(*_cuda(*arrs), check=True)
    torch.cuda.synchronize()
    assert rel_err(r.vs.cpu(), vs) < TOL
    assert rel_err(r.pg_advantages.cpu(), pg) < TOL
    assert rel_err(r.log_rhos.cpu(), lr) < TOL
    assert rel_err(r.behavior_action_log_probs.cpu(), blp) < TOL
    assert rel_err(r.target_action_log_probs.cpu(), tlp) < TOL


@pytest.mark.parametrize("clips", [(1.0, 1.0, 1.0), (1.3, 0.8, 0.9), (None, None, 1.0),
                                   (2.0, 1.0, 1.0)])
def test_from_logits_clip_thresholds(clips):
    from paper_1910_03552_b200 import vtrace

    rho, pg_rho, c = clips
    T, B, A = 30, 64, 6
    arrs = _inputs(3, T, B, A)
    beh, tgt, act, disc, rew, val, boot = [a.astype(np.float64) if a.dtype == np.float32 else a
                                           for a in arrs]
    lr = ov.gather_last(ov.log_softmax(tgt), act) - ov.gather_last(ov.log_softmax(beh), act)
    rhos = np.exp(lr)
    cfg = ov.VtraceConfig(discount=0.99, rho_bar=np.inf if rho is None else rho, c_bar=c)
    ref = ov.vtrace_targets(lr, disc, rew, val, boot, cfg,
                            pg_rho_bar=np.inf if pg_rho is None else pg_rho)
    r = vtrace.from_logits(*_cuda(*arrs), clip_rho_threshold=rho, clip_pg_rho_threshold=pg_rho,
                           clip_c_threshold=c)
    assert rel_err(r.vs.cpu(), ref.vs) < TOL
    assert rel_err(r.pg_advantages.cpu(), ref.pg_advantages) < TOL
    assert np.isfinite(rhos).all()


@pytest.mark.parametrize("T,B,A", [(20, 32, 6), (80, 4096, 18), (9, 5, 48)])
def test_action_gather_is_exact(T, B, A):
    """Target logits encode the index (x_j = j); the recovered index must equal the action."""
    from paper_1910_03552_b200 import vtrace

    rng = np.random.default_rng(7)
    act = rng.integers(0, A, size=(T, B)).astype(np.int64)
    tgt = np.broadcast_to(np.arange(A, dtype=np.float32), (T, B, A)).copy()
    beh = rng.normal(size=(T, B, A)).astype(np.float32)
    z = np.zeros((T, B), np.float32)
    r = vtrace.from_logits(*_cuda(beh, tgt, act, z, z, z, np.zeros(B, np.float32)))
    lse = np.log(np.exp(np.arange(A, dtype=np.float64)).sum())
    recovered = np.rint(r.target_action_log_probs.cpu().numpy().astype(np.float64) + lse)
    np.testing.assert_array_equal(recovered.astype(np.int64), act)


def test_done_masking_cuts_dependence_exactly():
    """A zero discount at row `cut` makes vs[:cut+1] bit-identical under later changes."""
    from paper_1910_03552_b200 import vtrace

    T, B, A = 40, 256, 6
    beh, tgt, act, disc, rew, val, boot = _inputs(11, T, B, A, done_p=0.0)
    cut = 17
    disc[cut] = 0.0
    base = vtrace.from_logits(*_cuda(beh, tgt, act, disc, rew, val, boot))
    rew2, val2 = rew.copy(), val.copy()
    rew2[cut + 1:] += 100.0
    val2[cut + 1:] -= 50.0
    tgt2 = tgt.copy()
    tgt2[cut + 1:] += np.random.default_rng(1).normal(size=tgt2[cut + 1:].shape).astype(np.float32)
    mod = vtrace.from_logits(*_cuda(beh, tgt2, act, disc, rew2, val2, boot + 9.0))
    torch.testing.assert_close(base.vs[:cut + 1], mod.vs[:cut + 1], rtol=0, atol=0)


def test_from_importance_weights_matches_oracle_and_definitional(rng):
    from paper_1910_03552_b200 import vtrace

    cfg = ov.VtraceConfig(discount=1.0)
    for _ in range(40):
        t_len = int(rng.integers(1, 11))
        b_len = int(rng.integers(1, 5))
        lr = rng.uniform(-2, 2, size=(t_len, b_len))
        gamma = float(rng.uniform(0.5, 1.0))
        disc = gamma * ~(rng.random((t_len, b_len)) < 0.2)
        rew = rng.uniform(-5, 5, size=(t_len, b_len))
        val = rng.uniform(-5, 5, size=(t_len, b_len))
        boot = rng.uniform(-5, 5, size=b_len)
        ref = ov.vtrace_definitional(lr, disc, rew, val, boot, cfg)
        f32 = [np.asarray(x, np.float32) for x in (lr, disc, rew, val, boot)]
        ret, cr = vtrace.from_importance_weights(*_cuda(*f32), return_clipped_rhos=True, check=True)
        assert rel_err(ret.vs.cpu(), ref.vs) < TOL
        assert rel_err(ret.pg_advantages.cpu(), ref.pg_advantages) < TOL
        assert rel_err(cr.cpu(), ref.clipped_rhos) < TOL


def test_on_policy_reduces_to_nstep_return(rng):
    from paper_1910_03552_b200 import vtrace

    T, B = 50, 300
    disc = (0.97 * ~(rng.random((T, B)) < 0.1)).astype(np.float32)
    rew = rng.uniform(-1, 1, size=(T, B)).astype(np.float32)
    val = rng.normal(size=(T, B)).astype(np.float32)
    boot = rng.normal(size=B).astype(np.float32)
    expected = np.zeros((T, B))
    acc = boot.astype(np.float64)
    for t in range(T - 1, -1, -1):
        acc = rew[t] + disc[t].astype(np.float64) * acc
        expected[t] = acc
    ret = vtrace.from_importance_weights(*_cuda(np.zeros((T, B), np.float32), disc, rew, val, boot))
    assert rel_err(ret.vs.cpu(), expected) < TOL


def test_status_word_raises_reference_exceptions():
    from paper_1910_03552_b200 import vtrace
    from paper_1910_03552_b200.errors import NonFiniteError, SchemaError

    T, B, A = 6, 8, 4
    arrs = list(_inputs(5, T, B, A))
    bad = [a.copy() for a in arrs]
    bad[2][3, 2] = A  # action out of range
    with pytest.raises(SchemaError):
        vtrace.from_logits(*_cuda(*bad), check=True)
    bad = [a.copy() for a in arrs]
    bad[4][1, 1] = np.nan  # reward
    with pytest.raises(NonFiniteError):
        vtrace.from_logits(*_cuda(*bad), check=True)
    bad = [a.copy() for a in arrs]
    bad[3][0, 0] = -0.5  # negative discount
    with pytest.raises(SchemaError):
        vtrace.from_logits(*_cuda(*bad), check=True)
    bad = [a.copy() for a in arrs]
    bad[0][2, 2, 1] = np.inf  # behaviour logit
    with pytest.raises(NonFiniteError):
        vtrace.from_logits(*_cuda(*bad), check=True)
    # clean call after the errors leaves the word clear
    vtrace.from_logits(*_cuda(*arrs), check=True)


def test_beastpipe_mirror_api_numpy_roundtrip():
    from paper_1910_03552_b200 import learner_ops as lo

    rng = np.random.default_rng(3)
    out = lo.action_log_rhos(np.array([[[0.0, 0.0]]]), np.array([[[1.0, 0.0]]]),
                             np.zeros((1, 1), np.int64))
    assert out[0, 0] == pytest.approx(0.3798854930417224, abs=1e-6)
    r = lo.vtrace_targets(np.zeros((2, 1)), np.full((2, 1), 0.9), np.ones((2, 1)),
                          np.zeros((2, 1)), np.zeros(1), lo.VtraceConfig(discount=0.9))
    np.testing.assert_allclose(r.vs[:, 0], [1.9, 1.0], atol=1e-6)
    np.testing.assert_allclose(r.pg_advantages[:, 0], [1.9, 1.0], atol=1e-6)
    logits = rng.normal(size=(4, 2, 3))
    np.testing.assert_allclose(lo.action_log_rhos(logits, logits, rng.integers(0, 3, (4, 2))), 0.0,
                               atol=1e-6)
