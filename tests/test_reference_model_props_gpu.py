"""The reference's model-helper tests (beastpipe tests/test_model.py: TestLogSoftmaxEntropy,
TestRmsProp, TestSamplingAndClipping) restated through this repo's CUDA path:

- log_softmax   -> `vtrace.action_log_probs` (the fused kernel's log-softmax + exact gather);
- entropy       -> `losses.compute_entropy_loss` (negative entropy, sum-reduced; one row per call);
- rmsprop_step  -> `optim.rmsprop_step` (bp_rmsprop_clip_f32);
- clip_global_norm -> `optim.clip_global_norm` (bp_sumsq_f32);
- sample_actions   -> bp_sample_actions_f32 (Gumbel-max, Philox keyed by seed / row / column).

The MLP forward / backward classes of that file test the reference's MLP, which the north star
replaces by AtariNet (tests/test_atari_gpu.py, tests/test_learn_parity_gpu.py).  Tolerances: the
reference asserts in f64; here the kernels run in f32, so 1e-12 absolute becomes 1e-6.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _log_softmax_rows(logits: np.ndarray) -> np.ndarray:
    """Every entry of log_softmax(logits) (N, A) through the kernel: one gather per action."""
    from paper_1910_03552_b200 import vtrace

    lg = torch.from_numpy(np.ascontiguousarray(logits, dtype=np.float32)).cuda()[None]
    n, a = logits.shape
    cols = [vtrace.action_log_probs(lg, torch.full((1, n), k, dtype=torch.int64, device="cuda"))[0]
            for k in range(a)]
    return torch.stack(cols, dim=-1).cpu().numpy()


def _entropy(logits: np.ndarray) -> float:
    from paper_1910_03552_b200 import losses

    lg = torch.from_numpy(np.ascontiguousarray(logits, dtype=np.float32)).cuda().reshape(1, -1)
    return -float(losses.compute_entropy_loss(lg, check=True))


def _sample(logits: np.ndarray, seed: int) -> np.ndarray:
    from paper_1910_03552_b200 import _native as N

    lg = torch.from_numpy(np.ascontiguousarray(logits, dtype=np.float32)).cuda()
    n, a = lg.shape
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    N.check(N.lib().bp_sample_actions_f32(N.ptr(lg), n, a, seed, 0, N.ptr(out), N.stream_handle(lg.device)),
            "bp_sample_actions_f32")
    return out.cpu().numpy()


class TestLogSoftmaxEntropy:
    def test_uniform_two_actions(self):
        np.testing.assert_allclose(_log_softmax_rows(np.array([[0.0, 0.0]])), [[-np.log(2)] * 2], atol=1e-6)

    def test_derived_values(self):
        np.testing.assert_allclose(_log_softmax_rows(np.array([[1.0, 0.0]])), [[-0.31326169, -1.31326169]],
                                   atol=1e-6)

    def test_large_logits_stay_finite(self):
        assert np.all(np.isfinite(_log_softmax_rows(np.array([[1000.0, 0.0]]))))

    def test_rows_sum_to_one(self, rng):
        logits = rng.normal(scale=10.0, size=(50, 7))
        probs = np.exp(_log_softmax_rows(logits).astype(np.float64))
        np.testing.assert_allclose(probs.sum(axis=-1), 1.0, atol=1e-5)

    def test_entropy_uniform_is_log_a(self):
        for a in (2, 3, 5, 11):
            assert _entropy(np.zeros(a)) == pytest.approx(np.log(a), abs=1e-6)

    def test_entropy_near_deterministic(self):
        assert _entropy(np.array([10.0, -10.0])) < 1e-3

    def test_entropy_bounds(self, rng):
        logits = rng.normal(scale=5.0, size=(200, 6))
        ent = np.array([_entropy(row) for row in logits])
        assert np.all(ent >= -1e-6)
        assert np.all(ent <= np.log(6) + 1e-6)


def _params(rng, shapes):
    return [rng.normal(size=s).astype(np.float32) for s in shapes]


SHAPES = [(4, 2), (4,), (3, 4), (3,), (1, 4), (1,)]  # W1 b1 Wp bp Wv bv of the reference MLP


class TestRmsProp:
    def test_zero_grad_keeps_params(self, rng):
        from paper_1910_03552_b200 import optim

        params = _params(rng, SHAPES)
        zero = [np.zeros_like(p) for p in params]
        new_params, _ = optim.rmsprop_step(params, zero, [np.zeros_like(p) for p in params])
        for a, b in zip(new_params, params):
            np.testing.assert_array_equal(a, b)

    def test_hand_evaluated_update(self):
        from paper_1910_03552_b200 import optim

        params = [np.array([[1.0]], np.float32)] + [np.zeros(1, np.float32)] * 5
        grads = [np.array([[1.0]], np.float32)] + [np.zeros(1, np.float32)] * 5
        g2 = [np.zeros_like(p) for p in params]
        new_params, new_g2 = optim.rmsprop_step(params, grads, g2, learning_rate=0.1, decay=0.99, epsilon=0.0)
        assert new_g2[0][0, 0] == pytest.approx(0.01, rel=1e-6)
        assert new_params[0][0, 0] == pytest.approx(0.0, abs=1e-6)

    def test_repeated_steps_shrink(self, rng):
        from paper_1910_03552_b200 import optim

        params = _params(rng, [(1, 1), (1,), (2, 1), (2,), (1, 1), (1,)])
        g = [np.ones_like(p) for p in params]
        g2 = [np.zeros_like(p) for p in params]
        p1, g2 = optim.rmsprop_step(params, g, g2, learning_rate=0.1)
        p2, g2 = optim.rmsprop_step(p1, g, g2, learning_rate=0.1)
        assert abs(params[1][0] - p2[1][0]) > abs(params[1][0] - p1[1][0])
        assert abs(p1[1][0] - p2[1][0]) < abs(params[1][0] - p1[1][0])

    def test_nonfinite_grad_rejected(self, rng):
        from paper_1910_03552_b200 import optim
        from paper_1910_03552_b200.errors import NonFiniteError

        params = _params(rng, [(1, 1), (1,), (2, 1), (2,), (1, 1), (1,)])
        g = [np.zeros_like(p) for p in params]
        g[0][0, 0] = np.nan
        with pytest.raises(NonFiniteError):
            optim.rmsprop_step(params, g, [np.zeros_like(p) for p in params])

    def test_epsilon_guards_division(self, rng):
        from paper_1910_03552_b200 import optim

        params = _params(rng, SHAPES)
        g = _params(rng, SHAPES)
        new_params, _ = optim.rmsprop_step(params, g, [np.zeros_like(p) for p in params], epsilon=0.01)
        for p in new_params:
            assert np.all(np.isfinite(p))


class TestSamplingAndClipping:
    def test_sampling_respects_sharp_logits(self):
        logits = np.tile(np.array([10.0, -10.0]), (10_000, 1))
        assert (_sample(logits, 7) == 0).mean() >= 0.999

    def test_sampling_reproducible_with_seed(self):
        logits = np.zeros((100, 4))
        np.testing.assert_array_equal(_sample(logits, 3), _sample(logits, 3))
        assert not np.array_equal(_sample(logits, 3), _sample(logits, 4))

    def test_clip_global_norm(self):
        from paper_1910_03552_b200 import optim

        g = [np.array([[3.0]], np.float32), np.array([4.0], np.float32)] + [np.zeros(1, np.float32)] * 4
        clipped, norm = optim.clip_global_norm(g, 1.0)
        assert norm == pytest.approx(5.0)
        assert np.sqrt(clipped[0][0, 0] ** 2 + clipped[1][0] ** 2) == pytest.approx(1.0, rel=1e-6)
        same, _ = optim.clip_global_norm(g, 10.0)
        np.testing.assert_array_equal(same[0], g[0])
