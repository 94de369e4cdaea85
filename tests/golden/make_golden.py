"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container only (it imports beastpipe from /root/reference,
which does not exist on the GPU box):

    python tests/golden/make_golden.py

Writes tests/golden/beastpipe_golden.npz.  The fixtures are committed; the
tests read only the npz.  Each case stores the reference inputs and the
reference's outputs (compute_losses -> bundle, d_logits, d_baseline, targets;
vtrace_oracle; clip_global_norm + rmsprop_step).
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"


def main(out_path: str) -> None:
    sys.path.insert(0, REF_SRC)
    from beastpipe import model as bm  # noqa: E402
    from beastpipe import vtrace as bv  # noqa: E402
    from beastpipe.rollout import TrainingBatch  # noqa: E402

    store: dict[str, np.ndarray] = {}

    def put(prefix, **arrs):
        for k, v in arrs.items():
            store[f"{prefix}/{k}"] = np.asarray(v)

    # --- compute_losses cases (vtrace.py:224-255) ---------------------------------
    loss_cases = [
        # name, T, B, A, dtype, cfg kwargs, seed, done_p
        ("cfg1_f32", 20, 32, 6, np.float32, {}, 0, 0.05),
        ("cfg1_f64", 20, 32, 6, np.float64, {}, 1, 0.05),
        ("t80_b8_a18_f32", 80, 8, 18, np.float32, {}, 2, 0.05),
        ("clipped_f64", 12, 5, 4, np.float64, dict(rho_bar=1.3, c_bar=0.9, discount=0.95,
                                                   baseline_cost=0.37, entropy_cost=0.021,
                                                   pg_cost=1.4), 3, 0.2),
        ("t1_b1_a1_f64", 1, 1, 1, np.float64, {}, 4, 0.5),
        ("alldone_f32", 6, 4, 3, np.float32, {}, 5, 1.0),
        ("ragged_t7_b3_a5_f32", 7, 3, 5, np.float32, dict(discount=1.0), 6, 0.3),
    ]
    names = []
    for name, t, b, a, dt, kw, seed, done_p in loss_cases:
        rng = np.random.default_rng(seed)
        cfg = bv.VtraceConfig(**kw)
        t1 = t + 1
        batch = TrainingBatch(
            observation=np.zeros((t1, b, 1), np.float32),
            reward=rng.uniform(-1, 1, size=(t1, b)).astype(np.float32),
            done=rng.random((t1, b)) < done_p,
            policy_logits=rng.normal(size=(t1, b, a)).astype(np.float32),
            baseline=np.zeros((t1, b), np.float32),
            action=rng.integers(0, a, size=(t1, b)).astype(np.int64),
            model_versions=np.zeros(b, np.int64),
        )
        learner_logits = rng.normal(size=(t, b, a)).astype(dt)
        learner_baseline = rng.normal(size=(t1, b)).astype(dt)
        bundle, d_logits, d_baseline, targets = bv.compute_losses(
            batch, learner_logits, learner_baseline, cfg)
        put(f"loss/{name}",
            T=t, B=b, A=a, cfg=np.array([cfg.discount, cfg.rho_bar, cfg.c_bar, cfg.baseline_cost,
                                         cfg.entropy_cost, cfg.pg_cost]),
            reward=batch.reward, done=batch.done, policy_logits=batch.policy_logits,
            action=batch.action, learner_logits=learner_logits,
            learner_baseline=learner_baseline,
            losses=np.array([bundle.pg_loss, bundle.baseline_loss, bundle.entropy_loss,
                             bundle.total]),
            d_logits=d_logits, d_baseline=d_baseline, vs=targets.vs,
            pg_advantages=targets.pg_advantages, clipped_rhos=targets.clipped_rhos)
        names.append(name)
    store["loss/_names"] = np.array(names)

    # --- vtrace_targets vs vtrace_oracle, test_vtrace.py:18-28 generator ---------
    rng = np.random.default_rng(20240817)
    for i in range(8):
        t_len = int(rng.integers(1, 11))
        b_len = int(rng.integers(1, 5))
        log_rhos = rng.uniform(-2.0, 2.0, size=(t_len, b_len))
        gamma = float(rng.uniform(0.5, 1.0))
        done = rng.random((t_len, b_len)) < 0.2
        discounts = gamma * ~done
        rewards = rng.uniform(-5.0, 5.0, size=(t_len, b_len))
        values = rng.uniform(-5.0, 5.0, size=(t_len, b_len))
        bootstrap = rng.uniform(-5.0, 5.0, size=b_len)
        cfg = bv.VtraceConfig(discount=1.0, rho_bar=1.0, c_bar=1.0)
        rec = bv.vtrace_targets(log_rhos, discounts, rewards, values, bootstrap, cfg)
        ora = bv.vtrace_oracle(log_rhos, discounts, rewards, values, bootstrap, cfg)
        put(f"vt/{i}", log_rhos=log_rhos, discounts=discounts, rewards=rewards, values=values,
            bootstrap=bootstrap, vs=rec.vs, pg=rec.pg_advantages, vs_oracle=ora.vs,
            pg_oracle=ora.pg_advantages)
    store["vt/_n"] = np.array(8)

    # --- clip_global_norm + rmsprop_step (model.py:224-268) ----------------------
    for i, (max_norm, lr, decay, eps) in enumerate([(40.0, 0.005, 0.99, 0.01),
                                                    (0.5, 0.1, 0.9, 0.01),
                                                    (1e9, 0.00048, 0.99, 0.01)]):
        rng = np.random.default_rng(100 + i)
        params = bm.init_params(obs_dim=7, num_actions=3, hidden=5, seed=i)
        params = bm.ModelParams(**{f: rng.normal(size=getattr(params, f).shape).astype(np.float32)
                                   for f in bm.PARAM_FIELDS})
        grads = bm.GradientSet(**{f: (3 * rng.normal(size=getattr(params, f).shape)
                                      ).astype(np.float32) for f in bm.PARAM_FIELDS})
        state = bm.init_rmsprop(params, learning_rate=lr, decay=decay, epsilon=eps)
        state = bm.RmsPropState(
            g2={f: rng.uniform(0, 2, size=getattr(params, f).shape).astype(np.float32)
                for f in bm.PARAM_FIELDS}, learning_rate=lr, decay=decay, epsilon=eps)
        clipped, norm = bm.clip_global_norm(grads, max_norm)
        new_params, new_state = bm.rmsprop_step(params, clipped, state)
        put(f"opt/{i}", hyper=np.array([max_norm, lr, decay, eps]), norm=norm,
            **{f"p_{f}": getattr(params, f) for f in bm.PARAM_FIELDS},
            **{f"g_{f}": getattr(grads, f) for f in bm.PARAM_FIELDS},
            **{f"s_{f}": state.g2[f] for f in bm.PARAM_FIELDS},
            **{f"np_{f}": getattr(new_params, f) for f in bm.PARAM_FIELDS},
            **{f"ns_{f}": new_state.g2[f] for f in bm.PARAM_FIELDS})
    store["opt/_n"] = np.array(3)
    store["opt/_fields"] = np.array(bm.PARAM_FIELDS)

    np.savez_compressed(out_path, **store)
    print(f"wrote {out_path} ({os.path.getsize(out_path)} bytes, {len(store)} arrays)")


if __name__ == "__main__":
    main(os.path.join(os.path.dirname(os.path.abspath(__file__)), "beastpipe_golden.npz"))
