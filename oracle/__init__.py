"""CPU oracle for the IMPALA learner-step hot path.

TEST INFRASTRUCTURE ONLY.  Nothing under `paper_1910_03552_b200/` may import
this package: only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs use it, and only as the checker or
the timed CPU baseline -- never as the thing measured or shipped.

Modules
-------
vtrace_np   numpy restatement of beastpipe `vtrace.py` (the in-tree reference)
            plus the upstream TorchBeast `from_logits` / `from_importance_weights`
            semantics (separate pg rho clip, c fixed at 1).
model_np    numpy restatement of beastpipe `model.py` softmax family, global-norm
            clip and RMSProp (and the torch `clip_grad_norm_` variant).
atari_ref   torch-CPU fp32 restatement of the north-star AtariNet (+LSTM) and of
            upstream `learn()`.  The reference has no conv/LSTM code
            (SPEC.md:108 non-goal), so this part is "parity unpinned" by the
            reference's own tests; it is pinned by finite differences instead.

Pinning: `tests/golden/make_golden.py` imports the reference package from
/root/reference (in the build container only) and writes npz fixtures that
`tests/test_oracle_golden.py` checks this oracle against, together with the
hand-derived known answers from the reference's tests.
"""
