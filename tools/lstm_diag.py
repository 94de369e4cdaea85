"""Diagnostics: end-to-end LSTM AtariNet errors vs the fp32 torch restatement."""
import sys
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from oracle import atari_ref
from test_lstm_gpu import _models, _batch, _state, rel_l2

for (T, B, A) in [(4, 5, 6), (20, 8, 18), (80, 32, 18)]:
    net, ref = _models(A, seed=4)
    flags = dict(atari_ref.DEFAULT_FLAGS)
    batch = _batch(T + 1, B, A, seed=20)
    state = _state(B, 513 + A, seed=30)
    with torch.no_grad():
        want, _ = ref(batch, state)
        got, _ = net({k: v.cuda() for k, v in batch.items()}, tuple(s.cuda() for s in state))
    e1 = rel_l2(got["policy_logits"], want["policy_logits"])
    e2 = rel_l2(got["baseline"], want["baseline"])
    # no-LSTM comparison at the same sizes for scale
    total_ref, parts_ref, _ = atari_ref.learn_losses(ref, batch, flags, state)[0], atari_ref.learn_losses(ref, batch, flags, state)[1], None
    from paper_1910_03552_b200 import learner
    L = learner.FusedLearner(net, flags, T, B)
    L.use_graphs = False
    L.step({k: v.cuda() for k, v in batch.items()}, None, None, tuple(s.cuda() for s in state))
    lv = L.losses.tolist()
    print(f"T={T} B={B} A={A} logits {e1:.2e} baseline {e2:.2e} total {lv[3]:.4f} vs {float(total_ref):.4f} "
          f"pg {lv[0]:.4f} vs {float(parts_ref[0]):.4f} base {lv[1]*0.5:.4f} vs {float(parts_ref[1]):.4f} "
          f"ent {lv[2]*0.0006:.5f} vs {float(parts_ref[2]):.5f}", flush=True)
