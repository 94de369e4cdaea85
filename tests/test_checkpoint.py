"""TBST1 checkpoint + logs.csv interop, pinned by files the reference itself
wrote (tests/golden/make_tbst1.py: beastpipe.pipeline.checkpoint / MetricsWriter)."""
import os
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from paper_1910_03552_b200 import checkpoint as ck

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_reads_reference_checkpoint_and_rewrites_it_byte_identically(tmp_path):
    path = os.path.join(GOLD, "beastpipe_mlp.tbst1")
    arrays, version = ck.load_params(path)
    assert version == 7 and list(arrays) == list(ck.PARAM_FIELDS)
    assert arrays["W1"].shape == (4, 10) and arrays["Wp"].shape == (3, 4) and arrays["bv"][0] == 0.25
    out = tmp_path / "again.tbst1"
    ck.save_params(SimpleNamespace(version=version, **arrays), str(out))
    assert out.read_bytes() == open(path, "rb").read()


def test_corrupt_and_mismatched_checkpoints_raise(tmp_path):
    good = open(os.path.join(GOLD, "beastpipe_mlp.tbst1"), "rb").read()
    for name, blob in (("magic", b"XXXXX" + good[5:]), ("trunc", good[:-3]), ("trail", good + b"\0")):
        p = tmp_path / name
        p.write_bytes(blob)
        with pytest.raises(ck.CheckpointError):
            ck.load_params(str(p))
    p = tmp_path / "other.tbst1"
    ck.write_tbst1(str(p), [("conv1.weight", np.zeros((2, 2), np.float32))], 1)
    with pytest.raises(ck.CheckpointError):
        ck.load_params(str(p))  # the MLP field order is enforced, as in restore()


def test_atari_state_dict_round_trip_cpu(tmp_path):
    from oracle import atari_ref

    torch.manual_seed(3)
    ref = atari_ref.AtariNetRef(num_actions=6)
    p = tmp_path / "atari.tbst1"
    ck.checkpoint(ref, str(p), version=42)
    other = atari_ref.AtariNetRef(num_actions=6)
    arrays, version = ck.restore(str(p), other, expected_num_actions=6)
    assert version == 42
    for k, v in ref.state_dict().items():
        assert torch.equal(other.state_dict()[k], v)
    with pytest.raises(ck.CheckpointError):
        ck.restore(str(p), expected_num_actions=18)
    with pytest.raises(ck.CheckpointError):
        ck.restore(str(p), atari_ref.AtariNetRef(num_actions=18))


def test_logs_csv_matches_reference_format(tmp_path):
    w = ck.MetricsWriter(str(tmp_path))
    w.append(ck.MetricsRecord(1, 160, 1.5, -0.25, 3.125, -0.0125, 2.8625, 1234.5678))
    w.append(ck.MetricsRecord.from_stats(2, 320, dict(mean_episode_return=float("nan"), pg_loss=0.5,
                                                       baseline_loss=1.0, entropy_loss=-0.01,
                                                       total_loss=1.49), 99.999))
    w.close()
    assert (tmp_path / "logs.csv").read_text() == open(os.path.join(GOLD, "beastpipe_logs.csv")).read()


@pytest.mark.gpu
def test_gpu_trained_atari_net_checkpoint_round_trip(tmp_path):
    from oracle import atari_ref
    from paper_1910_03552_b200 import learner, optim
    from paper_1910_03552_b200.atari_net import AtariNet

    flags = dict(atari_ref.DEFAULT_FLAGS)
    torch.manual_seed(0)
    net = AtariNet(num_actions=6)
    opt = optim.RMSprop(net.parameters(), lr=flags["learning_rate"], alpha=0.99, eps=0.01)
    batch = {k: v.cuda() for k, v in atari_ref.synthetic_batch(4, 4, 6, seed=2).items()}
    learner.learn(flags, None, net, batch, (), opt, None)
    p = tmp_path / "trained.tbst1"
    ck.checkpoint(net, str(p), version=1)
    # the reference-layout state loads into the torch-CPU restatement and into a fresh net
    ref = atari_ref.AtariNetRef(num_actions=6)
    ck.restore(str(p), ref)
    fresh = AtariNet(num_actions=6)
    ck.restore(str(p), fresh)
    assert torch.equal(fresh.flat_params, net.flat_params)
