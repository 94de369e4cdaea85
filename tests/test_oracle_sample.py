"""The sampler oracle's Philox4x32-10 against the published known-answer vectors
(Random123 kat_vectors, philox4x32_10), CPU only."""
import numpy as np

from oracle import sample_np


def test_philox_known_answers():
    kat = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for ctr, key, want in kat:
        got = sample_np.philox4x32_10(*[[c] for c in ctr], *key)
        assert tuple(int(w[0]) for w in got) == want


def test_gumbel_max_distribution():
    logits = np.tile(np.array([[2.0, 0.0, -1.0, 0.5, -3.0, 1.0]]), (100_000, 1))
    acts = sample_np.sample_actions(logits, seed=12345)
    freq = np.bincount(acts, minlength=6) / len(acts)
    p = np.exp(logits[0]) / np.exp(logits[0]).sum()
    assert np.abs(freq - p).max() < 6e-3
    assert np.array_equal(sample_np.sample_actions(logits[:5], 1, greedy=True), np.zeros(5))
