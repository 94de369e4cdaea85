"""A few learner steps for ncu launch lists / captures.

    python tools/prof_step.py [steps] [lstm]
lstm=0: configs[1] (T=80 B=32 A=6, no LSTM); lstm=1: configs[2] (T=80 B=32 A=18, LSTM core).
"""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa
from paper_1910_03552_b200 import learner, optim
from paper_1910_03552_b200.atari_net import AtariNet
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
use_lstm = len(sys.argv) > 2 and sys.argv[2] == "1"
T, B, A = (80, 32, 18) if use_lstm else (80, 32, 6)
model = AtariNet(num_actions=A, use_lstm=use_lstm)
opt = optim.RMSprop(model.parameters(), lr=4.8e-4, alpha=0.99, eps=0.01)
batch = bench.make_batch(T, B, A, torch.device("cuda"), 0)
L = learner.FusedLearner(model, bench.FLAGS, T, B)
L.use_graphs = False  # eager: every launch is a separate ncu record in step order
state = model.initial_state(B)
for _ in range(steps):
    L.step(batch, opt, None, state)
torch.cuda.synchronize()
