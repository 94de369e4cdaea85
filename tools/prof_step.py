"""A few learner steps (T=80 B=32 A=6) for ncu launch lists."""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa
from paper_1910_03552_b200 import learner, optim
from paper_1910_03552_b200.atari_net import AtariNet
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
T, B, A = 80, 32, 6
model = AtariNet(num_actions=A)
opt = optim.RMSprop(model.parameters(), lr=4.8e-4, alpha=0.99, eps=0.01)
batch = bench.make_batch(T, B, A, torch.device("cuda"), 0)
L = learner.FusedLearner(model, bench.FLAGS, T, B)
for _ in range(steps):
    L.step(batch, opt)
torch.cuda.synchronize()
