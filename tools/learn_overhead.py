"""Host-side cost of the public learn() call per step (device-resident batch)."""
import sys, time
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1910_03552_b200 import learner, optim  # noqa: E402
from paper_1910_03552_b200.atari_net import AtariNet  # noqa: E402

T, B, A = 80, 32, 6
dev = torch.device("cuda")
model = AtariNet(num_actions=A)
opt = optim.RMSprop(model.parameters(), lr=4.8e-4, alpha=0.99, eps=0.01)
batch = bench.make_batch(T, B, A, dev, 0)
for _ in range(5):
    learner.learn(bench.FLAGS, None, model, batch, (), opt, None)
torch.cuda.synchronize()
L = model._fused_learners[(T, B)]
# pieces
n = 50
t0 = time.perf_counter()
for _ in range(n):
    learner.learn(bench.FLAGS, None, model, batch, (), opt, None)
t1 = time.perf_counter()
print(f"learn() wall per step {(t1 - t0) / n * 1e6:.1f} us")
t0 = time.perf_counter()
for _ in range(n):
    L.step(batch, opt)
    L._stats_event.record()
    L._stats_event.synchronize()
t1 = time.perf_counter()
print(f"step()+sync wall per step {(t1 - t0) / n * 1e6:.1f} us")
t0 = time.perf_counter()
for _ in range(n):
    L.step(batch, opt)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"step() host enqueue only {(t1 - t0) / n * 1e6:.1f} us")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n):
    L.stats(batch)
t1 = time.perf_counter()
print(f"stats() on an idle GPU {(t1 - t0) / n * 1e6:.1f} us")
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    learner.learn(bench.FLAGS, None, model, batch, (), opt, None)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
