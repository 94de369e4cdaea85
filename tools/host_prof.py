import sys, time, statistics, cProfile, pstats
import torch
sys.path.insert(0, ".")
import bench
from paper_1910_03552_b200 import learner, optim
from paper_1910_03552_b200.atari_net import AtariNet
dev = torch.device("cuda")
T, B, A = 80, 32, 6
model = AtariNet(num_actions=A, device=dev)
opt = optim.RMSprop(model.parameters(), lr=0.0006, alpha=0.99, eps=0.01)
batch = bench.make_plane_batch(T, B, A, dev, seed=1)
L = learner.FusedLearner(model, bench.FLAGS, T, B)
for _ in range(5):
    L.step(batch, opt); L.stats(batch)
torch.cuda.synchronize()
# host-only timings with the GPU kept busy
ts = {"key": [], "step": [], "replay_only": [], "stats_host": [], "learn": []}
g = next(iter(L._graphs.values()))
for i in range(300):
    t0 = time.perf_counter_ns(); L._graph_key(batch, opt); t1 = time.perf_counter_ns()
    ts["key"].append(t1 - t0)
for i in range(200):
    torch.cuda.synchronize()
    t0 = time.perf_counter_ns(); L.step(batch, opt); t1 = time.perf_counter_ns()
    ts["step"].append(t1 - t0)
    torch.cuda.synchronize()
    t0 = time.perf_counter_ns(); g.replay(); t1 = time.perf_counter_ns()
    ts["replay_only"].append(t1 - t0)
    torch.cuda.synchronize()
    t0 = time.perf_counter_ns(); L.stats(batch); t1 = time.perf_counter_ns()
    ts["stats_host"].append(t1 - t0)
    torch.cuda.synchronize()
for k, v in ts.items():
    if v: print(f"{k:12s} median {statistics.median(v)/1e3:7.2f} us")
pr = cProfile.Profile()
pr.enable()
for i in range(300):
    learner.learn(bench.FLAGS, None, model, batch, (), opt, None)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
