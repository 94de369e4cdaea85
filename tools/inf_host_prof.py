"""Host-side cost of one ActorInference call (graph path, k = 32): cProfile hot spots."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1910_03552_b200.atari_net import AtariNet  # noqa: E402
from paper_1910_03552_b200.inference import ActorInference  # noqa: E402

dev = torch.device("cuda")
m = AtariNet(num_actions=6, device=dev)
m.eval()
inf = ActorInference(m, graph_buckets=(32,))
ib = bench.make_batch(0, 32, 6, dev, seed=1)
obs = {k: ib[k] for k in ("frame", "reward", "done", "last_action")}
for _ in range(10):
    inf(obs)
torch.cuda.synchronize()
ts = []
for _ in range(200):
    t0 = time.perf_counter()
    inf(obs)
    ts.append(time.perf_counter() - t0)
torch.cuda.synchronize()
ts.sort()
print(f"host time per call (no sync) median {ts[100] * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(300):
    inf(obs)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
g, st, _ = inf._graphs[32]
ts = []
for _ in range(200):
    t0 = time.perf_counter()
    g.replay()
    ts.append(time.perf_counter() - t0)
torch.cuda.synchronize()
ts.sort()
print(f"graph.replay() alone median {ts[100] * 1e6:.1f} us")
ts = []
for _ in range(200):
    t0 = time.perf_counter()
    g.replay()
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
ts.sort()
print(f"graph.replay() + sync median {ts[100] * 1e6:.1f} us")
# per-part breakdown of the graph-path call
import ctypes as C  # noqa: E402
from paper_1910_03552_b200 import _native as N  # noqa: E402
parts = {k: [] for k in ("inputs", "prep", "copies", "replay", "clone", "out")}
for _ in range(300):
    t0 = time.perf_counter()
    frames, reward, last_action, done = inf._inputs(obs)
    t1 = time.perf_counter()
    k = frames.shape[0]
    m.buffers_for(32)
    m.mirror_stale()
    t2 = time.perf_counter()
    pairs = [(st["frames"], frames), (st["reward"], reward), (st["last_action"], last_action)]
    n = len(pairs)
    dsts, srcs, nbytes = (C.c_void_p * n)(), (C.c_void_p * n)(), (C.c_size_t * n)()
    for i, (d, src) in enumerate(pairs):
        dsts[i], srcs[i], nbytes[i] = d.data_ptr(), src.data_ptr(), src.numel() * src.element_size()
    N.lib().bp_copy_many(dsts, srcs, nbytes, n, torch.cuda.current_stream().cuda_stream)
    t3 = time.perf_counter()
    g.replay()
    t4 = time.perf_counter()
    o = st["outbuf"].clone()
    t5 = time.perf_counter()
    out = dict(action=o[:8 * 32].view(torch.int64)[:k].view(1, k), model_version=torch.full((1, k), 0, dtype=torch.int64, device=dev))
    t6 = time.perf_counter()
    for key, a, b in (("inputs", t0, t1), ("prep", t1, t2), ("copies", t2, t3), ("replay", t3, t4), ("clone", t4, t5), ("out", t5, t6)):
        parts[key].append(b - a)
torch.cuda.synchronize()
for key, v in parts.items():
    v.sort()
    print(f"  {key:8s} median {v[len(v) // 2] * 1e6:6.1f} us")
# eager path (no graph buckets): host time per call and the Python hot spots
eager = ActorInference(m)
for _ in range(10):
    eager(obs)
torch.cuda.synchronize()
ts = []
for _ in range(200):
    t0 = time.perf_counter()
    eager(obs)
    ts.append(time.perf_counter() - t0)
torch.cuda.synchronize()
ts.sort()
print(f"eager host time per call (no sync) median {ts[100] * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(300):
    eager(obs)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(16)
