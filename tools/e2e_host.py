"""Host-side timing of the e2e learn() loop (plane-store batches through DeviceInfeed):
per-step wall time split into infeed get / put / step launch / stats (sync) / release.

    python tools/e2e_host.py [STEPS]
"""
import statistics
import sys
import time
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1910_03552_b200 import learner, optim  # noqa: E402
from paper_1910_03552_b200.atari_net import AtariNet  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
dev = torch.device("cuda")
T, B, A = 80, 32, 6
model = AtariNet(num_actions=A, device=dev)
opt = optim.RMSprop(model.parameters(), lr=0.0006, alpha=0.99, eps=0.01)
src = [bench.make_plane_batch(T, B, A, dev, seed=200 + 7 * i) for i in range(2)]
infeed = learner.DeviceInfeed(src[0], dev)
host = []
for b in src:
    h = infeed.alloc_host()
    for k, v in b.items():
        h[k].copy_(v)
    host.append(h)
L = learner.FusedLearner(model, bench.FLAGS, T, B)
ph = {k: [] for k in ("get", "put", "step", "stats", "release", "total")}


def run(n, record):
    infeed.put(host[0])
    for i in range(n):
        t0 = time.perf_counter()
        b = infeed.get()
        t1 = time.perf_counter()
        if i + 1 < n:
            infeed.put(host[(i + 1) % 2])
        t2 = time.perf_counter()
        L.step(b, opt, None, ())
        t3 = time.perf_counter()
        L.stats(b)
        t4 = time.perf_counter()
        infeed.release()  # (optional: get() releases the previous slot itself)
        t5 = time.perf_counter()
        if record:
            for k, v in zip(("get", "put", "step", "stats", "release", "total"),
                            (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t5 - t0)):
                ph[k].append(v * 1e6)


run(8, False)
torch.cuda.synchronize()
run(steps, True)
for k, v in ph.items():
    print(f"{k:8s} median {statistics.median(v):8.1f} us  mean {statistics.mean(v):8.1f} us")

# host-only cost of stats() and learn() pieces with the GPU idle
infeed.put(host[0])
b = infeed.get()
L.step(b, opt, None, ())
torch.cuda.synchronize()
ts = []
for _ in range(50):
    t0 = time.perf_counter()
    L.stats(b)
    ts.append((time.perf_counter() - t0) * 1e6)
print(f"stats() with the GPU idle: median {statistics.median(ts):.1f} us")
ts = []
for _ in range(50):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L.step(b, opt, None, ())
    ts.append((time.perf_counter() - t0) * 1e6)
print(f"step() launch: median {statistics.median(ts):.1f} us")
