"""Where the e2e step time goes (cfg1, plane-store batches): the pinned H2D copy rate alone,
the copy rate while learner steps run on the compute stream, and the e2e loop itself."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1910_03552_b200 import learner, optim  # noqa: E402
from paper_1910_03552_b200.atari_net import AtariNet  # noqa: E402
from paper_1910_03552_b200.learner import DeviceInfeed  # noqa: E402

dev = torch.device("cuda")
T, B, A = 80, 32, 6
model = AtariNet(num_actions=A, device=dev)
opt = optim.RMSprop(model.parameters(), lr=0.0006, alpha=0.99, eps=0.01)
src = [bench.make_plane_batch(T, B, A, dev, seed=200 + i) for i in range(2)]
infeed = DeviceInfeed(src[0], dev, depth=2)
host = []
for b in src:
    h = infeed.alloc_host()
    for k, v in b.items():
        h[k].copy_(v)
    host.append(h)
nbytes = infeed.bytes_per_batch
flat_h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
flat_d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
cs = torch.cuda.Stream()
N = 40


def copies(n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        e0.record(cs)
        for _ in range(n):
            flat_d.copy_(flat_h, non_blocking=True)
        e1.record(cs)
    return e0, e1


for _ in range(3):
    learner.learn(bench.FLAGS, None, model, src[0], (), opt, None)
torch.cuda.synchronize()
e0, e1 = copies(N)
e1.synchronize()
alone = N * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9
# copies concurrent with learner steps (no dependency between them)
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
s0.record()
e0, e1 = copies(N)
k = 0
while not e1.query():
    learner.learn(bench.FLAGS, None, model, src[0], (), opt, None)
    k += 1
s1.record()
torch.cuda.synchronize()
under = N * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9
step_ms = s0.elapsed_time(s1) / k
print(f"bytes per batch {nbytes}; H2D alone {alone:.1f} GB/s; H2D under learner steps {under:.1f} GB/s "
      f"({k} steps, {step_ms:.3f} ms per step meanwhile)")


# device-only learner steps (FusedLearner.step, no stats read-back): alone / under copies
L = learner.FusedLearner(model, bench.FLAGS, T, B)
for _ in range(3):
    L.step(src[0], opt)
torch.cuda.synchronize()
import ctypes  # noqa: E402
rt = ctypes.CDLL("libcuda.so.1")
for label in ("alone", "under copies", "alone (uploaded)", "under copies (uploaded)"):
    if "uploaded" in label and rt is not None:
        for g in L._graphs.values():
            rc = rt.cuGraphUpload(ctypes.c_void_p(g.raw_cuda_graph_exec()),
                                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
            print("cuGraphUpload rc", rc)
        torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if "under" in label:
        e0, e1 = copies(N)
    s0.record()
    for _ in range(30):
        L.step(src[0], opt)
    s1.record()
    torch.cuda.synchronize()
    print(f"device-only step {label}: {s0.elapsed_time(s1) / 30:.4f} ms")
# learn() (stats read each step) alone / under copies
for label in ("alone", "under copies"):
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if label != "alone":
        e0, e1 = copies(N)
    s0.record()
    for _ in range(30):
        learner.learn(bench.FLAGS, None, model, src[0], (), opt, None)
    s1.record()
    torch.cuda.synchronize()
    print(f"learn() step {label}: {s0.elapsed_time(s1) / 30:.4f} ms")


def e2e_run(nsteps, sync_each=True):
    ahead = min(infeed.depth - 1, nsteps)
    for j in range(ahead):
        infeed.put(host[j % 2])
    for i in range(nsteps):
        b = infeed.get()
        if i + ahead < nsteps:
            infeed.put(host[(i + ahead) % 2])
        learner.learn(bench.FLAGS, None, model, b, (), opt, None)


e2e_run(6)
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    e2e_run(N)
    e1.record()
    e1.synchronize()
    print(f"e2e {e0.elapsed_time(e1) / N:.4f} ms per step (host {1e3 * (time.perf_counter() - t0) / N:.4f})")
