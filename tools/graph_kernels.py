"""In-graph kernel durations of the cfg1 learner step (CUPTI through torch.profiler):
per-kernel mean device time over replays and the idle gaps between kernels.

    python tools/graph_kernels.py [REPLAYS]
"""
import collections
import os
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1910_03552_b200 import learner, optim  # noqa: E402
from paper_1910_03552_b200.atari_net import AtariNet  # noqa: E402
from torch.profiler import profile, ProfilerActivity  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
work = sys.argv[2] if len(sys.argv) > 2 else "cfg1"
dev = torch.device("cuda")
if work.startswith("inf"):  # actor inference graph at k = int(work[3:])
    from paper_1910_03552_b200.inference import ActorInference
    k = int(work[3:])
    model = AtariNet(num_actions=6, device=dev)
    inf = ActorInference(model, graph_buckets=(k,))
    ib = bench.make_batch(0, k, 6, dev, seed=1)
    obs = {key: ib[key] for key in ("frame", "reward", "done", "last_action")}
    inf(obs)
    g = inf._graphs[k][0]
    run = g.replay
else:
    T, B, A, lstm = dict(cfg1=(80, 32, 6, False), cfg3=(80, 32, 18, True), cfg4=(80, 4096, 18, False),
                         cfg4s=(80, 512, 18, False))[work]
    model = AtariNet(num_actions=A, use_lstm=lstm, device=dev)
    opt = optim.RMSprop(model.parameters(), lr=0.0006, alpha=0.99, eps=0.01)
    batch = bench.make_batch(T, B, A, dev, seed=1)
    L = learner.FusedLearner(model, bench.FLAGS, T, B)
    run = lambda: L.step(batch, opt)  # noqa: E731
for _ in range(4):
    run()
torch.cuda.synchronize()
bg = int(os.environ.get("BP_GK_H2D_MB", "0"))  # background pinned H2D copies (e2e contention)
if bg:
    hbuf = torch.empty(bg << 20, dtype=torch.uint8, pin_memory=True)
    dbuf = torch.empty(bg << 20, dtype=torch.uint8, device=dev)
    cstream = torch.cuda.Stream()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    if bg:
        with torch.cuda.stream(cstream):
            for _ in range(reps * 2):
                dbuf.copy_(hbuf, non_blocking=True)
    for _ in range(reps):
        run()
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA" and not e.name.startswith("Memcpy")], key=lambda e: e.time_range.start)
# a step starts at prep_kernel, or (prep folded into conv1, the default) at the u8 conv1 GEMM
first = "prep_kernel" if any("prep_kernel" in e.name for e in ev) else "umma_gemm_kernel<32, 0, 0, 128, true, 1, "
steps, cur = [], []
for e in ev:
    if first in e.name and cur:
        steps.append(cur)
        cur = []
    cur.append(e)
steps.append(cur)
steps = [s for s in steps if s and first in s[0].name]
k = collections.Counter(len(s) for s in steps).most_common(1)[0][0]  # the usual kernel count
full = [s for s in steps if len(s) == k]
print(f"{len(steps)} replays ({len(full)} with the usual {k} kernels per step)")
steps = full
tot = 0.0
for i in range(k):
    d = sum(s[i].time_range.elapsed_us() for s in steps) / len(steps)
    gap = sum((s[i].time_range.start - s[i - 1].time_range.end) for s in steps if i > 0) / len(steps)
    tot += d
    print(f"{i:3d} {d:8.1f} us  gap-before {gap:6.1f}  {steps[0][i].name[:90]}")
span = sum(s[-1].time_range.end - s[0].time_range.start for s in steps) / len(steps)
print(f"sum of kernel times {tot:.1f} us, step span {span:.1f} us")
if len(sys.argv) > 3:  # timeline of the second replay: start / end offsets per kernel
    s = steps[1] if len(steps) > 1 else steps[0]
    t0 = s[0].time_range.start
    for e in s:
        print(f"  {e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f}  {e.name[:60]}")
    allev = [e for e in ev if s[0].time_range.start <= e.time_range.start <= s[-1].time_range.end]
    print("events in window:", len(allev), "step kernels:", len(s))
