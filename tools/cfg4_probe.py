"""Time the configs[3] learner step (AtariNet T=80 A=18, B=4096 and the B=512 shard) on one GPU."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1910_03552_b200 import learner, optim  # noqa: E402
from paper_1910_03552_b200.atari_net import AtariNet  # noqa: E402


def run(B, steps=5):
    T, A = 80, 18
    dev = torch.device("cuda")
    torch.manual_seed(0)
    m = AtariNet(num_actions=A, device=dev)
    opt = optim.RMSprop(m.parameters(), lr=4.8e-4, alpha=0.99, eps=0.01)
    batch = bench.make_batch(T, B, A, dev, seed=1)
    L = learner.FusedLearner(m, bench.FLAGS, T, B)
    t0 = time.time()
    for _ in range(3):
        L.step(batch, opt)
    torch.cuda.synchronize()
    print("warmup", time.time() - t0, "s; mem GB", torch.cuda.max_memory_allocated() / 1e9)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        L.step(batch, opt)
    e1.record()
    e1.synchronize()
    s = e0.elapsed_time(e1) / steps / 1e3
    n = (T + 1) * B
    flops = 2 * n * (3 * sum(bench.MACS.values()) - bench.MACS["conv1"])
    print(f"B={B}: {s*1e3:.2f} ms/step  {T*B/s/1e6:.3f} M env-frames/s  {flops/s/1e12:.0f} TFLOP/s")
    br = bench.kernel_breakdown(L, batch, opt, iters=3)
    print({k: round(v * 1e3, 3) for k, v in br.items()})


if __name__ == "__main__":
    for B in [int(x) for x in sys.argv[1:]] or [512, 4096]:
        run(B)
