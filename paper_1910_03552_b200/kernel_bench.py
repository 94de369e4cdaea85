"""Device-timed micro-benchmarks of the HBM-bound kernels (V-trace, fused loss,
clip + RMSProp), with algorithmic-byte rooflines.

    python -m paper_1910_03552_b200.kernel_bench [--iters 50]

Each measured launch is preceded by an L2 flush (a 256 MB memset, > 126 MB
L2) outside the timed window; time = CUDA events on the launching stream.
Algorithmic bytes per launch:
  from_logits : T*B*(8A + 8 + 3*4 + 5*4) + 4B     = T*B*(8A+40) + 4B
  learner loss: T*B*(8A + 8 + 1 + 4 + 4  +  4A + 4 + 4 + 4) + 8B  (reads beh +
                learner logits, action, done, reward, baseline; writes
                d_logits, d_baseline, vs, pg)   = T*B*(12A+29) + 8B
  clip+rmsprop: 4n (sumsq) + 20n (read p,g,s; write p,s) [+4n clipped grads]
"""
from __future__ import annotations

import argparse
import json
import os

import torch

from paper_1910_03552_b200._tensors import graph_capture


def _peaks():
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Timer:
    def __init__(self, flush_bytes=256 << 20):
        self.flush = torch.empty(flush_bytes, dtype=torch.uint8, device="cuda")

    def time(self, fn, iters=50, warmup=5, flush=True, graph=True):
        """Median / min device time of fn().  With graph=True fn is captured once in
        a CUDA graph so host-side Python overhead cannot leak into the window
        (the preceding flush keeps the GPU busy while the replay is submitted)."""
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        if graph:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                fn()
                with graph_capture(g, stream=side):
                    fn()
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            fn = g.replay
        s = torch.cuda.current_stream()
        ts = []
        for _ in range(iters):
            if flush:
                self.flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        ts.sort()
        return {"median_s": ts[len(ts) // 2], "min_s": ts[0]}


    def time_rotating(self, fns, reps=4, iters=5):
        """Steady-state device time per launch: the launches in `fns` (each on its own
        buffer set, together > 2x the 126 MB L2, so every launch streams from HBM) are
        captured back to back `reps` times in one CUDA graph; the replay is timed with
        CUDA events and divided by the launch count.  Unlike a single flushed launch,
        no graph-launch latency or event granularity (~2 us) enters the figure."""
        for f in fns:
            f()
        torch.cuda.synchronize()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with graph_capture(g, stream=side):
                for _ in range(reps):
                    for f in fns:
                        f()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        s = torch.cuda.current_stream()
        ts = []
        n = reps * len(fns)
        for _ in range(iters):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3 / n)
        ts.sort()
        return {"median_s": ts[len(ts) // 2], "min_s": ts[0], "launches": n}


def _nsets(set_bytes):
    return max(2, min(32, -(-(400 << 20) // set_bytes)))


def vtrace_bytes(T, B, A):
    return T * B * (8 * A + 40) + 4 * B


def loss_bytes(T, B, A):
    return T * B * (12 * A + 29) + 8 * B


def _vtrace_inputs(T, B, A, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    beh = torch.randn(T, B, A, device="cuda", generator=g)
    tgt = torch.randn(T, B, A, device="cuda", generator=g)
    act = torch.randint(0, A, (T, B), device="cuda", generator=g)
    disc = 0.99 * (torch.rand(T, B, device="cuda", generator=g) > 0.05).float()
    rew = torch.rand(T, B, device="cuda", generator=g) * 2 - 1
    val = torch.randn(T, B, device="cuda", generator=g)
    boot = torch.randn(B, device="cuda", generator=g)
    return beh, tgt, act, disc, rew, val, boot


def bench_vtrace(T, B, A, timer, iters=50, rotate=True):
    """from_logits device time per launch.  rotate=True: steady state over rotating
    HBM-resident buffer sets (Timer.time_rotating); False: one launch after an L2 flush."""
    from . import vtrace

    nbytes = vtrace_bytes(T, B, A)
    if rotate:
        fns = []
        for i in range(_nsets(nbytes)):
            x = _vtrace_inputs(T, B, A, i)
            fns.append(lambda x=x: vtrace.from_logits(*x))
        r = timer.time_rotating(fns, reps=max(1, 64 // len(fns)), iters=max(3, iters // 4))
    else:
        x = _vtrace_inputs(T, B, A, 0)
        r = timer.time(lambda: vtrace.from_logits(*x), iters)
    return dict(kernel="vtrace_from_logits", T=T, B=B, A=A, bytes=nbytes, **r,
                gbs=nbytes / r["median_s"] / 1e9, timing="rotating" if rotate else "flushed")


def _loss_call(T, B, A, seed, ll, cfg):
    g = torch.Generator(device="cuda").manual_seed(seed)
    logits = torch.randn(T, B, A, device="cuda", generator=g)
    baseline = torch.randn(T + 1, B, device="cuda", generator=g)
    beh = torch.randn(T, B, A, device="cuda", generator=g)
    act = torch.randint(0, A, (T, B), device="cuda", generator=g)
    rew = torch.rand(T, B, device="cuda", generator=g)
    done = torch.rand(T, B, device="cuda", generator=g) < 0.05
    vs = torch.empty(T, B, device="cuda")
    pg = torch.empty(T, B, device="cuda")
    dl = torch.empty(T, B, A, device="cuda")
    db = torch.empty(T + 1, B, device="cuda")
    return lambda: ll(logits, baseline, beh, act, rew, done, cfg, d_logits=dl, d_baseline=db,  # noqa
                      vs=vs, pg_advantages=pg)


def bench_loss(T, B, A, timer, iters=50, rotate=True):
    from . import learner_ops as lo

    ll = lo.LearnerLoss()
    cfg = lo.VtraceConfig()
    nbytes = loss_bytes(T, B, A)
    if rotate:
        fns = [_loss_call(T, B, A, i, ll, cfg) for i in range(_nsets(nbytes))]
        r = timer.time_rotating(fns, reps=max(1, 64 // len(fns)), iters=max(3, iters // 4))
    else:
        r = timer.time(_loss_call(T, B, A, 0, ll, cfg), iters)
    return dict(kernel="learner_loss", T=T, B=B, A=A, bytes=nbytes, **r,
                gbs=nbytes / r["median_s"] / 1e9, timing="rotating" if rotate else "flushed")


def bench_rmsprop(n, timer, iters=50):
    from . import optim

    p = torch.nn.Parameter(torch.randn(n, device="cuda"))
    opt = optim.RMSprop([p], lr=0.00048, alpha=0.99, eps=0.01)
    p.grad.normal_()
    fn = lambda: opt.step(max_norm=40.0)  # noqa: E731
    r = timer.time(fn, iters)
    nbytes = 28 * n
    return dict(kernel="clip_rmsprop", n=n, bytes=nbytes, **r, gbs=nbytes / r["median_s"] / 1e9)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--flushed", action="store_true", help="single flushed launches instead of rotation")
    args = ap.parse_args()
    peak, kind = _peaks()
    timer = Timer()
    rows = []
    cfgs = [(20, 32, 6), (80, 32, 18), (80, 512, 18), (80, 4096, 18), (80, 16384, 18),
            (80, 65536, 18)]
    if args.quick:
        cfgs = [(20, 32, 6), (80, 4096, 18)]
    for T, B, A in cfgs:
        rows.append(bench_vtrace(T, B, A, timer, args.iters, rotate=not args.flushed))
        rows.append(bench_loss(T, B, A, timer, args.iters, rotate=not args.flushed))
    for n in (1_694_000, 6_214_000):
        rows.append(bench_rmsprop(n, timer, args.iters))
    for r in rows:
        r["frac_of_hbm"] = r["gbs"] / peak
        r["peak_kind"] = kind
        print(json.dumps(r))


if __name__ == "__main__":
    main()
