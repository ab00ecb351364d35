"""Per-replay cost of CUDA graphs on this box: a graph of one / two tiny kernels and of the
ZoomR step, replayed back to back (CUDA events around N replays)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
x = torch.zeros(1024, device="cuda")


def per_replay(g, n=200):
    for _ in range(10):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


res = {}
for nk in (1, 2, 4):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        x.add_(1)
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        for _ in range(nk):
            x.add_(1)
    res[f"tiny_kernels_{nk}_us_per_replay"] = per_replay(g)
    # the same kernels launched eagerly
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        for _ in range(nk):
            x.add_(1)
    e1.record()
    torch.cuda.synchronize()
    res[f"tiny_kernels_{nk}_eager_us_per_iter"] = e0.elapsed_time(e1) * 1e3 / 200
print(json.dumps(res))
