"""Host<->device copy bandwidth probe (pinned, 1 GiB): H2D, D2H, both concurrently, and chunked."""
import json
import time

import torch

n = 1 << 28   # 1 GiB of fp32
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
out = {}


def timed(fn, reps=3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


out["h2d_GBs"] = 4 * n / timed(lambda: d.copy_(h, non_blocking=True)) / 1e9
out["d2h_GBs"] = 4 * n / timed(lambda: h.copy_(d, non_blocking=True)) / 1e9


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


out["both_GBs_each"] = 4 * n / timed(both) / 1e9
out["h2d_pageable_GBs"] = 4 * n / timed(lambda: d.copy_(torch.ones(1).expand(0) if False else h.clone(), non_blocking=False), 1) / 1e9
print(json.dumps(out))
