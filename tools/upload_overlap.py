"""Pipelined gather (thread pool, numpy -> pinned staging) + H2D (one stream),
the scheme DeviceH2.from_host uses, at several thread counts / chunk sizes:
how much of gather and DMA overlap on this host."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

nbytes = 864 << 20
blk = 256 * 256
arrs = [np.random.default_rng(i).standard_normal(blk) for i in range(nbytes // (8 * blk))]
total = sum(a.nbytes for a in arrs)
pinned = torch.empty(total // 8, dtype=torch.float64, pin_memory=True)
hv = pinned.numpy()
dev = torch.empty(total // 8, dtype=torch.float64, device="cuda")
st = torch.cuda.Stream()


def fill(lo, hi):
    for i in range(lo, hi):
        hv[i * blk:(i + 1) * blk] = arrs[i]


def pipelined(threads, chunk_blocks, split_dma=1):
    nb = len(arrs)
    bounds = [(i, min(nb, i + chunk_blocks)) for i in range(0, nb, chunk_blocks)]
    with ThreadPoolExecutor(threads) as ex:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        futs = [ex.submit(fill, lo, hi) for lo, hi in bounds]
        with torch.cuda.stream(st):
            for (lo, hi), fu in zip(bounds, futs):
                fu.result()
                dev[lo * blk:hi * blk].copy_(pinned[lo * blk:hi * blk], non_blocking=True)
        st.synchronize()
        return time.perf_counter() - t0


for threads in (4, 8, 12, 16):
    for cb in (8, 32, 128):
        pipelined(threads, cb)
        dt = min(pipelined(threads, cb) for _ in range(3))
        print(f"pipelined threads {threads:2d} chunk {cb * blk * 8 >> 20:4d} MB: {dt * 1e3:6.1f} ms "
              f"{total / dt / 1e9:5.1f} GB/s", flush=True)
# DMA alone and gather alone for reference
torch.cuda.synchronize()
t0 = time.perf_counter()
dev.copy_(pinned, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D alone {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
with ThreadPoolExecutor(16) as ex:
    t0 = time.perf_counter()
    list(ex.map(lambda b: fill(*b), [(i, min(len(arrs), i + 8)) for i in range(0, len(arrs), 8)]))
    print(f"gather alone (16 threads) {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
