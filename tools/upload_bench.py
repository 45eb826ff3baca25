"""Host->device upload rates on the GPU box: threaded numpy gather into pinned
staging, pinned H2D, pageable H2D, and DeviceH2.from_host of a real config."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, ".")
import numpy as np
import torch

nbytes = 864 << 20
blk = 256 * 256
arrs = [np.random.default_rng(i).standard_normal(blk) for i in range(nbytes // (8 * blk))]
total = sum(a.nbytes for a in arrs)
pinned = torch.empty(total // 8, dtype=torch.float64, pin_memory=True)
hv = pinned.numpy()
dev = torch.empty(total // 8, dtype=torch.float64, device="cuda")


def gather(threads):
    chunks = np.array_split(np.arange(len(arrs)), threads)

    def run(ix):
        for i in ix:
            hv[i * blk:(i + 1) * blk] = arrs[i]

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, chunks))


for th in (1, 4, 8, 16, 32):
    gather(th)
    t0 = time.perf_counter()
    gather(th)
    dt = time.perf_counter() - t0
    print(f"gather {th:2d} threads: {total / dt / 1e9:.1f} GB/s", flush=True)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(pinned, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(f"pinned H2D: {total / dt / 1e9:.1f} GB/s", flush=True)
big = np.concatenate(arrs)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(torch.from_numpy(big))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(f"pageable H2D: {total / dt / 1e9:.1f} GB/s", flush=True)
print("cpus", os.cpu_count())
