"""Microbenchmark of the grouped DMMA GEMM (both tile configs) vs torch.bmm (cuBLAS)."""
import sys, json
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2502_02395_b200.program import Program

def run(nb, m, n, k, ta, tb, cfg, beta=0.0, reps=20):
    A = torch.randn(nb, k if ta else m, m if ta else k, dtype=torch.float64, device="cuda")
    B = torch.randn(nb, n if tb else k, k if tb else n, dtype=torch.float64, device="cuda")
    C = torch.randn(nb, m, n, dtype=torch.float64, device="cuda")
    C0 = C.clone()
    probs = [(A[i].data_ptr(), B[i].data_ptr(), C[i].data_ptr(), m, n, k, A.shape[2], B.shape[2], n, 0, 1.0, beta)
             for i in range(nb)]
    prog = Program(torch.device("cuda"))
    prog.gemm(ta, tb, probs, tile_cfg=cfg)
    prog.finalize()
    prog.run(); torch.cuda.synchronize()
    opA = A.transpose(1, 2) if ta else A
    opB = B.transpose(1, 2) if tb else B
    ref = torch.bmm(opA, opB) + beta * C0
    err = ((C - ref).abs().max() / ref.abs().max()).item()
    if beta != 0.0:
        C.copy_(C0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        prog.run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    e0.record()
    for _ in range(reps):
        torch.bmm(opA, opB)
    e1.record(); torch.cuda.synchronize()
    msb = e0.elapsed_time(e1) / reps
    fl = 2.0 * nb * m * n * k
    return dict(nb=nb, m=m, n=n, k=k, ta=ta, tb=tb, cfg=cfg, tflops=fl / ms / 1e9, bmm_tflops=fl / msb / 1e9, err=err)

out = []
for (nb, m, n, k, ta, tb) in [(256, 256, 256, 256, 0, 0), (256, 256, 256, 256, 1, 0), (4096, 256, 256, 256, 0, 0),
                              (64, 512, 512, 512, 0, 0), (1024, 448, 64, 64, 0, 1), (1024, 192, 192, 64, 0, 1),
                              (16, 900, 900, 900, 1, 0)]:
    for cfg in (2, 7, 8):
        beta = 1.0 if (k == 64) else 0.0
        r = run(nb, m, n, k, ta, tb, cfg, beta)
        out.append(r)
        print(json.dumps(r), flush=True)
