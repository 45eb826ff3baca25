import sys
sys.path.insert(0, ".")
import torch
from paper_2502_02395_b200.program import Program
nb, m, n, k, ta, tb, cfg = [int(x) for x in sys.argv[1:8]]
A = torch.randn(nb, k if ta else m, m if ta else k, dtype=torch.float64, device="cuda")
B = torch.randn(nb, n if tb else k, k if tb else n, dtype=torch.float64, device="cuda")
C = torch.randn(nb, m, n, dtype=torch.float64, device="cuda")
beta = 1.0 if k == 64 else 0.0
probs = [(A[i].data_ptr(), B[i].data_ptr(), C[i].data_ptr(), m, n, k, A.shape[2], B.shape[2], n, 0, 1.0, beta) for i in range(nb)]
prog = Program(torch.device("cuda")); prog.gemm(ta, tb, probs, tile_cfg=cfg); prog.finalize()
for _ in range(3): prog.run()
torch.cuda.synchronize()
