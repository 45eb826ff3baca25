import torch
A = torch.randn(4096, 256, 256, dtype=torch.float64, device="cuda")
B = torch.randn(4096, 256, 256, dtype=torch.float64, device="cuda")
for _ in range(3): C = torch.bmm(A, B)
torch.cuda.synchronize()
