import torch
M = N = K = 8192
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
for _ in range(3):
    C = A @ B.T
A2 = torch.randn(6400, 1024, device="cuda").bfloat16()
W = torch.randn(50000, 1024, device="cuda").bfloat16()
for _ in range(3):
    L = A2 @ W.T
torch.cuda.synchronize()
