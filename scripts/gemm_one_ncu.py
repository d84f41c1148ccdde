"""One debug-GEMM launch for ncu (pair mode from argv)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_00562_b200 import binding
M, N, K, pair = (int(x) for x in sys.argv[1:5])
binding.attn_softmax_set_option("cta_pair", 8 if pair == 2 else 0)
binding.attn_softmax_set_option("wide_tiles", 8 if pair == 4 else 0)
binding.attn_softmax_set_option("debug_epilogue", 1)
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda")
for _ in range(3):
    binding.attn_debug_gemm_bf16(M, N, K, A, 0, B, 0, C)
torch.cuda.synchronize()
