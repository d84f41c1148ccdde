"""One GEMM shape through the tcgen05 debug entry, a few launches (for ncu).
usage: gemm_one.py M N K a_mn b_mn [pair=1|2] [epi=0|1]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_00562_b200 import binding
M, N, K, amn, bmn = (int(x) for x in sys.argv[1:6])
pair = int(sys.argv[6]) if len(sys.argv) > 6 else 2
epi = int(sys.argv[7]) if len(sys.argv) > 7 else 0
binding.attn_softmax_set_option("cta_pair", 8 if pair == 2 else 0)
binding.attn_softmax_set_option("debug_epilogue", epi)
A = torch.randn(K, M, device="cuda").bfloat16() if amn else torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(K, N, device="cuda").bfloat16() if bmn else torch.randn(N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda")
for _ in range(4):
    binding.attn_debug_gemm_bf16(M, N, K, A, amn, B, bmn, C)
torch.cuda.synchronize()
