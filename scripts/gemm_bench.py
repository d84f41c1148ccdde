"""tcgen05 GEMM core microbenchmark (debug entry, fp32 TMA-store epilogue)
vs torch.matmul (cuBLAS) on the same shapes: isolates the mainloop and the
operand majors from the stage's epilogues."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_00562_b200 import binding, build

build.build()
shapes = [  # name, M, N, K, a_mn, b_mn
    ("vocab_fwd T x V x d", 6400, 50000, 1024, 0, 0),
    ("dW_out chunk Vc x d x T", 2048, 1024, 6400, 1, 1),
    ("dHc chunk T x d x Vc", 6400, 1024, 2048, 0, 1),
    ("dlogits chunk T x Vc x d", 6400, 2048, 1024, 0, 0),
    ("square 8192", 8192, 8192, 8192, 0, 0),
    ("square 8192 MN/MN", 8192, 8192, 8192, 1, 1),
]
import itertools
for (name, M, N, K, amn, bmn), epi in itertools.product(shapes, (0, 1)):
    binding.attn_softmax_set_option("debug_epilogue", epi)
    name = name + (" [no store]" if epi else "")
    A = torch.randn(K, M, device="cuda").bfloat16() if amn else torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16() if bmn else torch.randn(N, K, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda")
    for _ in range(3):
        binding.attn_debug_gemm_bf16(M, N, K, A, amn, B, bmn, C)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        binding.attn_debug_gemm_bf16(M, N, K, A, amn, B, bmn, C)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    At = A.T if amn else A
    Bt = B if bmn else B.T
    for _ in range(3):
        Ct = At @ Bt
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        Ct = At @ Bt
    e1.record()
    torch.cuda.synchronize()
    ms_t = e0.elapsed_time(e1) / n
    err = (C - Ct.float()).abs().max().item() / max(1e-6, Ct.float().abs().max().item())
    fl = 2.0 * M * N * K
    print(f"{name:28s} ours {ms*1e3:8.1f} us {fl/ms/1e9:7.1f} TF/s | cublas(bf16 out) {ms_t*1e3:8.1f} us "
          f"{fl/ms_t/1e9:7.1f} TF/s | relerr {err:.1e}", flush=True)
