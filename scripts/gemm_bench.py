"""tcgen05 GEMM core microbenchmark (debug entry) vs torch.matmul (cuBLAS).
Both are timed under CUDA-graph replay, so host-side work (tensor-map
encoding, ctypes) is excluded and the numbers are device time."""
import itertools, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_00562_b200 import binding, build

build.build()
shapes = [  # name, M, N, K, a_mn, b_mn
    ("one tile", 128, 256, 64, 0, 0),
    ("vocab_fwd T x V x d", 6400, 50000, 1024, 0, 0),
    ("dW_out chunk Vc x d x T", 2048, 1024, 6400, 1, 1),
    ("dHc chunk T x d x Vc", 6400, 1024, 2048, 0, 1),
    ("dlogits chunk T x Vc x d", 6400, 2048, 1024, 0, 0),
    ("square 8192", 8192, 8192, 8192, 0, 0),
    ("square 8192 K/MN", 8192, 8192, 8192, 0, 1),
    ("square 8192 MN/MN", 8192, 8192, 8192, 1, 1),
]
sel = [a for a in sys.argv[1:] if "=" not in a]
opts = dict(a.split("=") for a in sys.argv[1:] if "=" in a)
for k, v in opts.items():
    binding.attn_softmax_set_option(k, int(v))
s = torch.cuda.Stream()


def gtime(fn, n=10):
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for (name, M, N, K, amn, bmn), epi in itertools.product(shapes, (1,)):
    if sel and not any(x in name for x in sel):
        continue
    binding.attn_softmax_set_option("debug_epilogue", epi)
    A = torch.randn(K, M, device="cuda").bfloat16() if amn else torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16() if bmn else torch.randn(N, K, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda")
    ms = gtime(lambda: binding.attn_debug_gemm_bf16(M, N, K, A, amn, B, bmn, C, stream=s))
    At = A.T if amn else A
    Bt = B if bmn else B.T
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ms_t = gtime(lambda: torch.matmul(At, Bt, out=out))
    fl = 2.0 * M * N * K
    tag = " [no store]" if epi else ""
    print(f"{name+tag:34s} ours {ms*1e3:8.1f} us {fl/ms/1e9:7.1f} TF/s | cublas {ms_t*1e3:8.1f} us "
          f"{fl/ms_t/1e9:7.1f} TF/s", flush=True)
binding.attn_softmax_set_option("debug_epilogue", 0)
