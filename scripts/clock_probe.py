"""Run our tcgen05 GEMM and cuBLAS back to back for ~2 s each (graph
replays) while NVML samples SM clock and power: separates kernel efficiency
from power/clock limits."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml
import torch
from paper_1909_00562_b200 import binding, build

build.build()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0]))
M = N = K = 8192
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda")
Cb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
s = torch.cuda.Stream()
for k, v in (a.split("=") for a in sys.argv[1:]):
    binding.attn_softmax_set_option(k, int(v))
binding.attn_softmax_set_option("debug_epilogue", 1)


def graph(fn, n=20):
    with torch.cuda.stream(s):
        fn(); fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n):
            fn()
    return g, n


def probe(name, fn):
    g, n = graph(fn)
    samples = []
    stop = threading.Event()

    def run():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            time.sleep(0.02)
    th = threading.Thread(target=run); th.start()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.time(); reps = 0
    e0.record()
    while time.time() - t0 < 2.0:
        g.replay(); reps += 1
        if reps % 5 == 0: torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    ms = e0.elapsed_time(e1) / (reps * n)
    sm = sorted(x[0] for x in samples[len(samples)//3:])
    pw = sorted(x[1] for x in samples[len(samples)//3:])
    rs = set(x[2] for x in samples[len(samples)//3:])
    print(f"{name:24s} {2*M*N*K/ms/1e9:7.1f} TF/s  sm {sm[len(sm)//2]} MHz  power {pw[len(pw)//2]:.0f} W  reasons {sorted(rs)}", flush=True)
    return 2*M*N*K/ms/1e9, sm[len(sm)//2]

for name, fn in (("ours", lambda: binding.attn_debug_gemm_bf16(M, N, K, A, 0, B, 0, C, stream=s)),
                 ("cublas", lambda: torch.matmul(A, B.T, out=Cb)),
                 ("ours", lambda: binding.attn_debug_gemm_bf16(M, N, K, A, 0, B, 0, C, stream=s)),
                 ("cublas", lambda: torch.matmul(A, B.T, out=Cb))):
    tf, mhz = probe(name, fn)
    print(f"   -> per-MHz {tf/mhz*1000:.1f} GF/s/MHz", flush=True)
