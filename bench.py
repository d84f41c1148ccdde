"""Benchmark of the B200 attention-softmax stage (fwd + bwd), bench contract.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config paper]
                  [--impl ours|reference] [--no-cpu-baseline]

N > 1 is launched by torchrun (one process per GPU, NCCL): each rank holds
its own B = 128 sentences (weak scaling, BASELINE.json configs[2]) and the
library allreduces dW_c / dW_out / loss over NVLink inside the call.

Printed (rank 0, one JSON line): target tokens/s of the whole job (`value`,
device-timed, inputs resident), `e2e` (the same metric through the C-ABI
host-buffer entry point with the per-step H2D copies of the activations and
the D2H read of the loss inside the timed region), `roofline` of the dominant
kernel (the V-chunked vocab-backward tcgen05 GEMM launches) from CUDA events
recorded by the library on the launching stream, `cpu_baseline` (the fp64
oracle on a bounded sample of the same workload, host cores), clocks sampled
during the timed region, and the launch count.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "attention-softmax fwd+bwd target tokens/sec at 1/2/4/8 B200; tensor-pipe % of peak"
UNIT = "target tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="paper")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-sentences", type=int, default=0)
    ap.add_argument("--no-next", action="store_true",
                    help="skip the SURVEY §8(f) NEXT-row measurements (general score, bias, Adam)")
    ap.add_argument("--force-comm", action="store_true",
                    help="use the NCCL communicator even with one rank (exercises the path)")
    return ap.parse_args()


def workload_desc(cfg, world):
    return {"workload": f"{cfg.name}: per-GPU B={cfg.B} sentences, N={cfg.N} target / "
                        f"M={cfg.M} source steps, d={cfg.d}, V={cfg.V}, {cfg.dtype}, "
                        f"lengths={cfg.lengths}",
            "B_per_gpu": cfg.B, "N": cfg.N, "M": cfg.M, "d": cfg.d, "V": cfg.V,
            "global_batch": cfg.B * world, "parallelism": f"dp{world}",
            "l2": "flushed between timed steps (256 MiB write outside the timed events)"}


def build_id(binding):
    """The library's version string and a hash of the sources it was built
    from (csrc/ and include/; .git does not travel to the GPU box)."""
    import hashlib
    h = hashlib.sha1()
    for sub in ("paper_1909_00562_b200/csrc", "include"):
        d = os.path.join(ROOT, sub)
        for f in sorted(os.listdir(d)):
            with open(os.path.join(d, f), "rb") as fh:
                h.update(f.encode() + fh.read())
    return {"library": binding.lib().attn_version().decode(), "source_sha1": h.hexdigest()[:12]}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=d.get("hbm_gbs", 6443.5), bf16=d.get("bf16_tflops", 1678.0),
                    bf16_sus=d.get("bf16_tflops_sustained", d.get("bf16_tflops", 1678.0)),
                    src="measured (MEASURED_PEAKS.json)")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0,
                src="fallback (B200_PROFILING.md)")


# ------------------------------------------------------------ clocks ------
class ClockSampler:
    """Samples SM clock, power and throttle reasons every 5 ms through NVML
    (nvidia-ml-py) while the timed region runs."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.stop_ev = threading.Event()
        self.err = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis else self.index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml unavailable: {e}"

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                self.samples.append((sm, rs, pw))
            except Exception as e:  # noqa: BLE001
                self.err = str(e)
                return
            time.sleep(0.005)

    def stop(self):
        if self.err and not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err]}
        self.stop_ev.set()
        self.th.join(timeout=2)
        sm = sorted(s[0] for s in self.samples)
        reasons = sorted({n for _, rs, _ in self.samples for n, bit in self.REASONS.items()
                          if rs & bit})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(sm),
                "power_w_max": max(s[2] for s in self.samples) if self.samples else None}


# ------------------------------------------------------------ reference ---
_W_CACHE = {}


def cpu_oracle_run(cfg, n_sent: int, seed_offset: int = 0):
    """Time the fp64 oracle (as it stands) on n_sent sentences of the
    workload with the full d and V.  Returns (valid tokens, seconds)."""
    import numpy as np
    from oracle import attn_softmax_oracle as O
    from synthetic import make_inputs, make_weights
    if cfg.name not in _W_CACHE:
        _W_CACHE[cfg.name] = make_weights(cfg)
    inp = make_inputs(cfg, sentences=range(seed_offset, seed_offset + n_sent),
                      with_weights=False)
    inp.update(_W_CACHE[cfg.name])
    scale = 1.0 / max(1, int(inp["tgt_len"].sum()))
    t0 = time.perf_counter()
    O.fwd_bwd(inp["H_dec"], inp["H_enc"], inp["src_len"], inp["tgt_len"], inp["tgt_ids"],
              inp["W_c"], inp["W_out"], scale)
    dt = time.perf_counter() - t0
    return int(np.sum(inp["tgt_len"])), dt


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        if n:
            return int(max(n))
    except Exception:
        pass
    return os.cpu_count()


def cpu_baseline(cfg, target_s=12.0, fixed=0):
    """Bounded sample: grow the sentence count until one run takes ~target_s."""
    n = fixed or 2
    tok, dt = cpu_oracle_run(cfg, n)
    if not fixed:
        while dt < target_s / 3 and n < cfg.B:
            n = min(cfg.B, max(n + 1, int(n * target_s / max(dt, 1e-3) * 0.6)))
            tok, dt = cpu_oracle_run(cfg, n)
    res = {"value": tok / dt, "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
           "sample": f"{n} of {cfg.B} sentences of {cfg.name} (full d={cfg.d}, V={cfg.V}), "
                     f"{tok} target tokens, one fwd+bwd in {dt:.2f} s, numpy fp64",
           "cpu_model": cpu_model(), "nproc": os.cpu_count()}
    # the same oracle on one BLAS thread, on a smaller sample
    try:
        from threadpoolctl import threadpool_limits
        n1 = max(1, min(n, 8))
        with threadpool_limits(limits=1, user_api="blas"):
            tok1, dt1 = cpu_oracle_run(cfg, n1)
        res["one_thread"] = {"value": tok1 / dt1, "sample": f"{n1} sentences, {tok1} tokens, "
                                                            f"{dt1:.2f} s"}
    except Exception as e:  # noqa: BLE001
        res["one_thread"] = {"value": None, "error": str(e)[:200]}
    return res


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    # sized so the whole --steps K --warmup W run ends within minutes
    per_step_target = max(1.0, 150.0 / max(1, args.steps + args.warmup))
    n = 1
    tok, dt = cpu_oracle_run(cfg, n)
    n = max(1, min(cfg.B, int(per_step_target / max(dt, 1e-3))))
    for i in range(args.warmup):
        cpu_oracle_run(cfg, n, seed_offset=i)
    total_tok, total_t = 0, 0.0
    for i in range(args.steps):
        tok, dt = cpu_oracle_run(cfg, n, seed_offset=i)
        total_tok += tok
        total_t += dt
    v = total_tok / total_t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total_t / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_desc(cfg, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
                             "sample": f"{n} sentences per step of {cfg.name} (full d, V)",
                             "cpu_model": cpu_model(), "nproc": os.cpu_count()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ ours --------
def verify_exchange(binding, st, call_args, out, comm, stream, barrier):
    """X step check (N > 1, or --force-comm): the gradients the call
    allreduces in flight (dW_out per chunk group, dW_c, loss) must equal the
    local (comm = NULL) call's gradients summed by attn_grad_allreduce, and the
    local outputs (dH_dec, dH_enc) must be unchanged by the communicator.
    Bitwise when the two reductions sum in the same order (always at 2 ranks);
    `max_rel` bounds the reordering otherwise."""
    import torch
    loc = st.alloc_outputs()
    st(*call_args, out=loc, comm=None, stream=stream)
    for k in ("dW_out", "dW_c", "loss"):
        binding.attn_grad_allreduce(comm, loc[k], stream=stream)
    st(*call_args, out=out, comm=comm, stream=stream)
    binding.attn_comm_poll(comm, 60000)
    barrier()
    res = {"bitwise": True, "max_rel": 0.0}
    for k in ("dW_out", "dW_c", "loss", "dH_dec", "dH_enc"):
        a, b = out[k].float(), loc[k].float()
        same = bool(torch.equal(out[k], loc[k]))
        rel = float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))
        res["bitwise"] &= same
        res["max_rel"] = max(res["max_rel"], rel)
        res[k] = "bitwise" if same else f"max_rel {rel:.2e}"
    res["verified"] = bool(res["bitwise"] or res["max_rel"] <= 1e-5)
    if not res["verified"]:
        raise SystemExit(f"bench.py: allreduced gradients disagree with attn_grad_allreduce: {res}")
    del loc
    return res


def measure_next_rows(binding, st, dv, cfg, scale, comm, stream, dev, pk, tok_local, world,
                      steps=10):
    """SURVEY §8(f) rows beyond the hot path, each timed with CUDA events on
    the launching stream (not part of `value`): NEXT-1 the stage with the
    Eq. 2 general score (W_alpha) and with the F_c bias b_out; NEXT-2 the Adam
    step over the stage's parameters (sharded reduce-scatter / update /
    all-gather when a communicator exists), HBM-bound: 30 B per parameter."""
    import numpy as np
    import torch
    from synthetic import make_weights

    def timed(fn, n=steps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(n):
            fn()
        b.record(stream)
        torch.cuda.synchronize(dev)
        return a.elapsed_time(b) / n

    res = {}
    extra = make_weights(cfg, with_alpha=True, with_bias=True)
    td = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    Wa = torch.from_numpy(extra["W_alpha"]).to(device=dev, dtype=td)
    bo = torch.from_numpy(extra["b_out"]).to(device=dev, dtype=td)
    args = (dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"],
            dv["W_c"], dv["W_out"], scale)
    outs = st.alloc_outputs(True, True)
    for name, kw in (("general_score", dict(W_alpha=Wa)), ("output_bias", dict(b_out=bo))):
        ms = timed(lambda: st(*args, out=outs, comm=comm, stream=stream, **kw))
        res[name] = {"ms_per_step": ms, "target_tokens_per_s": tok_local * world / (ms / 1e3)}
    # ablation (NOT the product path: north_star forbids round-tripping the
    # logits through HBM): the forward stores the logits as fp16 and the
    # backward reads them instead of recomputing them per V-chunk
    if cfg.dtype == "bf16" and comm is None:
        from paper_1909_00562_b200.stage import AttnSoftmaxStage
        binding.attn_softmax_set_option("store_logits", 1)
        try:
            st_sl = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype, device=dev)
            ms = timed(lambda: st_sl(*args, out=outs, stream=stream))
            res["ablation_store_logits"] = {
                "ms_per_step": ms, "target_tokens_per_s": tok_local * world / (ms / 1e3),
                "note": "ablation only: fp16 logits [T, V] stored by the forward and read by the "
                        "backward (2 T V x 2 B of HBM per step); not the product path"}
            del st_sl
        finally:
            binding.attn_softmax_set_option("store_logits", 0)
    # context rows, NOT the product path: the same stage as a
    # torch eager bf16 composition with autograd (cuBLAS / cuDNN kernels, the
    # logits materialised), and one cuBLAS GEMM at the vocabulary shape
    if cfg.dtype == "bf16" and comm is None:
        import torch.nn.functional as F
        B_, N_, M_, d_ = cfg.B, cfg.N, cfg.M, cfg.d
        srcl = torch.as_tensor(np.asarray(dv["src_len"]), device=dev)
        tgtl = torch.as_tensor(np.asarray(dv["tgt_len"]), device=dev)
        kmask = (torch.arange(M_, device=dev)[None, :] < srcl[:, None])[:, None, :]
        valid = (torch.arange(N_, device=dev)[None, :] < tgtl[:, None]).reshape(-1)
        y = dv["tgt_ids"].long().reshape(-1)

        def eager():
            H = dv["H_dec"].detach().requires_grad_()
            S = dv["H_enc"].detach().requires_grad_()
            Wc = dv["W_c"].detach().requires_grad_()
            Wo = dv["W_out"].detach().requires_grad_()
            e = torch.bmm(H, S.transpose(1, 2)).float().masked_fill(~kmask, float("-inf"))
            a = torch.softmax(e, -1).to(torch.bfloat16)
            C = torch.bmm(a, S)
            Hc = torch.tanh(torch.cat([H, C], -1) @ Wc.T).reshape(-1, d_)
            logits = Hc @ Wo.T
            loss = F.cross_entropy(logits[valid].float(), y[valid], reduction="sum") * scale
            loss.backward()
            return loss

        ms = timed(eager, n=5)
        hc = torch.randn(B_ * N_, d_, device=dev).to(torch.bfloat16)
        ms_mm = timed(lambda: hc @ dv["W_out"].T, n=5)
        res["context_torch_eager"] = {
            "ms_per_step": ms, "target_tokens_per_s": tok_local / (ms / 1e3),
            "vocab_gemm_ms": ms_mm, "vocab_gemm_tflops": 2.0 * B_ * N_ * d_ * cfg.V / (ms_mm / 1e3) / 1e12,
            "note": "context only (not the product): the stage as torch eager bf16 ops + autograd "
                    "(logits [T, V] materialised), and one cuBLAS GEMM H_c W_out^T at the vocabulary shape"}
        del hc
        torch.cuda.empty_cache()
    # NEXT-4: one beam-search decoding step, beam 5 on the config's sentences
    # (rows = B x 5 hypotheses; fused vocab GEMM + online LSE + top-k epilogue)
    if cfg.dtype == "bf16":
        from dataclasses import replace
        from paper_1909_00562_b200.stage import DecodeStep
        from synthetic import make_inputs as _mk
        dcfg = replace(cfg, N=5, lengths="full")
        dinp = _mk(dcfg, with_weights=False)
        dH = torch.from_numpy(dinp["H_dec"]).to(device=dev, dtype=td)
        dS = torch.from_numpy(dinp["H_enc"]).to(device=dev, dtype=td)
        dstep = DecodeStep(cfg.B, 5, cfg.M, cfg.d, cfg.V, 5, device=dev)
        ms = timed(lambda: dstep(dH, dS, dinp["src_len"], dv["W_c"], dv["W_out"], stream=stream))
        rows = cfg.B * 5
        res["decode_step"] = {"beam": 5, "k": 5, "hypotheses": rows, "us_per_step": ms * 1e3,
                              "hypothesis_steps_per_s": rows / (ms / 1e3),
                              "vocab_tflops": 2.0 * rows * cfg.d * cfg.V / (ms / 1e3) / 1e12}
    # NEXT-3: the encoder-decoder forward that produces H_enc / H_dec (Table 1
    # sizes: embedding 512, 4 layers, the config's hidden size and batch;
    # wavefront kernel, one per side), when the shape fits it (B <= 128)
    if cfg.dtype == "bf16" and cfg.B <= 128 and cfg.d % 64 == 0:
        from paper_1909_00562_b200.stage import EncoderDecoder
        from synthetic import make_lstm_inputs
        L_, e_ = 4, 512
        li = make_lstm_inputs(cfg, layers=L_, emb=e_)
        bfd = lambda a: torch.from_numpy(np.asarray(a, np.float32)).to(device=dev, dtype=torch.bfloat16)
        ed = EncoderDecoder(cfg.B, cfg.M, cfg.N, e_, cfg.d, L_, cfg.V, cfg.V, device=dev)
        ed.set_weights([tuple(bfd(w) for w in ws) for ws in li["enc"]],
                       [tuple(bfd(w) for w in ws) for ws in li["dec"]])
        s_ids = torch.from_numpy(li["src_ids"]).to(dev)
        t_ids = torch.from_numpy(li["tgt_ids"]).to(dev)
        Es, Et = bfd(li["E_src"]), bfd(li["E_tgt"])
        He = torch.empty(cfg.B, cfg.M, cfg.d, dtype=torch.bfloat16, device=dev)
        Hd = torch.empty(cfg.B, cfg.N, cfg.d, dtype=torch.bfloat16, device=dev)
        ms = timed(lambda: ed(s_ids, t_ids, li["src_len"], Es, Et, He, Hd, stream=stream))
        fl = sum(2.0 * cfg.B * T * 4 * cfg.d * ((e_ if l == 0 else cfg.d) + cfg.d)
                 for T in (cfg.M, cfg.N) for l in range(L_))
        res["encoder_decoder"] = {
            "layers": L_, "emb": e_, "hidden": cfg.d, "ms": ms,
            "source_plus_target_tokens_per_s": cfg.B * (cfg.M + cfg.N) / (ms / 1e3),
            "tflops": fl / (ms / 1e3) / 1e12,
            "us_per_wavefront_step": ms * 1e3 / (cfg.M + cfg.N + 2 * (L_ - 1)),
            "note": "forward only; one persistent cooperative kernel per side, SM groups in the "
                    "role of the paper's per-layer GPUs"}
        del ed
        # HybridNMTIF: the same with input feeding -- the decoder
        # steps run one after another (per step a wavefront over the layers, then
        # the fused attention step), the paper's reason to remove it
        li = make_lstm_inputs(cfg, layers=L_, emb=e_, input_feeding=True)
        ed = EncoderDecoder(cfg.B, cfg.M, cfg.N, e_, cfg.d, L_, cfg.V, cfg.V, device=dev,
                            input_feeding=True)
        ed.set_weights([tuple(bfd(w) for w in ws) for ws in li["enc"]],
                       [tuple(bfd(w) for w in ws) for ws in li["dec"]])
        Wc_if = bfd(li["W_c"])
        Ht = torch.empty(cfg.B, cfg.N, cfg.d, dtype=torch.bfloat16, device=dev)
        ms_if = timed(lambda: ed(s_ids, t_ids, li["src_len"], Es, Et, He, Hd, stream=stream,
                                 W_c=Wc_if, Htilde=Ht))
        res["encoder_decoder_input_feeding"] = {
            "ms": ms_if, "vs_no_input_feeding": ms_if / ms,
            "source_plus_target_tokens_per_s": cfg.B * (cfg.M + cfg.N) / (ms_if / 1e3),
            "note": "HybridNMTIF forward: decoder step t waits for Htilde_{t-1} (attention + Eq. 4)"}
        del ed
        # one whole HybridNMT training step on this GPU (Fig. 3): MP forward
        # keeping the activations, the DP stage (forward + backward) on its
        # H_enc / H_dec, then the MP backward (reverse wavefront + dW GEMMs)
        if comm is None:
            from paper_1909_00562_b200.stage import EncoderDecoderTrainer
            li = make_lstm_inputs(cfg, layers=L_, emb=e_)
            tr = EncoderDecoderTrainer(cfg.B, cfg.M, cfg.N, e_, cfg.d, L_, cfg.V, cfg.V, device=dev)
            tr.set_weights([tuple(bfd(w) for w in ws) for ws in li["enc"]],
                           [tuple(bfd(w) for w in ws) for ws in li["dec"]])
            hout = st.alloc_outputs()

            def hybrid():
                He_, Hd_ = tr.forward(s_ids, t_ids, li["src_len"], Es, Et, stream=stream)
                st(Hd_, He_, dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"], dv["W_out"],
                   scale, out=hout, stream=stream)
                tr.backward(hout["dH_enc"], hout["dH_dec"], stream=stream)
            ms_h = timed(hybrid)
            res["hybrid_training_step"] = {
                "ms": ms_h, "target_tokens_per_s": tok_local / (ms_h / 1e3),
                "note": "MP forward (activations kept) + DP stage + MP backward (reverse wavefront, "
                        "dW GEMMs, embedding gradients) on one GPU; no optimizer step"}
            del tr
    # NEXT-2: Adam over W_out, W_c (and W_alpha, b_out would add d^2 + V)
    n = cfg.V * cfg.d + 2 * cfg.d * cfg.d
    h = binding.adam_params(1)
    if comm is None:
        w = torch.zeros(n, device=dev)
        m, v, g = torch.zeros_like(w), torch.zeros_like(w), torch.full_like(w, 1e-3)
        wb = torch.empty(n, dtype=torch.bfloat16, device=dev)
        ms = timed(lambda: binding.attn_adam_step(h, w, m, v, g, wb, stream=stream))
        nbytes = 30.0 * n
        res["adam"] = {"params": n, "ms": ms, "sharded": False,
                       "roofline": {"bound": "hbm", "achieved": nbytes / (ms / 1e3) / 1e9,
                                    "peak": pk["hbm"], "unit": "GB/s",
                                    "frac": nbytes / (ms / 1e3) / 1e9 / pk["hbm"],
                                    "traffic": None}}
    else:
        S = binding.attn_adam_shard_len(comm, n)
        g = torch.full((S * world,), 1e-3, device=dev)
        w, m, v = (torch.zeros(S, device=dev) for _ in range(3))
        wb = torch.empty(S * world, dtype=torch.bfloat16, device=dev)
        ms = timed(lambda: binding.attn_adam_step_sharded(comm, h, n, g, w, m, v, wb,
                                                          stream=stream))
        res["adam"] = {"params": n, "ms": ms, "sharded": True, "shard": S,
                       "wire_bytes_per_param": 6}
    return res


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(args) -> int:
    """`bench.py --gpus N` without a torchrun environment: start the N
    ranks itself (one process per GPU, torchrun on 127.0.0.1) and return
    their exit code.  A box with fewer than N GPUs is an error, not a
    smaller run."""
    if args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this box has {have}",
                  file=sys.stderr, flush=True)
            return 3
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    print("bench.py: launching " + " ".join(cmd[1:]), file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(launch_ranks(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr, flush=True)
        sys.exit(2)
    from synthetic import CONFIGS
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1909_00562_b200 import binding, build
    from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
    from synthetic import global_valid_tokens, make_inputs, shard_range

    if rank == 0:
        build.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        dist.barrier()
        build.build()   # no-op unless stale; every rank loads the same .so
    lib = binding.lib()

    comm = None
    if world > 1 or args.force_comm:
        uid = [binding.attn_comm_get_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(uid, src=0)
        comm = binding.attn_comm_init(uid[0], world, rank, local)
        print(f"bench.py: attn_comm_init nranks={binding.attn_comm_nranks(comm)} rank={rank} "
              f"device={local}", file=sys.stderr, flush=True)

    # ---- inputs: this rank's sentences of the global batch (weak scaling)
    B_global = cfg.B * world
    lo, hi = shard_range(B_global, world, rank)
    inp = make_inputs(cfg, sentences=range(lo, hi))
    scale = 1.0 / global_valid_tokens(cfg, B_global)
    tok_local = int(inp["tgt_len"].sum())
    st = AttnSoftmaxStage(hi - lo, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype, device=dev)
    dv = to_device(inp, cfg.dtype, device=dev)
    out = st.alloc_outputs()
    stream = torch.cuda.current_stream(dev)
    call_args = (dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"],
                 dv["W_c"], dv["W_out"], scale)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        st(*call_args, out=out, comm=comm, stream=stream)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    launches_per_step = binding.attn_softmax_last_launches()
    verify = verify_exchange(binding, st, call_args, out, comm, stream, barrier) \
        if comm is not None else None

    # ---- device-timed region: K steps, L2 flushed between steps
    # only the events around the vocab GEMMs (the roofline's kernels): every
    # event between kernels costs a little of the programmatic-launch overlap
    binding.attn_softmax_set_option("stage_events", 2)
    clk = ClockSampler(local)
    clk.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    stage_ms = {}
    barrier()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
        for k, v in binding.attn_softmax_stage_times().items():
            stage_ms[k] = stage_ms.get(k, 0.0) + v
    barrier()
    clocks = clk.stop()
    binding.attn_softmax_set_option("stage_events", 0)
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    ntok = torch.tensor([tok_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(ntok, op=dist.ReduceOp.SUM)
    total_ms = float(t.item())
    tok_job = float(ntok.item())
    value = tok_job * args.steps / (total_ms / 1e3)
    loss = float(out["loss"].item())
    if not math.isfinite(loss):   # abort on a non-finite loss
        print(f"bench.py: non-finite loss {loss} on rank {rank}", file=sys.stderr)
        sys.exit(1)

    # ---- e2e through the C ABI with HOST buffers: every step copies its own
    # activations (H_dec, H_enc, tgt_ids) host->device from pinned memory and
    # reads its loss back; step i+1's copy is prefetched on the library's copy
    # stream while step i computes (attn_softmax_prefetch_host +
    # attn_softmax_fwd_bwd_staged, double-buffered staging).
    pin = {k: dv[k].cpu().pin_memory() for k in ("H_dec", "H_enc", "tgt_ids")}
    stg_bytes = binding.attn_softmax_host_staging_size(st.shape)
    staging = [torch.empty(stg_bytes, dtype=torch.uint8, device=dev) for _ in range(2)]
    h2d = sum(v.numel() * v.element_size() for v in pin.values())

    loss_pin = [torch.empty(1, dtype=torch.float32).pin_memory() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]

    def e2e_run(nsteps):
        # every step's loss is read on the host; step i's is read right after
        # step i+1 has been enqueued, so the host's enqueue of the next step
        # never leaves the GPU idle (one step of lag, two pinned loss slots)
        vals = []
        binding.attn_softmax_prefetch_host(st.shape, pin["H_dec"], pin["H_enc"], pin["tgt_ids"],
                                           staging[0], stream=stream)
        for i in range(nsteps):
            if i + 1 < nsteps:
                binding.attn_softmax_prefetch_host(st.shape, pin["H_dec"], pin["H_enc"],
                                                   pin["tgt_ids"], staging[(i + 1) % 2],
                                                   stream=stream)
            binding.attn_softmax_fwd_bwd_staged(
                st.shape, staging[i % 2], dv["src_len"], dv["tgt_len"], dv["W_c"], dv["W_out"],
                scale, loss_pin[i % 2], out["dH_dec"], out["dH_enc"], out["dW_c"], out["dW_out"],
                st.workspace, comm=comm, stream=stream)
            done[i % 2].record(stream)
            if i > 0:
                done[(i - 1) % 2].synchronize()
                vals.append(float(loss_pin[(i - 1) % 2].item()))
        done[(nsteps - 1) % 2].synchronize()
        vals.append(float(loss_pin[(nsteps - 1) % 2].item()))
        return vals
    e2e_run(3)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall = time.perf_counter()
    e0.record(stream)
    e2e_run(args.steps)
    e1.record(stream)
    barrier()
    t_wall = time.perf_counter() - t_wall
    # the copies run on the library's copy stream, so time on the host clock
    # around the whole loop (it brackets every copy and every compute)
    e2e_ms = torch.tensor([max(e0.elapsed_time(e1), 1e3 * t_wall)], dtype=torch.float64,
                          device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = tok_job * args.steps / (float(e2e_ms.item()) / 1e3)
    assert abs(float(loss_pin[(args.steps - 1) % 2].item()) - loss) <= 1e-6 * max(1.0, abs(loss)), \
        "e2e loss mismatch"

    # ---- roofline of the dominant kernel: the persistent vocab-backward
    # launch.  Algorithmic FLOPs per valid token: 4 d V (dW_out and dHc).
    pk = peaks()
    T_valid = tok_local
    # the dominant kernel is the persistent vocabulary launch (vocab_kernel):
    # the backward alone ("vocab_bwd": 4 d V useful FLOP per valid token,
    # + 2 d V of recomputed logits) or, option vb_fwd_fused, forward and
    # backward together ("vocab": 6 d V useful, 8 d V executed)
    fused = "vocab" in stage_ms
    vb_ms = stage_ms.get("vocab" if fused else "vocab_bwd", 0.0) / args.steps
    useful_per_tok = (6.0 if fused else 4.0) * cfg.d * cfg.V
    hw_per_tok = (8.0 if fused else 6.0) * cfg.d * cfg.V
    vb_flops = useful_per_tok * T_valid
    vf_ms = stage_ms.get("vocab_fwd", 0.0) / args.steps
    vf_flops = 2.0 * cfg.d * cfg.V * T_valid
    achieved = vb_flops / (vb_ms / 1e3) / 1e12 if vb_ms > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(cfg.name, {}).get("vocab_kernel_bytes_per_launch")
        except Exception:
            traffic = None
    # denominator: the burst peak when the timed region ran at (near) max SM
    # clock, the sustained (power-capped) peak otherwise (B200_PROFILING.md)
    at_max = (clocks.get("sm_mhz") and clocks.get("sm_max_mhz")
              and clocks["sm_mhz"] >= 0.95 * clocks["sm_max_mhz"])
    peak = pk["bf16"] if at_max else pk["bf16_sus"]
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": (achieved / peak) if achieved else None,
                "traffic": traffic,
                "kernel": ("vocab_kernel, one persistent tcgen05 launch: " +
                           ("F4 logits tiles -> online LSE, then " if fused else "") +
                           "per V-chunk the logits recomputed into bf16 dL = "
                           "rs (softmax - onehot) (the logits never stored; the dL chunk "
                           "scratch is written back to DRAM, DESIGN.md 6.1), dHc += dL W_out, "
                           "dW_out = dL^T H_c; achieved counts " +
                           ("6" if fused else "4") + " d V useful FLOP per valid token "
                           "(the recomputed logits not counted); traffic: DRAM bytes of one "
                           "launch (ncu full set, profiles/traffic.json)"),
                "executed_tflops": hw_per_tok * T_valid / (vb_ms / 1e3) / 1e12 if vb_ms > 0 else None,
                "peak_source": pk["src"] + (", burst bf16 (timed region at max SM clock)" if at_max
                                            else ", sustained bf16 (clocks below max)"),
                # context: the kernel runs power-capped (clock64 / globaltimer traces
                # put its SM clock at 1.54-1.65 GHz), i.e. nearer the
                # sustained figure than the burst one that `frac` divides by
                "frac_vs_sustained": (achieved / pk["bf16_sus"]) if achieved else None,
                "vocab_fwd": {"achieved": vf_flops / (vf_ms / 1e3) / 1e12 if vf_ms > 0 else None,
                              "peak": pk["bf16"], "unit": "TFLOP/s"},
                "stage_ms": {k: v / args.steps for k, v in stage_ms.items()}}

    next_rows = None if args.no_next else measure_next_rows(
        binding, st, dv, cfg, scale, comm, stream, dev, pk, tok_local, world)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype,
            "data": "synthetic (seeded, DESIGN.md input recipe)",
            "config": workload_desc(cfg, world),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 4},
            "roofline": roofline,
            "gpu_launches": int(launches_per_step) * args.steps,
            "clocks": clocks,
            "build": build_id(binding),
            "loss": loss,
            "comm": None if comm is None else {"nranks": binding.attn_comm_nranks(comm),
                                               "exchange_check": verify},
            "useful_tflops": tok_job * (6 * cfg.d * cfg.V + 12 * cfg.d ** 2 + 12 * cfg.M * cfg.d)
                             * args.steps / (total_ms / 1e3) / 1e12 / world}
    if next_rows is not None:
        line["next_rows"] = next_rows
    if world > 1:
        dist.barrier()
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg, fixed=args.cpu_sample_sentences)
        print(json.dumps(line), flush=True)
    if comm is not None:
        binding.attn_comm_destroy(comm)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
