"""One fwd+bwd of the stage per case, for compute-sanitizer (memcheck /
racecheck / synccheck): tiny (fp32 SIMT path), small and odd (bf16 tcgen05
path: persistent vocab launch on CTA pairs and on single CTAs, and with the
forward fused; small / edge_min through the fused attention kernels, odd
through the generic batched attention), edge_min; then the decoding step,
Adam and the NEXT-3 encoder-decoder wavefront; small512 (the 512-column G2 /
G3 tiles) and lstm_train (the NEXT-3 training forward and the reverse
wavefront with its K split and dz multicast) on request or by default.
Exits non-zero on a library error."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1909_00562_b200 import binding
from paper_1909_00562_b200.stage import AttnSoftmaxStage, DecodeStep, to_device
from synthetic import CONFIGS, global_valid_tokens, make_inputs

from dataclasses import replace as _replace

CONFIGS = dict(CONFIGS, small512=_replace(CONFIGS["small"], name="small512", d=512, V=3001),
               small_o2=_replace(CONFIGS["small"], name="small_o2"))
cases = [("tiny", {}), ("small", {}), ("small", {"vb_pair": 0}), ("odd", {"vb_fwd_fused": 1}),
         ("edge_min", {}), ("small", {"bias": 1}), ("small512", {}),   # small512: 512-column G2 / G3 tiles
         # the row-interleaved dispatch with T-split dW_out tiles, 3 and 1 dL buffers
         ("small_o2", {"vb_order": 2, "vocab_chunk": 512}),
         ("small_o2", {"vb_order": 2, "dl_buffers": 1, "vocab_chunk": 512})]
only = sys.argv[1:]
for name, opts in cases:
    if only and name not in only:
        continue
    cfg = CONFIGS[name]
    bias = bool(opts.pop("bias", 0))
    for k, v in opts.items():
        binding.attn_softmax_set_option(k, v)
    inp = make_inputs(cfg, with_bias=bias)
    st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
    dv = to_device(inp, cfg.dtype)
    out = st(dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"],
             dv["W_out"], 1.0 / global_valid_tokens(cfg, cfg.B), b_out=dv.get("b_out"))
    torch.cuda.synchronize()
    print(f"{name} {opts} bias={bias}: loss {out['loss'].item():.6f}", flush=True)
    for k in opts:
        binding.attn_softmax_set_option(k, {"vb_pair": 1, "vb_fwd_fused": 0, "vb_order": 1,
                                            "dl_buffers": 3, "vocab_chunk": 0}[k])
if not only:
    cfg = CONFIGS["small"]
    inp = make_inputs(cfg)
    dv = to_device(inp, cfg.dtype)
    ds = DecodeStep(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, 5)
    ids, logp, lse = ds(dv["H_dec"], dv["H_enc"], inp["src_len"], dv["W_c"], dv["W_out"])
    torch.cuda.synchronize()
    print("decode ok", float(lse.float().mean()), flush=True)
    n = 100003
    w = torch.zeros(n, device="cuda")
    m, v, g = torch.zeros_like(w), torch.zeros_like(w), torch.full_like(w, 1e-3)
    binding.attn_adam_step(binding.adam_params(1), w, m, v, g, torch.empty(n, dtype=torch.bfloat16, device="cuda"))
    torch.cuda.synchronize()
    print("adam ok", flush=True)

if not only or "lstm" in only:
    import numpy as np
    from paper_1909_00562_b200.stage import EncoderDecoder
    from synthetic import make_lstm_inputs
    cfg = CONFIGS["small"]
    li = make_lstm_inputs(cfg, layers=2, emb=128)
    bf = lambda a: torch.from_numpy(np.asarray(a, np.float32)).cuda().to(torch.bfloat16)
    ed = EncoderDecoder(cfg.B, cfg.M, cfg.N, 128, cfg.d, 2, cfg.V, cfg.V)
    ed.set_weights([tuple(bf(w) for w in ws) for ws in li["enc"]], [tuple(bf(w) for w in ws) for ws in li["dec"]])
    He, Hd = ed(torch.from_numpy(li["src_ids"]).cuda(), torch.from_numpy(li["tgt_ids"]).cuda(), li["src_len"],
                bf(li["E_src"]), bf(li["E_tgt"]))
    torch.cuda.synchronize()
    print("lstm ok", float(Hd.float().abs().mean()), flush=True)

if not only or "lstm_train" in only:
    # the reverse wavefront: K split in two with dz multicast over CTA pairs
    # (hidden 256: G = 8, two column groups of 4 per K half)
    import numpy as np
    from paper_1909_00562_b200.stage import EncoderDecoderTrainer
    from synthetic import make_lstm_inputs
    cfg = CONFIGS["small"]
    li = make_lstm_inputs(cfg, layers=2, emb=128)
    bf = lambda a: torch.from_numpy(np.asarray(a, np.float32)).cuda().to(torch.bfloat16)
    tr = EncoderDecoderTrainer(cfg.B, cfg.M, cfg.N, 128, cfg.d, 2, cfg.V, cfg.V)
    tr.set_weights([tuple(bf(w) for w in ws) for ws in li["enc"]], [tuple(bf(w) for w in ws) for ws in li["dec"]])
    He, Hd = tr.forward(torch.from_numpy(li["src_ids"]).cuda(), torch.from_numpy(li["tgt_ids"]).cuda(),
                        li["src_len"], bf(li["E_src"]), bf(li["E_tgt"]))
    g = tr.backward(torch.randn_like(He) * 1e-3, torch.randn_like(Hd) * 1e-3)
    torch.cuda.synchronize()
    print("lstm train ok", float(g["dE_src"].abs().sum()), flush=True)
