"""Per-step error of the HybridNMTIF forward against the fp64 oracle (development)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import lstm_oracle as LO
from paper_1909_00562_b200.stage import EncoderDecoder
from synthetic import CONFIGS, make_lstm_inputs
name = sys.argv[1] if len(sys.argv) > 1 else "paper"
feed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = CONFIGS[name]
L, e = (4, 512) if name == "paper" else (4, 256)
inp = make_lstm_inputs(cfg, layers=L, emb=e, input_feeding=bool(feed))
dev = torch.device("cuda")
bf = lambda a: torch.from_numpy(np.asarray(a, np.float32)).to(dev, torch.bfloat16)
ed = EncoderDecoder(cfg.B, cfg.M, cfg.N, e, cfg.d, L, cfg.V, cfg.V, input_feeding=bool(feed))
ed.set_weights([tuple(bf(w) for w in ws) for ws in inp["enc"]], [tuple(bf(w) for w in ws) for ws in inp["dec"]])
src, tgt = torch.from_numpy(inp["src_ids"]).to(dev), torch.from_numpy(inp["tgt_ids"]).to(dev)
if feed:
    He, Hd, Ht = ed(src, tgt, inp["src_len"], bf(inp["E_src"]), bf(inp["E_tgt"]), W_c=bf(inp["W_c"]))
    S, H, Htl = LO.encoder_decoder_if(inp["src_ids"], inp["tgt_ids"], inp["src_len"], inp["E_src"], inp["E_tgt"], inp["enc"], inp["dec"], inp["W_c"])
else:
    He, Hd = ed(src, tgt, inp["src_len"], bf(inp["E_src"]), bf(inp["E_tgt"]))
    S, H = LO.encoder_decoder(inp["src_ids"], inp["tgt_ids"], inp["src_len"], inp["E_src"], inp["E_tgt"], inp["enc"], inp["dec"])
torch.cuda.synchronize()
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
gd = Hd.double().cpu().numpy()
ge = He.double().cpu().numpy()
print("H_enc", rel(ge, S), "H_dec", rel(gd, H))
print("H_dec per step:", " ".join(f"{rel(gd[:, t], H[:, t]):.4f}" for t in range(0, cfg.N, 5)))
print("|H| per step:", " ".join(f"{np.abs(H[:, t]).mean():.3f}" for t in range(0, cfg.N, 5)))
if feed:
    gt = Ht.double().cpu().numpy()
    print("Htilde", rel(gt, Htl), "per step:", " ".join(f"{rel(gt[:, t], Htl[:, t]):.4f}" for t in range(0, cfg.N, 5)))
