"""Gradient error against the fp64 oracle with the logits stored as fp16
(store_logits = 1) and recomputed (store_logits = 0), same inputs: the
numbers behind DESIGN.md reading R15.  GPU; development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_parity import run_gpu, oracle, rel_l2, set_modes   # noqa: E402
from paper_1909_00562_b200 import binding   # noqa: E402
from synthetic import CONFIGS, make_inputs, global_valid_tokens   # noqa: E402

for name in sys.argv[1:] or ["small", "medium"]:
    cfg = CONFIGS[name]
    inp = make_inputs(cfg)
    scale = 1.0 / global_valid_tokens(cfg, cfg.B)
    f, b = oracle(inp, scale)
    for mode in ("default+sl", "default+rc"):
        set_modes(binding, mode)
        g = run_gpu(cfg, inp, scale)
        errs = {k: rel_l2(g[k], b[k]) for k in ("dH_dec", "dH_enc", "dW_c", "dW_out")}
        print(name, mode, f"loss {abs(g['loss'] - f['loss']) / abs(f['loss']):.2e}",
              " ".join(f"{k} {v:.2e}" for k, v in errs.items()), flush=True)
    set_modes(binding, "default")
