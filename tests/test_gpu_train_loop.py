"""The stage and the optimizer composed as a training loop (NEXT-2 wired to
the hot path): a few Adam steps on W_c and W_out driven by the GPU stage's
gradients track the same loop driven by the fp64 oracle (stage + Adam), and
the loss goes down.  fp32 path (tight tolerances) and bf16 path."""
import numpy as np
import pytest
import torch

from oracle import attn_softmax_oracle as O
from oracle.adam_oracle import adam_step
from synthetic import CONFIGS, make_inputs, global_valid_tokens, round_bf16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,tol", [("small_f32", 1e-4), ("small", 3e-2)])
def test_adam_training_loop_tracks_oracle(cuda_lib, name, tol):
    from paper_1909_00562_b200 import binding
    from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
    cfg = CONFIGS[name]
    inp = make_inputs(cfg)
    scale = 1.0 / global_valid_tokens(cfg, cfg.B)
    lr = 1e-2
    st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
    dv = to_device(inp, cfg.dtype)
    td = dv["W_c"].dtype
    # fp32 masters + moments on the device, the stage reads their dtype copies
    masters = {k: torch.tensor(inp[k], device="cuda", dtype=torch.float32).reshape(-1)
               for k in ("W_c", "W_out")}
    mom = {k: (torch.zeros_like(v), torch.zeros_like(v)) for k, v in masters.items()}
    work = {k: v.to(td).clone() for k, v in masters.items()}
    # oracle loop state (fp64)
    ow = {k: inp[k].astype(np.float64) for k in ("W_c", "W_out")}
    om = {k: (np.zeros(v.size), np.zeros(v.size)) for k, v in ow.items()}
    losses, olosses = [], []
    for t in range(1, 5):
        out = st(dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"],
                 work["W_c"].view(cfg.d, 2 * cfg.d), work["W_out"].view(cfg.V, cfg.d), scale)
        for k, gk in (("W_c", "dW_c"), ("W_out", "dW_out")):
            wb = torch.empty_like(masters[k], dtype=torch.bfloat16) if cfg.dtype == "bf16" else None
            binding.attn_adam_step(binding.adam_params(t, lr=lr), masters[k], mom[k][0], mom[k][1],
                                   out[gk].reshape(-1), wb)
            work[k] = wb if wb is not None else masters[k].clone()
        torch.cuda.synchronize()
        losses.append(float(out["loss"].item()))
        # oracle: the stage on the same (dtype-rounded) weights, then Adam in fp64
        wc = ow["W_c"] if cfg.dtype == "f32" else round_bf16(ow["W_c"].astype(np.float32))
        wo = ow["W_out"] if cfg.dtype == "f32" else round_bf16(ow["W_out"].astype(np.float32))
        f, g = O.fwd_bwd(inp["H_dec"], inp["H_enc"], inp["src_len"], inp["tgt_len"],
                         inp["tgt_ids"], wc, wo, scale)
        olosses.append(f["loss"])
        for k, gk in (("W_c", "dW_c"), ("W_out", "dW_out")):
            w, m, v = adam_step(ow[k].reshape(-1), om[k][0], om[k][1], g[gk].reshape(-1), t,
                                lr=lr)
            ow[k] = w.reshape(ow[k].shape)
            om[k] = (m, v)
    assert losses[-1] < losses[0], losses
    np.testing.assert_allclose(losses, olosses, rtol=tol)
    for k in ("W_c", "W_out"):
        w = masters[k].cpu().numpy().astype(np.float64)
        d0 = ow[k].reshape(-1) - inp[k].reshape(-1)       # the oracle's total update
        assert np.linalg.norm(w - ow[k].reshape(-1)) <= 5 * tol * np.linalg.norm(d0), k
