"""Shape sweep of the fused attention kernels (csrc/attn_tc.cuh) and the split
projection backward through the whole stage, against the fp64 oracle: odd
decoder / source lengths up to the fused kernels' limit (N, M <= 128), hidden
sizes that are and are not multiples of 128 (context chunks of 64), ragged
lengths with degenerate sentences (src_len = 1, tgt_len = 0), a small
vocabulary so the oracle stays fast.  Every output and the stashed
intermediates (alpha, C, H_c) are compared; the exactness properties I1-I4
are checked on each shape."""
from dataclasses import replace

import numpy as np
import pytest

from oracle import attn_softmax_oracle as O
from synthetic import CONFIGS, global_valid_tokens, make_inputs

from test_gpu_parity import TOL, rel_l2, run_gpu

pytestmark = pytest.mark.gpu

SHAPES = [  # (B, N, M, d)
    (3, 1, 1, 64), (2, 16, 17, 128), (5, 33, 64, 192), (4, 63, 65, 320),
    (3, 64, 128, 256), (2, 127, 5, 448), (3, 128, 128, 64), (6, 50, 50, 1088),
    (1, 7, 120, 2048), (9, 100, 31, 576),
]


@pytest.mark.parametrize("B,N,M,d", SHAPES)
def test_fused_attention_shapes(cuda_lib, B, N, M, d):
    cfg = replace(CONFIGS["small"], name=f"s{B}_{N}_{M}_{d}", B=B, N=N, M=M, d=d, V=777,
                  seed=100 + B + N + M + d)
    inp = make_inputs(cfg)
    scale = 1.0 / max(1, global_valid_tokens(cfg, cfg.B))
    if global_valid_tokens(cfg, cfg.B) == 0:
        pytest.skip("no valid target tokens in this draw")
    g = run_gpu(cfg, inp, scale)
    f, b = O.fwd_bwd(inp["H_dec"], inp["H_enc"], inp["src_len"], inp["tgt_len"], inp["tgt_ids"],
                     inp["W_c"], inp["W_out"], scale)
    tol = TOL["bf16"]
    assert abs(g["loss"] - f["loss"]) <= tol["loss"] * abs(f["loss"]), (g["loss"], f["loss"])
    for k in ("dH_dec", "dH_enc", "dW_c", "dW_out"):
        if np.linalg.norm(b[k]) == 0.0:
            assert np.all(g[k] == 0.0), k
            continue
        assert rel_l2(g[k], b[k]) <= tol["grad"], (k, rel_l2(g[k], b[k]))
    assert rel_l2(g["alpha"], f["alpha"]) <= tol["inter"]
    assert rel_l2(g["C"], f["C"]) <= tol["inter"]
    assert rel_l2(g["Hc"], f["Hc"]) <= tol["inter"]
    for bb in range(cfg.B):
        L, Tb = int(inp["src_len"][bb]), int(inp["tgt_len"][bb])
        assert np.all(g["alpha"][bb, :, L:] == 0.0)
        assert np.all(g["dH_enc"][bb, L:] == 0.0)
        assert np.all(g["dH_dec"][bb, Tb:] == 0.0)
    assert np.abs(g["alpha"].sum(-1) - 1).max() < 1e-5
