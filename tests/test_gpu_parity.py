"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on
the same seeded inputs.  Bars (BASELINE.json north_star): bf16 -- loss rel
<= 2e-3, every gradient rel-L2 <= 2e-2; fp32 -- 1e-5 and 1e-4."""
import numpy as np
import pytest
import torch

from oracle import attn_softmax_oracle as O
from synthetic import CONFIGS, make_inputs, global_valid_tokens

pytestmark = pytest.mark.gpu

TOL = {"f32": dict(loss=1e-5, grad=1e-4, inter=1e-5),
       "bf16": dict(loss=2e-3, grad=2e-2, inter=1e-2)}


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def run_gpu(cfg, inp, scale, vocab_chunk=0, comm=None):
    from paper_1909_00562_b200 import binding
    from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
    binding.attn_softmax_set_option("vocab_chunk", vocab_chunk)
    try:
        st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
        dv = to_device(inp, cfg.dtype)
        out = st(dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"],
                 dv["W_c"], dv["W_out"], scale, W_alpha=dv.get("W_alpha"), comm=comm,
                 b_out=dv.get("b_out"))
        torch.cuda.synchronize()
    finally:
        binding.attn_softmax_set_option("vocab_chunk", 0)
    res = {k: v.float().cpu().numpy() for k, v in out.items()}
    res["loss"] = float(res["loss"][0])
    views = st.views()
    for k in ("alpha", "C", "Hc", "lse", "nll"):
        res[k] = views[k].float().cpu().numpy()
    res["vocab_chunk"] = views["vocab_chunk"]
    return res


def oracle(inp, scale):
    return O.fwd_bwd(inp["H_dec"], inp["H_enc"], inp["src_len"], inp["tgt_len"],
                     inp["tgt_ids"], inp["W_c"], inp["W_out"], scale,
                     W_alpha=inp.get("W_alpha"), b_out=inp.get("b_out"))


# ------------------------------------------------------------ GEMM core ----
@pytest.mark.parametrize("wide", [0, 1])
@pytest.mark.parametrize("mn3d", [0, 1])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (296, 520, 200), (1000, 264, 1536),
                                   (320, 640, 192)])
def test_tcgen05_gemm_core(cuda_lib, a_mn, b_mn, M, N, K, mn3d, wide):
    """The tcgen05 engine alone: 128x256 tiles (two accumulators) and wide
    256x256 single-CTA tiles; all operand majors (MN-major via per-atom boxes
    or one box per stage), with M/N/K tails."""
    from paper_1909_00562_b200 import binding
    binding.attn_softmax_set_option("mn_3d_tma", mn3d)
    binding.attn_softmax_set_option("wide_tiles", 8 if wide else 0)
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, generator=g).bfloat16()
    B = torch.randn(N, K, generator=g).bfloat16()
    ref = A.double() @ B.double().T
    Ad = (A.T.contiguous() if a_mn else A).cuda()
    Bd = (B.T.contiguous() if b_mn else B).cuda()
    C = torch.full((M, N), float("nan"), device="cuda")
    binding.attn_debug_gemm_bf16(M, N, K, Ad, a_mn, Bd, b_mn, C)
    torch.cuda.synchronize()
    set_modes(binding, "default")
    binding.attn_softmax_set_option("mn_3d_tma", 1)
    err = (C.double().cpu() - ref).abs().max().item()
    assert err < 1e-3 * max(1.0, ref.abs().max().item()), err


# ------------------------------------------------------ end-to-end parity --
_DEFAULTS = {"store_logits": 0, "wide_tiles": 2, "db_gemm": -1, "vb_pair": 1, "vb_fwd_fused": 0,
             "vb_order": 1, "dl_buffers": 3, "dl_budget_mb": 200, "vb_last_g2_first": 1,
             "attn_fused": 1, "vb_wide": 1, "vb_lag": 2, "vb_g2split": 1, "vb_claim": 1,
             "vb_g1wide": 0, "gemm_claim": 4}
_MODES = {
    "default": {},                                  # persistent vocab launch on CTA pairs
    "single": {"vb_pair": 0},                       # ... on single-CTA 128 x 256 tiles
    "fused": {"vb_fwd_fused": 1},                   # F4 + F5 inside the persistent launch
    "fused_single": {"vb_fwd_fused": 1, "vb_pair": 0},
    "order0": {"vb_order": 0, "dl_buffers": 2},     # [G3, G2, G1(next)] dispatch, 2 buffers
    "nb1": {"dl_buffers": 1},                       # one dL buffer (dispatch order 0 forced)
    "g3last": {"vb_last_g2_first": 0},
    "sl": {"store_logits": 1},                      # ablation: stored fp16 logits, wide tiles
    "sl128": {"store_logits": 1, "wide_tiles": 0},  # ... on 128 x 256 tiles
    "sl2": {"store_logits": 2},                     # ... serialised dlogits kernels
    "attn_generic": {"attn_fused": 0},              # attention on the generic engine's batched GEMMs
    "narrow": {"vb_wide": 0},                       # G2 / G3 on 256-column tiles (default: 512 when d % 512 == 0)
    "order2": {"vb_order": 2},                      # row-interleaved dispatch, G2 split in two row halves
    "claim0": {"vb_claim": 0},                      # next tile claimed right after the first load
    "g1wide": {"vb_g1wide": 1},                     # 512-column G1 (dL) tiles, both accumulators
    "gclaim": {"gemm_claim": 15},                   # generic engine: late tile claim in every group
    "g1wide_o2": {"vb_g1wide": 1, "vb_order": 2},
    "order2_single": {"vb_order": 2, "vb_pair": 0},
    "order2_nosplit": {"vb_order": 2, "vb_g2split": 0},
    "order2_lag0": {"vb_order": 2, "vb_lag": 0, "dl_buffers": 2},
    "order2_lag9": {"vb_order": 2, "vb_lag": 9},
    "order2_narrow": {"vb_order": 2, "vb_wide": 0},
    "order2_fused": {"vb_order": 2, "vb_fwd_fused": 1},
    "order2_nb1": {"vb_order": 2, "dl_buffers": 1},  # one dL buffer, reused per row half
}


def set_modes(binding, mode):
    """Library options of a parity case: a _MODES key, optionally with "+cs" /
    "+ew" (stored-logits ablation with the F_c bias: db_out by column-sum
    kernels / by the dlogits kernels' own sums)."""
    mode, *flags = mode.split("+")
    opts = dict(_DEFAULTS, **_MODES[mode])
    if "cs" in flags:
        opts["db_gemm"] = 0
    if "ew" in flags:
        opts["db_gemm"] = 2
    for k, v in opts.items():
        binding.attn_softmax_set_option(k, v)


@pytest.mark.parametrize("name,vc,mode", [("tiny", 0, "default"), ("tiny_ragged", 0, "default"),
                                          ("small_f32", 0, "default"), ("small_f32", 256, "default"),
                                          ("odd_f32", 0, "default"),
                                          ("small", 0, "default"), ("small", 256, "default"),
                                          ("small", 1024, "default"), ("medium", 0, "default"),
                                          ("medium", 512, "default"), ("medium", 2048, "default"),
                                          ("odd", 0, "default"), ("odd", 256, "default"),
                                          ("edge_min", 0, "default"), ("edge_max_src", 0, "default"),
                                          ("edge_max_src", 256, "default"),
                                          ("small", 0, "single"), ("small", 256, "single"),
                                          ("medium", 512, "single"), ("odd", 256, "single"),
                                          ("edge_min", 0, "single"),
                                          ("small", 0, "fused"), ("medium", 512, "fused"),
                                          ("odd", 256, "fused"), ("edge_min", 0, "fused"),
                                          ("edge_max_src", 256, "fused"),
                                          ("small", 256, "fused_single"), ("odd", 0, "fused_single"),
                                          ("small", 256, "order0"), ("medium", 512, "order0"),
                                          ("small", 256, "nb1"), ("odd", 256, "nb1"),
                                          ("medium", 512, "g3last"),
                                          ("medium", 0, "narrow"), ("medium", 512, "narrow"),
                                          ("small", 256, "claim0"), ("medium", 512, "claim0"),
                                          ("small", 0, "gclaim"), ("medium", 512, "gclaim"),
                                          ("odd", 256, "gclaim"), ("small_f32", 0, "gclaim"),
                                          ("edge_max_src", 256, "gclaim"), ("edge_min", 0, "gclaim"),
                                          ("small", 0, "g1wide"), ("small", 256, "g1wide"),
                                          ("medium", 512, "g1wide"), ("medium", 0, "g1wide"),
                                          ("odd", 256, "g1wide"), ("edge_min", 0, "g1wide"),
                                          ("edge_max_src", 256, "g1wide"), ("medium", 512, "g1wide_o2"),
                                          ("small", 0, "order2"), ("small", 256, "order2"),
                                          ("medium", 0, "order2"), ("medium", 512, "order2"),
                                          ("odd", 256, "order2"), ("edge_min", 0, "order2"),
                                          ("edge_max_src", 256, "order2"),
                                          ("small", 256, "order2_single"), ("medium", 512, "order2_single"),
                                          ("medium", 512, "order2_nosplit"), ("medium", 512, "order2_lag0"),
                                          ("medium", 512, "order2_lag9"), ("medium", 512, "order2_narrow"),
                                          ("small", 256, "order2_fused"), ("medium", 0, "order2_fused"),
                                          ("small", 256, "order2_nb1"), ("medium", 512, "order2_nb1"),
                                          ("odd", 256, "order2_nb1"),
                                          ("tiny_ragged", 0, "sl"), ("small", 0, "sl"),
                                          ("small", 1024, "sl"), ("medium", 0, "sl"),
                                          ("medium", 2048, "sl128"), ("odd", 256, "sl"),
                                          ("edge_min", 0, "sl"), ("edge_max_src", 256, "sl128"),
                                          ("small", 0, "sl2"), ("odd", 256, "sl2"),
                                          ("small", 0, "attn_generic"), ("medium", 0, "attn_generic"),
                                          ("edge_max_src", 0, "attn_generic"),
                                          ("edge_min", 0, "attn_generic")])
def test_parity_vs_oracle(cuda_lib, name, vc, mode):
    """mode = library options (see set_modes); vc = V-chunk width (0 = auto)."""
    from paper_1909_00562_b200 import binding
    cfg = CONFIGS[name]
    inp = make_inputs(cfg)
    scale = 1.0 / global_valid_tokens(cfg, cfg.B)
    set_modes(binding, mode)
    try:
        g = run_gpu(cfg, inp, scale, vocab_chunk=vc)
    finally:
        set_modes(binding, "default")
    f, b = oracle(inp, scale)
    tol = TOL[cfg.dtype]
    assert abs(g["loss"] - f["loss"]) <= tol["loss"] * abs(f["loss"]), (g["loss"], f["loss"])
    for k in ("dH_dec", "dH_enc", "dW_c", "dW_out"):
        e = rel_l2(g[k], b[k])
        assert e <= tol["grad"], (k, e)
    # stage by stage (intermediates stashed in the workspace)
    assert rel_l2(g["alpha"], f["alpha"]) <= tol["inter"]
    assert rel_l2(g["C"], f["C"]) <= tol["inter"]
    assert rel_l2(g["Hc"], f["Hc"]) <= tol["inter"]
    lse_tol = 1e-4 if cfg.dtype == "f32" else 2e-2
    assert np.max(np.abs(g["lse"] - f["lse"])) <= lse_tol
    # exactness properties (I2, I3, I4)
    for bb in range(cfg.B):
        L, Tb = int(inp["src_len"][bb]), int(inp["tgt_len"][bb])
        assert np.all(g["alpha"][bb, :, L:] == 0.0)
        assert np.all(g["dH_enc"][bb, L:] == 0.0)
        assert np.all(g["dH_dec"][bb, Tb:] == 0.0)
        assert np.all(g["nll"][bb * cfg.N + Tb:(bb + 1) * cfg.N] == 0.0)
    # I1 rows sum to 1
    assert np.abs(g["alpha"].sum(-1) - 1).max() < 1e-5


@pytest.mark.parametrize("name,vc,mode", [("tiny_ragged", 0, "default"), ("small_f32", 0, "default"),
                                          ("odd_f32", 0, "default"), ("small", 0, "default"),
                                          ("small", 1024, "single"), ("medium", 0, "default"),
                                          ("medium", 512, "fused"), ("odd", 256, "default"),
                                          ("odd", 256, "sl"), ("small", 0, "attn_generic"),
                                          ("medium", 0, "attn_generic")])
def test_parity_general_score(cuda_lib, name, vc, mode):
    """NEXT-1: the Eq. 2 "general" score alpha_hat = H^T W_alpha S
     -- Q = H W_alpha on the tensor cores, dW_alpha = H^T dQ,
    dH_dec = dH_part + dQ W_alpha^T -- against the oracle's W_alpha branch."""
    from paper_1909_00562_b200 import binding
    cfg = CONFIGS[name]
    inp = make_inputs(cfg, with_alpha=True)
    scale = 1.0 / global_valid_tokens(cfg, cfg.B)
    set_modes(binding, mode)
    try:
        g = run_gpu(cfg, inp, scale, vocab_chunk=vc)
    finally:
        set_modes(binding, "default")
    f, b = oracle(inp, scale)
    tol = TOL[cfg.dtype]
    assert abs(g["loss"] - f["loss"]) <= tol["loss"] * abs(f["loss"]), (g["loss"], f["loss"])
    for k in ("dH_dec", "dH_enc", "dW_c", "dW_out", "dW_alpha"):
        e = rel_l2(g[k], b[k])
        assert e <= tol["grad"], (k, e)
    assert rel_l2(g["alpha"], f["alpha"]) <= tol["inter"]
    for bb in range(cfg.B):
        L, Tb = int(inp["src_len"][bb]), int(inp["tgt_len"][bb])
        assert np.all(g["alpha"][bb, :, L:] == 0.0)
        assert np.all(g["dH_enc"][bb, L:] == 0.0)
        assert np.all(g["dH_dec"][bb, Tb:] == 0.0)


@pytest.mark.parametrize("name,vc,mode,alpha", [("tiny_ragged", 0, "default", False),
                                                ("small_f32", 256, "default", True),
                                                ("odd_f32", 0, "default", False),
                                                ("small", 0, "default", False),
                                                ("small", 256, "default", True),
                                                ("medium", 0, "default", False),
                                                ("medium", 512, "single", True),
                                                ("odd", 256, "default", False),
                                                ("odd", 0, "fused", True),
                                                ("edge_min", 0, "default", False),
                                                ("small", 0, "sl", True),
                                                ("odd", 256, "sl+cs", False),
                                                ("medium", 0, "sl+cs", True),
                                                ("odd", 0, "sl2", False),
                                                ("tiny_ragged", 0, "sl+ew", False),
                                                ("medium", 2048, "sl+ew", True)])
def test_parity_output_bias(cuda_lib, name, vc, mode, alpha):
    """NEXT-1: the F_c bias b_out of Eq. 5 -- added in the
    forward LSE and the backward dlogits epilogues, db_out = column sums of
    dL (the persistent launch's per-32-row warp sums, added in order; the
    stored-logits ablation's kernels) -- against the oracle (with and without
    W_alpha)."""
    from paper_1909_00562_b200 import binding
    cfg = CONFIGS[name]
    inp = make_inputs(cfg, with_alpha=alpha, with_bias=True)
    scale = 1.0 / global_valid_tokens(cfg, cfg.B)
    set_modes(binding, mode)
    try:
        g = run_gpu(cfg, inp, scale, vocab_chunk=vc)
    finally:
        set_modes(binding, "default")
    f, b = oracle(inp, scale)
    tol = TOL[cfg.dtype]
    assert abs(g["loss"] - f["loss"]) <= tol["loss"] * abs(f["loss"]), (g["loss"], f["loss"])
    keys = ["dH_dec", "dH_enc", "dW_c", "dW_out", "db_out"] + (["dW_alpha"] if alpha else [])
    for k in keys:
        e = rel_l2(g[k], b[k])
        assert e <= tol["grad"], (k, e)
    lse_tol = 1e-4 if cfg.dtype == "f32" else 2e-2
    assert np.max(np.abs(g["lse"] - f["lse"])) <= lse_tol
    for bb in range(cfg.B):
        Tb = int(inp["tgt_len"][bb])
        assert np.all(g["dH_dec"][bb, Tb:] == 0.0)


@pytest.mark.parametrize("name", ["tiny_ragged", "small"])
def test_padding_garbage_is_bitwise_inert(cuda_lib, name):
    """I5: finite garbage in padded slots changes no GPU output bit."""
    cfg = CONFIGS[name]
    inp = make_inputs(cfg)
    alt = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in inp.items()}
    rng = np.random.default_rng(5)
    for b in range(cfg.B):
        L, Tb = int(inp["src_len"][b]), int(inp["tgt_len"][b])
        alt["H_enc"][b, L:] = np.float32(rng.uniform(-3, 3))
        alt["H_dec"][b, Tb:] = np.float32(rng.uniform(-3, 3))
        alt["tgt_ids"][b, Tb:] = rng.integers(-5000, 5000)
    scale = 1.0 / global_valid_tokens(cfg, cfg.B)
    g0 = run_gpu(cfg, inp, scale)
    g1 = run_gpu(cfg, alt, scale)
    assert g0["loss"] == g1["loss"]
    for k in ("dW_c", "dW_out"):
        np.testing.assert_array_equal(g0[k], g1[k])
    for b in range(cfg.B):
        np.testing.assert_array_equal(g0["dH_dec"][b], g1["dH_dec"][b])
        np.testing.assert_array_equal(g0["dH_enc"][b], g1["dH_enc"][b])


def test_dw_out_column_sums_vanish(cuda_lib):
    """I6 on the GPU result: sum_v dW_out[v,:] = 0 (each dlogits row sums to 0)."""
    cfg = CONFIGS["medium"]
    inp = make_inputs(cfg)
    g = run_gpu(cfg, inp, 1.0 / global_valid_tokens(cfg, cfg.B))
    col = g["dW_out"].astype(np.float64).sum(0)
    scale = np.abs(g["dW_out"]).sum(0).max()
    assert np.abs(col).max() < 2e-2 * scale


def test_deterministic(cuda_lib):
    cfg = CONFIGS["small"]
    inp = make_inputs(cfg)
    s = 1.0 / global_valid_tokens(cfg, cfg.B)
    a, b = run_gpu(cfg, inp, s), run_gpu(cfg, inp, s)
    assert a["loss"] == b["loss"]
    for k in ("dH_dec", "dH_enc", "dW_c", "dW_out"):
        np.testing.assert_array_equal(a[k], b[k])


def test_host_buffer_paths_match_device_path(cuda_lib):
    """attn_softmax_fwd_bwd_host and the pipelined prefetch + staged entry
    points give bit-identical results to the device-pointer call."""
    from paper_1909_00562_b200 import binding
    from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
    cfg = CONFIGS["small"]
    inp = make_inputs(cfg)
    scale = 1.0 / global_valid_tokens(cfg, cfg.B)
    st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
    dv = to_device(inp, cfg.dtype)
    ref = st(dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"],
             dv["W_c"], dv["W_out"], scale)
    ref = {k: v.clone() for k, v in ref.items()}
    pin = {k: dv[k].cpu().pin_memory() for k in ("H_dec", "H_enc", "tgt_ids")}
    nbytes = binding.attn_softmax_host_staging_size(st.shape)
    staging = [torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
    loss_host = torch.empty(1).pin_memory()
    out = st.alloc_outputs()
    binding.attn_softmax_fwd_bwd_host(st.shape, pin["H_dec"], pin["H_enc"], dv["src_len"],
                                      dv["tgt_len"], pin["tgt_ids"], dv["W_c"], dv["W_out"], scale,
                                      loss_host, out["dH_dec"], out["dH_enc"], out["dW_c"],
                                      out["dW_out"], staging[0], st.workspace)
    torch.cuda.synchronize()
    assert loss_host.item() == ref["loss"].item()
    for k in ("dH_dec", "dH_enc", "dW_c", "dW_out"):
        assert torch.equal(out[k], ref[k]), k
    for i in range(3):   # pipelined: prefetch step i+1 while step i runs
        if i == 0:
            binding.attn_softmax_prefetch_host(st.shape, pin["H_dec"], pin["H_enc"],
                                               pin["tgt_ids"], staging[0])
        binding.attn_softmax_prefetch_host(st.shape, pin["H_dec"], pin["H_enc"], pin["tgt_ids"],
                                           staging[(i + 1) % 2])
        out = st.alloc_outputs()
        binding.attn_softmax_fwd_bwd_staged(st.shape, staging[i % 2], dv["src_len"],
                                            dv["tgt_len"], dv["W_c"], dv["W_out"], scale,
                                            loss_host, out["dH_dec"], out["dH_enc"],
                                            out["dW_c"], out["dW_out"], st.workspace)
        torch.cuda.synchronize()
        assert loss_host.item() == ref["loss"].item()
        for k in ("dH_dec", "dH_enc", "dW_c", "dW_out"):
            assert torch.equal(out[k], ref[k]), k


@pytest.mark.parametrize("name,reserve", [("small", 0), ("small", 1), ("medium", 1)])
def test_single_rank_nccl_communicator(cuda_lib, name, reserve):
    """The NCCL path of attn_softmax_fwd_bwd (dlopen'ed libnccl, comm stream,
    per-chunk dW_out allreduce, dW_c and loss allreduce, join) on a 1-rank
    communicator: the sum over one rank is the identity, so results must be
    bitwise equal to the local call.  attn_grad_allreduce is checked too.
    reserve = 1 leaves the communicator's SMs free as with several ranks (the
    persistent launches on a reduced grid: fixed summation orders, so still
    bitwise)."""
    from paper_1909_00562_b200 import binding
    from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
    binding.attn_softmax_set_option("comm_reserve_1rank", reserve)
    cfg = CONFIGS[name]
    inp = make_inputs(cfg)
    scale = 1.0 / global_valid_tokens(cfg, cfg.B)
    st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
    dv = to_device(inp, cfg.dtype)
    args = (dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"],
            dv["W_c"], dv["W_out"], scale)
    ref = {k: v.clone() for k, v in st(*args).items()}
    uid = binding.attn_comm_get_unique_id()
    comm = binding.attn_comm_init(uid, 1, 0, torch.cuda.current_device())
    try:
        out = st(*args, comm=comm)
        torch.cuda.synchronize()
        for k in ("loss", "dH_dec", "dH_enc", "dW_c", "dW_out"):
            assert torch.equal(out[k], ref[k]), k
        # general score (NEXT-1): dW_alpha joins the allreduce
        inp_a = make_inputs(cfg, with_alpha=True)
        Wa = to_device(inp_a, cfg.dtype)["W_alpha"]
        ref_a = {k: v.clone() for k, v in st(*args, W_alpha=Wa).items()}
        out_a = st(*args, W_alpha=Wa, comm=comm)
        torch.cuda.synchronize()
        for k in ("loss", "dH_dec", "dH_enc", "dW_c", "dW_out", "dW_alpha"):
            assert torch.equal(out_a[k], ref_a[k]), k
        # F_c bias (NEXT-1): db_out joins the allreduce
        bo = to_device(make_inputs(cfg, with_bias=True), cfg.dtype)["b_out"]
        ref_b = {k: v.clone() for k, v in st(*args, b_out=bo).items()}
        out_b = st(*args, b_out=bo, comm=comm)
        torch.cuda.synchronize()
        for k in ("loss", "dH_dec", "dH_enc", "dW_c", "dW_out", "db_out"):
            assert torch.equal(out_b[k], ref_b[k]), k
        buf = torch.arange(1000, dtype=torch.float32, device="cuda")
        binding.attn_grad_allreduce(comm, buf)
        torch.cuda.synchronize()
        assert torch.equal(buf, torch.arange(1000, dtype=torch.float32, device="cuda"))
    finally:
        binding.attn_comm_destroy(comm)
        binding.attn_softmax_set_option("comm_reserve_1rank", 0)


@pytest.mark.gpu
def test_nonfinite_loss_aborts(cuda_lib):
    """a non-finite loss is reported (check_finite), a finite one passes."""
    from paper_1909_00562_b200.stage import AttnSoftmaxStage, NonFiniteLoss, to_device
    cfg = CONFIGS["small"]
    inp = make_inputs(cfg)
    scale = 1.0 / global_valid_tokens(cfg, cfg.B)
    st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
    dv = to_device(inp, cfg.dtype)
    args = (dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"])
    st(*args, dv["W_out"], scale, check_finite=True)
    bad = dv["W_out"].clone()
    bad[int(inp["tgt_ids"][0, 0])] = float("nan")
    with pytest.raises(NonFiniteLoss):
        st(*args, bad, scale, check_finite=True)
