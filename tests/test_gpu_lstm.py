"""NEXT-3 parity: the wavefront stacked-LSTM encoder-decoder kernels
(attn_encoder_decoder_fwd, csrc/lstm.cu) against the fp64 oracle
(oracle/lstm_oracle.py, pinned by tests/test_lstm_oracle_pins.py) on the same
seeded bf16 inputs, and the MP -> DP hidden-state scatter.

Tolerance: the kernels keep h in bf16 between steps (it is the next step's
MMA operand) and accumulate in fp32, so the states carry bf16 rounding through
every recurrence; rel-L2 <= 2e-2 per output (the bf16 gradient bar of
north_star), also per sentence and per step band so an error confined to one
layer-step or sentence cannot hide in the global norm."""
import numpy as np
import pytest
import torch

from oracle import lstm_oracle as LO
from synthetic import CONFIGS, make_lstm_inputs

pytestmark = pytest.mark.gpu

TOL = 2e-2


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _run(cfg, layers, emb):
    from paper_1909_00562_b200.stage import EncoderDecoder
    inp = make_lstm_inputs(cfg, layers=layers, emb=emb)
    dev = torch.device("cuda")
    bf = lambda a: torch.from_numpy(np.asarray(a, np.float32)).to(dev, torch.bfloat16)
    ed = EncoderDecoder(cfg.B, cfg.M, cfg.N, emb, cfg.d, layers, cfg.V, cfg.V)
    ed.set_weights([tuple(bf(w) for w in ws) for ws in inp["enc"]],
                   [tuple(bf(w) for w in ws) for ws in inp["dec"]])
    src = torch.from_numpy(inp["src_ids"]).to(dev)
    tgt = torch.from_numpy(inp["tgt_ids"]).to(dev)
    H_enc, H_dec = ed(src, tgt, inp["src_len"], bf(inp["E_src"]), bf(inp["E_tgt"]))
    torch.cuda.synchronize()
    S, H = LO.encoder_decoder(inp["src_ids"], inp["tgt_ids"], inp["src_len"], inp["E_src"],
                              inp["E_tgt"], inp["enc"], inp["dec"])
    return inp, H_enc.double().cpu().numpy(), H_dec.double().cpu().numpy(), S, H


@pytest.mark.parametrize("name,layers,emb", [("small", 2, 128), ("medium", 4, 256), ("odd", 3, 64),
                                             ("edge_min", 1, 64), ("edge_max_src", 2, 64)])
def test_encoder_decoder_matches_oracle(cuda_lib, name, layers, emb):
    cfg = CONFIGS[name]
    if cfg.B > 128:
        pytest.skip("B > 128")
    inp, ge, gd, S, H = _run(cfg, layers, emb)
    assert np.isfinite(ge).all() and np.isfinite(gd).all()
    assert _rel(ge, S) <= TOL, ("H_enc", _rel(ge, S))
    assert _rel(gd, H) <= TOL, ("H_dec", _rel(gd, H))
    for b in range(cfg.B):
        L = int(inp["src_len"][b])
        assert _rel(ge[b, :L], S[b, :L]) <= TOL, ("H_enc sentence", b)
        assert _rel(gd[b], H[b]) <= TOL, ("H_dec sentence", b)
    for t0 in range(0, cfg.N, 16):   # step bands: the recurrence does not drift
        assert _rel(gd[:, t0:t0 + 16], H[:, t0:t0 + 16]) <= TOL, ("H_dec steps", t0)


def test_encoder_decoder_paper_shape(cuda_lib):
    """Table 1 sizes (embedding 512, hidden 1024, 4 layers)
    at the C1 batch (128 sentences, 50 / 50 steps): the launch configuration
    bench.py times (4 layers x 32 CTAs)."""
    cfg = CONFIGS["paper"]
    inp, ge, gd, S, H = _run(cfg, 4, 512)
    assert _rel(ge, S) <= TOL, _rel(ge, S)
    assert _rel(gd, H) <= TOL, _rel(gd, H)
    for b in (0, 63, 127):
        assert _rel(gd[b], H[b]) <= TOL, b


def test_hidden_scatter_single_rank(cuda_lib):
    """MP -> DP hand-over on a 1-rank communicator: the shard is the whole batch."""
    from paper_1909_00562_b200 import binding
    full = torch.randn(5, 7, 64, device="cuda").to(torch.bfloat16)
    shard = torch.empty_like(full)
    uid = binding.attn_comm_get_unique_id()
    comm = binding.attn_comm_init(uid, 1, 0, torch.cuda.current_device())
    try:
        binding.attn_hidden_scatter(comm, 0, 5, 7, 64, full, shard)
        torch.cuda.synchronize()
        assert torch.equal(shard, full)
    finally:
        binding.attn_comm_destroy(comm)


def test_lstm_rejects_bad_shapes(cuda_lib):
    from paper_1909_00562_b200 import binding
    with pytest.raises(binding.AttnError):
        binding.attn_lstm_workspace_size(binding.lstm_shape(129, 5, 5, 64, 64, 1, 10, 10))
    with pytest.raises(binding.AttnError):
        binding.attn_lstm_workspace_size(binding.lstm_shape(4, 5, 5, 48, 64, 1, 10, 10))


@pytest.mark.parametrize("name,layers,emb", [("small", 2, 128), ("medium", 4, 256), ("edge_min", 1, 64),
                                             ("paper", 4, 512)])
def test_input_feeding_matches_oracle(cuda_lib, name, layers, emb):
    """HybridNMTIF: the input-feeding decoder (one wavefront
    launch per step + the fused attention step) against the fp64 oracle.

    With input feeding the decoder is a closed loop (Htilde_t enters step
    t+1), and at these sizes it amplifies perturbations by ~8% per step
    (R17): the fp64 oracle itself moves by 5% over 50 steps when its
    decoder inputs are perturbed by one bf16 unit (2^-9 relative).  So each
    step's error must stay within 2e-2 or within that measured sensitivity of
    the exact result, whichever is larger -- the encoder and the early steps
    are held to 2e-2."""
    from paper_1909_00562_b200.stage import EncoderDecoder
    cfg = CONFIGS[name]
    inp = make_lstm_inputs(cfg, layers=layers, emb=emb, input_feeding=True)
    dev = torch.device("cuda")
    bf = lambda a: torch.from_numpy(np.asarray(a, np.float32)).to(dev, torch.bfloat16)
    ed = EncoderDecoder(cfg.B, cfg.M, cfg.N, emb, cfg.d, layers, cfg.V, cfg.V, input_feeding=True)
    ed.set_weights([tuple(bf(w) for w in ws) for ws in inp["enc"]],
                   [tuple(bf(w) for w in ws) for ws in inp["dec"]])
    H_enc, H_dec, Ht = ed(torch.from_numpy(inp["src_ids"]).to(dev), torch.from_numpy(inp["tgt_ids"]).to(dev),
                          inp["src_len"], bf(inp["E_src"]), bf(inp["E_tgt"]), W_c=bf(inp["W_c"]))
    torch.cuda.synchronize()
    S, H, Htl = LO.encoder_decoder_if(inp["src_ids"], inp["tgt_ids"], inp["src_len"], inp["E_src"],
                                      inp["E_tgt"], inp["enc"], inp["dec"], inp["W_c"])
    # the problem's own sensitivity: the oracle on decoder inputs perturbed by 2^-9
    rng = np.random.default_rng(7)
    pert = lambda a: np.asarray(a, np.float64) * (1 + 2.0 ** -9 * rng.choice([-1.0, 1.0], size=np.shape(a)))
    _, H2, Ht2 = LO.encoder_decoder_if(inp["src_ids"], inp["tgt_ids"], inp["src_len"], inp["E_src"],
                                       pert(inp["E_tgt"]), inp["enc"],
                                       [tuple(pert(w) for w in ws) for ws in inp["dec"]], pert(inp["W_c"]))
    ge, gd, gt = (x.double().cpu().numpy() for x in (H_enc, H_dec, Ht))
    assert _rel(ge, S) <= TOL, ("H_enc", _rel(ge, S))
    for t in range(cfg.N):
        for got, ref, alt, nm in ((gd, H, H2, "H_dec"), (gt, Htl, Ht2, "Htilde")):
            bound = max(TOL, _rel(alt[:, t], ref[:, t]))
            assert _rel(got[:, t], ref[:, t]) <= bound, (nm, t, _rel(got[:, t], ref[:, t]), bound)


@pytest.mark.parametrize("name,layers,emb", [("small", 2, 128), ("medium", 4, 256), ("paper", 4, 512),
                                             ("odd", 3, 64), ("edge_min", 1, 64), ("edge_max_src", 2, 64)])
def test_encoder_decoder_backward_matches_oracle(cuda_lib, name, layers, emb):
    """NEXT-3 training: the reverse wavefront (attn_encoder_decoder_bwd) against
    the fp64 BPTT oracle (pinned by torch autograd) for upstream gradients of
    the stage's size on H_enc / H_dec: every layer's dW_ih, dW_hh, db and the
    embedding gradients, rel-L2 <= 2e-2 each.  The shapes cover the product's
    launch variants: K split in two with dz multicast over CTA pairs (small,
    medium, paper), K split without clusters (odd: G / 2 = 5 column groups;
    edge_min: one sentence of one step, G = 2), no K split (edge_max_src: 192
    output columns in layer 0)."""
    from paper_1909_00562_b200.stage import EncoderDecoderTrainer, unpack_lstm_grad
    cfg = CONFIGS[name]
    inp = make_lstm_inputs(cfg, layers=layers, emb=emb)
    dev = torch.device("cuda")
    bf = lambda a: torch.from_numpy(np.asarray(a, np.float32)).to(dev, torch.bfloat16)
    tr = EncoderDecoderTrainer(cfg.B, cfg.M, cfg.N, emb, cfg.d, layers, cfg.V, cfg.V)
    tr.set_weights([tuple(bf(w) for w in ws) for ws in inp["enc"]],
                   [tuple(bf(w) for w in ws) for ws in inp["dec"]])
    src = torch.from_numpy(inp["src_ids"]).to(dev)
    tgt = torch.from_numpy(inp["tgt_ids"]).to(dev)
    tr.forward(src, tgt, inp["src_len"], bf(inp["E_src"]), bf(inp["E_tgt"]))
    rng = np.random.default_rng(11)
    scale = 1.0 / (cfg.B * cfg.N)   # the stage's gradients carry the 1 / tokens loss scale
    dS = (rng.normal(size=(cfg.B, cfg.M, cfg.d)) * scale).astype(np.float32)
    dH = (rng.normal(size=(cfg.B, cfg.N, cfg.d)) * scale).astype(np.float32)
    dS_b, dH_b = bf(dS), bf(dH)
    g = tr.backward(dS_b, dH_b)
    torch.cuda.synchronize()
    ref = LO.encoder_decoder_backward(inp["src_ids"], inp["tgt_ids"], inp["src_len"], inp["E_src"],
                                      inp["E_tgt"], inp["enc"], inp["dec"],
                                      dS_b.double().cpu().numpy(), dH_b.double().cpu().numpy())
    for side in ("enc", "dec"):
        for l in range(layers):
            fin = emb if l == 0 else cfg.d
            dWi, dWh, db = unpack_lstm_grad(g[f"dW_{side}"][l], g[f"db_{side}"][l], fin, cfg.d)
            rWi, rWh, rb = ref[side][l]
            for nm, got, want in (("dW_ih", dWi, rWi), ("dW_hh", dWh, rWh), ("db", db, rb)):
                e = _rel(got.double().cpu().numpy(), want)
                assert e <= TOL, (side, l, nm, e)
    for nm in ("dE_src", "dE_tgt"):
        e = _rel(g[nm].double().cpu().numpy(), ref[nm])
        assert e <= TOL, (nm, e)
