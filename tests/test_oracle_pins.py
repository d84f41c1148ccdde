"""Pins for the fp64 oracle against things other than itself (CPU only).

* E1-E5: worked examples / closed forms (SPEC.md examples).
* I1-I8: invariants of the method.
* central finite differences of the oracle's own forward (pins the backward).
* an independent torch float64 composition + autograd (pins both passes).
* library special cases: scaled_dot_product_attention (F1+F2) and
  cross_entropy (F4).
Each of these fails on a dropped term, a wrong sign or index, or a
transposed / swapped operand in the oracle.
"""
import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import attn_softmax_oracle as O
from synthetic import CONFIGS, make_inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _run(inp, scale=None, W_alpha=None):
    if scale is None:
        scale = 1.0 / max(1, int(np.sum(inp["tgt_len"])))
    return O.fwd_bwd(inp["H_dec"], inp["H_enc"], inp["src_len"],
                     inp["tgt_len"], inp["tgt_ids"], inp["W_c"], inp["W_out"],
                     scale, W_alpha=W_alpha)


def _e1_inputs():
    return dict(H_dec=np.array([[[1.0]]]),
                H_enc=np.array([[[math.log(2.0)], [0.0]]]),
                src_len=np.array([2]), tgt_len=np.array([1]),
                tgt_ids=np.array([[0]]),
                W_c=np.array([[0.5, 1.0]]),
                W_out=np.array([[1.0], [-1.0]]))


# ---------------------------------------------------------------- E1 ----
def test_e1_golden():
    """Worked example E1 (tests/golden/e1_worked_example.json)."""
    g = json.load(open(os.path.join(GOLDEN, "e1_worked_example.json")))
    ex, tol = g["expected"], g["abs_tol"]
    fwd, bwd = _run(_e1_inputs(), scale=1.0)
    np.testing.assert_allclose(fwd["alpha"][0, 0], ex["alpha"], atol=tol)
    assert abs(fwd["C"][0, 0, 0] - ex["C"]) < tol
    assert abs(fwd["z"][0, 0, 0] - ex["z"]) < tol
    assert abs(fwd["Hc"][0, 0, 0] - ex["Hc"]) < tol
    assert abs(fwd["loss"] - ex["loss"]) < tol
    np.testing.assert_allclose(bwd["dW_out"][:, 0], ex["dW_out"], atol=tol)
    np.testing.assert_allclose(bwd["dW_c"][0], ex["dW_c"], atol=tol)
    assert abs(bwd["dH_dec"][0, 0, 0] - ex["dH_dec"]) < tol
    np.testing.assert_allclose(bwd["dH_enc"][0, :, 0], ex["dH_enc"], atol=tol)


def test_e1_closed_form():
    """E1 from the scalar closed forms (math module only):
    loss = softplus((u1-u0) t); dH_dec = dz a + dC Var_alpha(S);
    dH_enc_j = alpha_j dC (1 + h (S_j - C))."""
    h, S, a, c, u0, u1 = 1.0, [math.log(2.0), 0.0], 0.5, 1.0, 1.0, -1.0
    al = [2.0 / 3.0, 1.0 / 3.0]
    C = al[0] * S[0] + al[1] * S[1]
    t = math.tanh(a * h + c * C)
    loss = math.log1p(math.exp((u1 - u0) * t))
    p1 = 1.0 / (1.0 + math.exp(-(u1 - u0) * t))
    dz = p1 * (u1 - u0) * (1 - t * t)
    dC = c * dz
    var = al[0] * S[0] ** 2 + al[1] * S[1] ** 2 - C * C
    fwd, bwd = _run(_e1_inputs(), scale=1.0)
    assert abs(fwd["loss"] - loss) < 1e-14
    np.testing.assert_allclose(bwd["dW_out"][:, 0], [-p1 * t, p1 * t], atol=1e-14)
    np.testing.assert_allclose(bwd["dW_c"][0], [dz * h, dz * C], atol=1e-14)
    assert abs(bwd["dH_dec"][0, 0, 0] - (dz * a + dC * var)) < 1e-14
    np.testing.assert_allclose(
        bwd["dH_enc"][0, :, 0],
        [al[j] * dC * (1 + h * (S[j] - C)) for j in range(2)], atol=1e-14)


# ---------------------------------------------------------------- E2 ----
def test_e2_masked_position_is_inert():
    """E2: E1 plus a padded third source position (S_3 = 123) gives the same
    loss and gradients, and exactly 0 for the padded dH_enc row and alpha."""
    base = _e1_inputs()
    ext = dict(base)
    ext["H_enc"] = np.array([[[math.log(2.0)], [0.0], [123.0]]])
    f0, b0 = _run(base, scale=1.0)
    f1, b1 = _run(ext, scale=1.0)
    assert f1["alpha"][0, 0, 2] == 0.0
    assert b1["dH_enc"][0, 2, 0] == 0.0
    assert f1["loss"] == f0["loss"]
    for k in ("dW_out", "dW_c", "dH_dec"):
        np.testing.assert_array_equal(b1[k], b0[k])
    np.testing.assert_array_equal(b1["dH_enc"][:, :2], b0["dH_enc"])


# ---------------------------------------------------------------- E3 ----
def test_e3_zero_wc():
    """E3: W_c = 0 -> H_c = 0 -> logits 0 -> per-token loss ln V exactly;
    dW_out = 0, dH = 0 and dz_i = scale (mean_v W_out[v] - W_out[y_i])."""
    cfg = CONFIGS["small_f32"]
    inp = make_inputs(cfg)
    inp["W_c"] = np.zeros_like(inp["W_c"])
    T_valid = int(inp["tgt_len"].sum())
    scale = 0.37
    fwd, bwd = _run(inp, scale=scale)
    assert abs(fwd["loss"] - scale * T_valid * math.log(cfg.V)) < 1e-10
    assert np.all(bwd["dW_out"] == 0.0)
    assert np.all(bwd["dH_dec"] == 0.0) and np.all(bwd["dH_enc"] == 0.0)
    W_out = inp["W_out"].astype(np.float64)
    mean_w = W_out.mean(axis=0)
    d = cfg.d
    dWc = np.zeros((d, 2 * d))
    for b in range(cfg.B):
        for i in range(int(inp["tgt_len"][b])):
            dz = scale * (mean_w - W_out[inp["tgt_ids"][b, i]])
            hc = np.concatenate([inp["H_dec"][b, i], fwd["C"][b, i]])
            dWc += np.outer(dz, hc)
    np.testing.assert_allclose(bwd["dW_c"], dWc, rtol=1e-10, atol=1e-14)


# ---------------------------------------------------------------- E4 ----
def test_e4_single_source_position():
    """E4: src_len = 1 -> alpha = 1 on j=0, C = S_0, de = 0."""
    cfg = CONFIGS["small_f32"]
    inp = make_inputs(cfg)
    inp["src_len"] = np.ones(cfg.B, np.int32)
    fwd, bwd = _run(inp)
    assert np.all(fwd["alpha"][:, :, 0] == 1.0)
    assert np.all(fwd["alpha"][:, :, 1:] == 0.0)
    np.testing.assert_array_equal(
        fwd["C"], np.broadcast_to(inp["H_enc"][:, :1, :].astype(np.float64),
                                  fwd["C"].shape))
    assert np.all(bwd["de"] == 0.0)


def test_e4_zero_query_gives_uniform_attention():
    """E4: H_dec = 0 -> alpha uniform 1/src_len, C = mean of unmasked rows
    (SPEC.md:216, :225)."""
    cfg = CONFIGS["small_f32"]
    inp = make_inputs(cfg)
    inp["H_dec"] = np.zeros_like(inp["H_dec"])
    fwd, _ = _run(inp)
    for b in range(cfg.B):
        L = int(inp["src_len"][b])
        np.testing.assert_allclose(fwd["alpha"][b, :, :L], 1.0 / L, rtol=1e-15)
        mean = inp["H_enc"][b, :L].astype(np.float64).mean(axis=0)
        np.testing.assert_allclose(fwd["C"][b], np.broadcast_to(mean, fwd["C"][b].shape),
                                   rtol=1e-12, atol=1e-15)


def test_e4_softmax_no_overflow():
    """softmax([1000, 0]) = [1, 0]; softmax([ln2, 0]) = [2/3, 1/3]
    (SPEC.md:55); softmax([0, 0]) = [.5, .5]."""
    e = np.array([[[1000.0, 0.0], [math.log(2.0), 0.0], [0.0, 0.0]]])
    a = O.attention_weights(e, [2])
    np.testing.assert_allclose(a[0, 0], [1.0, 0.0], atol=1e-300)
    np.testing.assert_allclose(a[0, 1], [2 / 3, 1 / 3], rtol=1e-15)
    np.testing.assert_allclose(a[0, 2], [0.5, 0.5], rtol=1e-15)
    assert np.all(np.isfinite(a))


def test_attention_rejects_empty_source():
    with pytest.raises(ValueError):
        O.attention_weights(np.zeros((1, 2, 3)), [0])


# ---------------------------------------------------------------- E5 ----
def test_e5_one_hot_target_gives_zero_loss():
    """E5: when P(y) -> 1 the loss -> 0.  One valid row whose
    target row of W_out is 100 sign(h_c) and every other row 0: the target
    logit is m = 100 sum|h_c| and the rest 0, so the loss is the closed form
    log(1 + (V-1) e^{-m})."""
    cfg = CONFIGS["tiny"]
    inp = make_inputs(cfg)
    inp["tgt_len"] = np.array([1, 0], np.int32)
    fwd0, _ = _run(inp, scale=1.0)
    hc = fwd0["Hc"][0, 0]
    y = int(inp["tgt_ids"][0, 0])
    W = np.zeros((cfg.V, cfg.d), np.float64)
    W[y] = 100.0 * np.sign(hc)
    inp["W_out"] = W
    fwd, bwd = _run(inp, scale=1.0)
    m = 100.0 * np.abs(hc).sum()
    assert m > 40
    closed = math.log1p((cfg.V - 1) * math.exp(-m))
    # lse = m + log1p(..) rounds to m in fp64, so compare absolutely
    assert 0.0 <= fwd["loss"] < 1e-14
    assert abs(fwd["loss"] - closed) < 1e-14
    assert np.abs(bwd["dlogits"]).max() < 1e-15


# ------------------------------------------------------------ invariants --
@pytest.mark.parametrize("name", ["tiny_ragged", "small_f32"])
def test_invariants_i1_to_i6(name):
    cfg = CONFIGS[name]
    inp = make_inputs(cfg)
    fwd, bwd = _run(inp)
    for b in range(cfg.B):
        L, Tb = int(inp["src_len"][b]), int(inp["tgt_len"][b])
        # I1 rows sum to 1; I2 masked alpha exactly 0
        np.testing.assert_allclose(fwd["alpha"][b].sum(axis=1), 1.0, atol=1e-12)
        assert np.all(fwd["alpha"][b, :, L:] == 0.0)
        # I3 dH_enc rows j >= src_len exactly 0; I4 dH_dec rows i >= tgt_len 0
        assert np.all(bwd["dH_enc"][b, L:] == 0.0)
        assert np.all(bwd["dH_dec"][b, Tb:] == 0.0)
    # I6: each dlogits row sums to 0 -> column sums of dW_out vanish
    assert np.abs(bwd["dlogits"].sum(axis=1)).max() < 1e-15
    colsum = bwd["dW_out"].sum(axis=0)
    assert np.abs(colsum).max() < 1e-13 * max(1.0, np.abs(bwd["dW_out"]).max())


@pytest.mark.parametrize("name", ["tiny_ragged", "small_f32"])
def test_i5_padding_contents_do_not_matter(name):
    """I5: finite garbage in padded slots changes no output (bitwise)."""
    cfg = CONFIGS[name]
    inp = make_inputs(cfg)
    alt = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in inp.items()}
    rng = np.random.default_rng(99)
    for b in range(cfg.B):
        L, Tb = int(inp["src_len"][b]), int(inp["tgt_len"][b])
        alt["H_enc"][b, L:] = rng.uniform(-50, 50, alt["H_enc"][b, L:].shape)
        alt["H_dec"][b, Tb:] = rng.uniform(-50, 50, alt["H_dec"][b, Tb:].shape)
        alt["tgt_ids"][b, Tb:] = rng.integers(-1000, 1000, cfg.N - Tb)
    f0, b0 = _run(inp)
    f1, b1 = _run(alt)
    assert f0["loss"] == f1["loss"]
    for k in ("dW_c", "dW_out"):
        np.testing.assert_array_equal(b0[k], b1[k])
    for b in range(cfg.B):
        L, Tb = int(inp["src_len"][b]), int(inp["tgt_len"][b])
        np.testing.assert_array_equal(b0["dH_dec"][b], b1["dH_dec"][b])
        np.testing.assert_array_equal(b0["dH_enc"][b], b1["dH_enc"][b])


def test_i7_dp_additivity():
    """I7: shard losses / weight gradients at a
    common (global) scale sum to the full-batch values."""
    cfg = CONFIGS["small_f32"]
    inp = make_inputs(cfg)
    scale = 1.0 / int(inp["tgt_len"].sum())
    f, b = _run(inp, scale=scale)
    loss, dWc, dWo = 0.0, 0.0, 0.0
    for lo, hi in [(0, 2), (2, 3), (3, 5)]:
        part = {k: (v[lo:hi] if k in ("H_dec", "H_enc", "src_len", "tgt_len",
                                      "tgt_ids") else v) for k, v in inp.items()}
        fp, bp = _run(part, scale=scale)
        loss += fp["loss"]
        dWc = dWc + bp["dW_c"]
        dWo = dWo + bp["dW_out"]
        np.testing.assert_allclose(bp["dH_dec"], b["dH_dec"][lo:hi], rtol=1e-12, atol=1e-18)
    assert abs(loss - f["loss"]) < 1e-12 * abs(f["loss"])
    np.testing.assert_allclose(dWc, b["dW_c"], rtol=1e-10, atol=1e-16)
    np.testing.assert_allclose(dWo, b["dW_out"], rtol=1e-10, atol=1e-16)


def test_i8_sentence_permutation():
    """I8: permuting sentences permutes dH and leaves loss and dW unchanged."""
    cfg = CONFIGS["small_f32"]
    inp = make_inputs(cfg)
    perm = np.array([3, 0, 4, 1, 2])
    p = {k: (v[perm] if k in ("H_dec", "H_enc", "src_len", "tgt_len", "tgt_ids")
             else v) for k, v in inp.items()}
    f0, b0 = _run(inp)
    f1, b1 = _run(p)
    assert abs(f0["loss"] - f1["loss"]) < 1e-12 * abs(f0["loss"])
    np.testing.assert_allclose(b1["dW_out"], b0["dW_out"], rtol=1e-9, atol=1e-16)
    np.testing.assert_allclose(b1["dW_c"], b0["dW_c"], rtol=1e-9, atol=1e-16)
    np.testing.assert_allclose(b1["dH_dec"], b0["dH_dec"][perm], rtol=1e-12, atol=1e-18)
    np.testing.assert_allclose(b1["dH_enc"], b0["dH_enc"][perm], rtol=1e-12, atol=1e-18)


# --------------------------------------------------- finite differences --
def _rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("with_alpha,with_bias", [(False, False), (True, False), (False, True),
                                                  (True, True)])
def test_finite_differences(with_alpha, with_bias):
    """Central differences in fp64 (SPEC.md:131-142 grad_check): every
    gradient, including W_alpha for the Eq. 2 'general' score and the F_c
    bias b_out (NEXT-1)."""
    cfg = CONFIGS["tiny_ragged"]
    inp = make_inputs(cfg, with_alpha=with_alpha, with_bias=with_bias)
    inp = {k: (v.astype(np.float64) if v.dtype == np.float32 else v)
           for k, v in inp.items()}
    Wa = inp.get("W_alpha")
    if Wa is not None:
        Wa = Wa * 10.0  # make the general score matter
    scale = 1.0 / int(inp["tgt_len"].sum())

    def loss_of(**over):
        x = dict(inp, **over)
        f = O.forward(x["H_dec"], x["H_enc"], x["src_len"], x["tgt_len"],
                      x["tgt_ids"], x["W_c"], x["W_out"], scale,
                      W_alpha=over.get("W_alpha", Wa), b_out=x.get("b_out"))
        return f["loss"]

    f, g = O.fwd_bwd(inp["H_dec"], inp["H_enc"], inp["src_len"], inp["tgt_len"],
                     inp["tgt_ids"], inp["W_c"], inp["W_out"], scale, W_alpha=Wa,
                     b_out=inp.get("b_out"))
    names = [("H_dec", "dH_dec"), ("H_enc", "dH_enc"), ("W_c", "dW_c"),
             ("W_out", "dW_out")]
    base = dict(inp)
    if Wa is not None:
        base["W_alpha"] = Wa
        names.append(("W_alpha", "dW_alpha"))
    if with_bias:
        names.append(("b_out", "db_out"))
    eps = 1e-6
    for x_name, g_name in names:
        x = base[x_name]
        fd = np.zeros_like(x)
        it = np.nditer(x, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            xp = x.copy(); xp[idx] += eps
            xm = x.copy(); xm[idx] -= eps
            fd[idx] = (loss_of(**{x_name: xp}) - loss_of(**{x_name: xm})) / (2 * eps)
        err = _rel_l2(g[g_name], fd)
        assert err < 1e-6, (x_name, err)


# ----------------------------------------- independent torch float64 ----
def _torch_stage(inp, scale, W_alpha=None, b_out=None):
    """Direct composition of Eqs. 1-6 with torch ops (float64, CPU)."""
    t = lambda a: torch.tensor(np.asarray(a, np.float64), requires_grad=True)
    Hd, He, Wc, Wo = t(inp["H_dec"]), t(inp["H_enc"]), t(inp["W_c"]), t(inp["W_out"])
    Wa = t(W_alpha) if W_alpha is not None else None
    bo = t(b_out) if b_out is not None else None
    B, N, d = Hd.shape
    M = He.shape[1]
    src = torch.tensor(inp["src_len"]).long()
    tgt = torch.tensor(inp["tgt_len"]).long()
    key_ok = torch.arange(M)[None, None, :] < src[:, None, None]
    q = Hd if Wa is None else Hd @ Wa
    e = torch.einsum("bid,bjd->bij", q, He).masked_fill(~key_ok, float("-inf"))
    a = torch.softmax(e, dim=-1)
    C = torch.einsum("bij,bjd->bid", a, He)
    Hc = torch.tanh(torch.cat([Hd, C], dim=-1) @ Wc.T)
    logits = F.linear(Hc.reshape(B * N, d), Wo, bo)
    valid = (torch.arange(N)[None, :] < tgt[:, None]).reshape(-1)
    y = torch.tensor(inp["tgt_ids"]).long().reshape(-1).clamp(0, Wo.shape[0] - 1)
    nll = F.cross_entropy(logits, y, reduction="none")
    loss = scale * torch.where(valid, nll, torch.zeros_like(nll)).sum()
    loss.backward()
    out = dict(loss=loss.item(), alpha=a.detach().numpy(), C=C.detach().numpy(),
               Hc=Hc.detach().numpy(), dH_dec=Hd.grad.numpy(),
               dH_enc=He.grad.numpy(), dW_c=Wc.grad.numpy(), dW_out=Wo.grad.numpy())
    if Wa is not None:
        out["dW_alpha"] = Wa.grad.numpy()
    if bo is not None:
        out["db_out"] = bo.grad.numpy()
    return out


@pytest.mark.parametrize("name,with_alpha,with_bias", [("tiny_ragged", False, False),
                                                       ("small_f32", False, False),
                                                       ("small_f32", True, False),
                                                       ("small_f32", False, True),
                                                       ("tiny_ragged", True, True)])
def test_torch_float64_autograd(name, with_alpha, with_bias):
    cfg = CONFIGS[name]
    inp = make_inputs(cfg, with_alpha=with_alpha, with_bias=with_bias)
    Wa = inp.get("W_alpha")
    bo = inp.get("b_out")
    scale = 1.0 / int(inp["tgt_len"].sum())
    ref = _torch_stage(inp, scale, Wa, bo)
    f, g = O.fwd_bwd(inp["H_dec"], inp["H_enc"], inp["src_len"], inp["tgt_len"],
                     inp["tgt_ids"], inp["W_c"], inp["W_out"], scale, W_alpha=Wa, b_out=bo)
    assert abs(f["loss"] - ref["loss"]) < 1e-12 * abs(ref["loss"])
    for k in ("alpha", "C", "Hc"):
        np.testing.assert_allclose(f[k], ref[k], rtol=1e-11, atol=1e-14)
    keys = (["dH_dec", "dH_enc", "dW_c", "dW_out"] + (["dW_alpha"] if with_alpha else [])
            + (["db_out"] if with_bias else []))
    for k in keys:
        assert _rel_l2(g[k], ref[k]) < 1e-11, k


# ------------------------------------------------ library special cases --
def test_sdpa_special_case():
    """F1+F2 equal torch's scaled_dot_product_attention(q=H, k=v=S,
    scale=1.0) with a key-padding mask (a library routine)."""
    cfg = CONFIGS["small_f32"]
    inp = make_inputs(cfg)
    H = torch.tensor(inp["H_dec"], dtype=torch.float64)
    S = torch.tensor(inp["H_enc"], dtype=torch.float64)
    mask = torch.arange(cfg.M)[None, None, :] < torch.tensor(inp["src_len"])[:, None, None]
    C_ref = F.scaled_dot_product_attention(H, S, S, attn_mask=mask, scale=1.0)
    e, _ = O.attention_scores(inp["H_dec"], inp["H_enc"])
    C = O.context_vectors(O.attention_weights(e, inp["src_len"]), inp["H_enc"])
    np.testing.assert_allclose(C, C_ref.numpy(), rtol=1e-12, atol=1e-14)


def test_cross_entropy_special_case():
    """F4: sum of token NLL equals F.cross_entropy(logits, y, 'sum')."""
    rng = np.random.default_rng(3)
    logits = rng.normal(0, 3, size=(17, 101))
    y = rng.integers(0, 101, size=17)
    lse = O.log_sum_exp(logits)
    nll = O.token_nll(logits, lse, y)
    ref = F.cross_entropy(torch.tensor(logits), torch.tensor(y), reduction="sum")
    assert abs(nll.sum() - ref.item()) < 1e-12 * abs(ref.item())
    # lse of a constant row is c + ln V exactly (closed form)
    assert abs(O.log_sum_exp(np.full((1, 50), 2.5))[0] - (2.5 + math.log(50))) < 1e-14


# ------------------------------------------------------ F_c bias (NEXT-1) --
def test_e6_bias_only_closed_form():
    """E6: W_out = 0 with a bias b: every valid row's logits are b, so
    loss = scale * sum_valid (logsumexp(b) - b_y) and
    db_out = scale * (T_valid softmax(b) - count_valid(y)); dHc = dl W_out = 0,
    so dW_c, dH_dec and dH_enc vanish exactly."""
    cfg = CONFIGS["tiny_ragged"]
    inp = make_inputs(cfg, with_bias=True)
    b = inp["b_out"].astype(np.float64)
    V = cfg.V
    W0 = np.zeros((V, cfg.d))
    scale = 0.37
    f, g = O.fwd_bwd(inp["H_dec"], inp["H_enc"], inp["src_len"], inp["tgt_len"],
                     inp["tgt_ids"], inp["W_c"], W0, scale, b_out=b)
    lse_b = math.log(sum(math.exp(x) for x in b))
    ys = [int(inp["tgt_ids"][i, j]) for i in range(cfg.B) for j in range(int(inp["tgt_len"][i]))]
    loss = scale * sum(lse_b - b[y] for y in ys)
    assert abs(f["loss"] - loss) < 1e-12 * abs(loss)
    p = np.array([math.exp(x - lse_b) for x in b])
    counts = np.bincount(ys, minlength=V)
    np.testing.assert_allclose(g["db_out"], scale * (len(ys) * p - counts), rtol=1e-11, atol=1e-14)
    assert np.all(g["dW_c"] == 0) and np.all(g["dH_dec"] == 0) and np.all(g["dH_enc"] == 0)


def test_bias_shift_invariance_and_zero_sum():
    """Softmax is invariant to a constant shift of the bias: b_out + c gives
    the same loss and gradients; and db_out sums to zero (each dl row does)."""
    cfg = CONFIGS["small_f32"]
    inp = make_inputs(cfg, with_bias=True)
    scale = 1.0 / int(inp["tgt_len"].sum())
    args = (inp["H_dec"], inp["H_enc"], inp["src_len"], inp["tgt_len"], inp["tgt_ids"],
            inp["W_c"], inp["W_out"], scale)
    f0, g0 = O.fwd_bwd(*args, b_out=inp["b_out"])
    f1, g1 = O.fwd_bwd(*args, b_out=inp["b_out"].astype(np.float64) + 3.25)
    assert abs(f0["loss"] - f1["loss"]) < 1e-11 * abs(f0["loss"])
    for k in ("dW_out", "dW_c", "dH_dec", "dH_enc", "db_out"):
        np.testing.assert_allclose(g1[k], g0[k], rtol=1e-8, atol=1e-15)
    assert abs(g0["db_out"].sum()) < 1e-12
    # and a nonzero bias really changes the result (the term is not dropped)
    f2, _ = O.fwd_bwd(*args)
    assert abs(f2["loss"] - f0["loss"]) > 1e-3


# ------------------------------------------------ decoding step (NEXT-4) --
def test_decode_step_against_torch_log_softmax_and_topk():
    """decode_step's log-probabilities equal torch.log_softmax of the logits of
    an independent torch composition, and its top-k equals torch.topk (no
    ties in random data); with k = V the probabilities sum to 1."""
    cfg = CONFIGS["small_f32"]
    inp = make_inputs(cfg, with_bias=True)
    k = 5
    ids, logp, lse = O.decode_step(inp["H_dec"], inp["H_enc"], inp["src_len"], inp["W_c"],
                                   inp["W_out"], k, b_out=inp["b_out"])
    t = lambda a: torch.tensor(np.asarray(a, np.float64))
    Hd, He = t(inp["H_dec"]), t(inp["H_enc"])
    B, N, d = Hd.shape
    M = He.shape[1]
    key_ok = torch.arange(M)[None, None, :] < torch.tensor(inp["src_len"])[:, None, None]
    e = torch.einsum("bid,bjd->bij", Hd, He).masked_fill(~key_ok, float("-inf"))
    C = torch.einsum("bij,bjd->bid", torch.softmax(e, -1), He)
    Hc = torch.tanh(torch.cat([Hd, C], -1) @ t(inp["W_c"]).T)
    lp = torch.log_softmax(F.linear(Hc.reshape(B * N, d), t(inp["W_out"]), t(inp["b_out"])), -1)
    tv, ti = torch.topk(lp, k, dim=-1)
    np.testing.assert_array_equal(ids.reshape(-1, k), ti.numpy())
    np.testing.assert_allclose(logp.reshape(-1, k), tv.numpy(), rtol=1e-12, atol=1e-12)
    _, lp_all, _ = O.decode_step(inp["H_dec"][:1], inp["H_enc"][:1], inp["src_len"][:1],
                                 inp["W_c"], inp["W_out"], cfg.V)
    np.testing.assert_allclose(np.exp(lp_all).sum(-1), 1.0, rtol=1e-12)
    assert np.all(np.diff(lp_all, axis=-1) <= 0)


def test_decode_step_ties_prefer_lower_ids():
    """Duplicated W_out rows give exactly equal logits: in the full ranking
    (k = V) the tied tokens appear consecutively, lower id first."""
    cfg = CONFIGS["tiny"]
    inp = make_inputs(cfg)
    W = inp["W_out"].astype(np.float64).copy()
    W[7] = W[3]
    W[40] = W[3]
    ids, logp, _ = O.decode_step(inp["H_dec"], inp["H_enc"], inp["src_len"], inp["W_c"], W, cfg.V)
    flat, lp = ids.reshape(-1, cfg.V), logp.reshape(-1, cfg.V)
    for r in range(flat.shape[0]):
        pos = [int(np.where(flat[r] == v)[0][0]) for v in (3, 7, 40)]
        assert pos[1] == pos[0] + 1 and pos[2] == pos[1] + 1, pos
        assert lp[r, pos[0]] == lp[r, pos[2]]
