"""Property-based pins of the stage oracle (hypothesis): on random small shapes,
lengths, scales and weights, the oracle must agree with an independent
float64 torch composition + autograd, and keep the invariants of SURVEY.md
§8(c) -- I1 rows of alpha sum to 1, I2 masked alpha exactly 0, I3 / I4
padded dH rows exactly 0, I6 the column sums of dW_out vanish -- and the
loss equals the mean cross-entropy of torch.nn.functional.cross_entropy on the
logits it implies.  A dropped term, a wrong sign or index, or a transposed
operand anywhere in the oracle fails one of these for most draws."""
import numpy as np
import torch
import torch.nn.functional as F
from hypothesis import given, settings, strategies as st

from oracle import attn_softmax_oracle as O


@st.composite
def problems(draw):
    B = draw(st.integers(1, 3))
    N = draw(st.integers(1, 5))
    M = draw(st.integers(1, 6))
    d = draw(st.integers(1, 6))
    V = draw(st.integers(2, 9))
    seed = draw(st.integers(0, 2**31 - 1))
    rng = np.random.default_rng(seed)
    src = rng.integers(1, M + 1, size=B).astype(np.int32)
    tgt = rng.integers(0, N + 1, size=B).astype(np.int32)
    if tgt.sum() == 0:
        tgt[0] = 1
    wscale = draw(st.sampled_from([0.1, 1.0, 3.0]))
    return dict(H_dec=rng.normal(size=(B, N, d)), H_enc=rng.normal(size=(B, M, d)),
                src_len=src, tgt_len=tgt, tgt_ids=rng.integers(0, V, size=(B, N)).astype(np.int32),
                W_c=rng.normal(size=(d, 2 * d)) * wscale, W_out=rng.normal(size=(V, d)) * wscale,
                scale=float(draw(st.sampled_from([1.0, 0.25]))))


def _torch_reference(p):
    H = torch.tensor(p["H_dec"], requires_grad=True)
    S = torch.tensor(p["H_enc"], requires_grad=True)
    Wc = torch.tensor(p["W_c"], requires_grad=True)
    Wo = torch.tensor(p["W_out"], requires_grad=True)
    B, N, d = H.shape
    M = S.shape[1]
    mask = torch.arange(M)[None, None, :] < torch.tensor(p["src_len"])[:, None, None]
    e = (H @ S.transpose(1, 2)).masked_fill(~mask, float("-inf"))
    a = torch.softmax(e, -1)
    C = a @ S
    Hc = torch.tanh(torch.cat([H, C], -1) @ Wc.T)
    logits = Hc @ Wo.T
    valid = torch.arange(N)[None, :] < torch.tensor(p["tgt_len"])[:, None]
    y = torch.tensor(p["tgt_ids"], dtype=torch.long)
    ce = F.cross_entropy(logits[valid], y[valid], reduction="sum")
    loss = p["scale"] * ce
    loss.backward()
    return loss.item(), {"dH_dec": H.grad.numpy(), "dH_enc": S.grad.numpy(),
                         "dW_c": Wc.grad.numpy(), "dW_out": Wo.grad.numpy()}, a.detach().numpy()


@settings(max_examples=60, deadline=None)
@given(problems())
def test_oracle_matches_torch_and_keeps_invariants(p):
    f, b = O.fwd_bwd(p["H_dec"], p["H_enc"], p["src_len"], p["tgt_len"], p["tgt_ids"], p["W_c"],
                     p["W_out"], p["scale"])
    loss, grads, alpha = _torch_reference(p)
    assert abs(f["loss"] - loss) <= 1e-10 * max(1.0, abs(loss))
    for k, g in grads.items():
        assert np.allclose(b[k], g, rtol=1e-9, atol=1e-11), k
    A = np.asarray(f["alpha"]).reshape(alpha.shape)
    assert np.allclose(A, alpha, rtol=1e-12, atol=1e-14)
    for bb in range(len(p["src_len"])):
        L, Tb = int(p["src_len"][bb]), int(p["tgt_len"][bb])
        assert np.all(A[bb, :, L:] == 0.0)                       # I2
        assert np.allclose(A[bb].sum(-1), 1.0, atol=1e-12)       # I1
        assert np.all(b["dH_enc"][bb, L:] == 0.0)                # I3
        assert np.all(b["dH_dec"][bb, Tb:] == 0.0)               # I4
    assert np.allclose(b["dW_out"].sum(0), 0.0, atol=1e-10 * max(1.0, np.abs(b["dW_out"]).max()))   # I6
