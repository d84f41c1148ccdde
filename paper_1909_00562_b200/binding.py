"""ctypes binding of libattnsm.so (include/attn_softmax.h).

Argument marshalling only: every step of the stage runs in the library's
CUDA kernels.  PyTorch supplies device memory and streams.  There is no CPU
fallback -- if the library is missing, lib() raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ATTNSM_LIB: load another build of the same library (same-box A/B timing)
LIB_PATH = os.environ.get("ATTNSM_LIB") or os.path.join(_HERE, "lib", "libattnsm.so")

ATTN_F32, ATTN_BF16 = 0, 1
STATUS = {0: "ATTN_OK", 1: "ATTN_ERR_INVALID_ARG", 2: "ATTN_ERR_SHAPE",
          3: "ATTN_ERR_EMPTY_SOURCE", 4: "ATTN_ERR_NO_TARGETS",
          5: "ATTN_ERR_TOKEN_RANGE", 6: "ATTN_ERR_WORKSPACE",
          7: "ATTN_ERR_UNSUPPORTED", 8: "ATTN_ERR_CUDA", 9: "ATTN_ERR_NCCL"}

# every symbol include/attn_softmax.h and attn_softmax_debug.h declare
EXPORTS = [
    "attn_softmax_workspace_size", "attn_softmax_fwd_bwd", "attn_softmax_fwd_bwd_ex",
    "attn_softmax_host_staging_size", "attn_softmax_fwd_bwd_host",
    "attn_softmax_prefetch_host", "attn_softmax_fwd_bwd_staged",
    "attn_softmax_check_ids", "attn_grad_allreduce", "attn_comm_get_unique_id",
    "attn_comm_init", "attn_comm_destroy", "attn_comm_poll", "attn_comm_nranks",
    "attn_last_error", "attn_version",
    "attn_softmax_workspace_views", "attn_debug_gemm_bf16",
    "attn_softmax_set_option", "attn_softmax_stage_count",
    "attn_softmax_stage_time", "attn_softmax_last_launches",
    "attn_adam_step", "attn_adam_shard_len", "attn_adam_step_sharded",
    "attn_softmax_decode_workspace_size", "attn_softmax_decode_step",
    "attn_lstm_workspace_size", "attn_lstm_packed_bytes", "attn_lstm_pack_layer",
    "attn_encoder_decoder_fwd", "attn_hidden_scatter", "attn_lstm_if_workspace_size",
    "attn_encoder_decoder_if_fwd", "attn_lstm_train_workspace_size",
    "attn_encoder_decoder_fwd_train", "attn_encoder_decoder_bwd",
]


class AttnError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class AttnShape(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("tgt_len", ctypes.c_int32),
                ("src_len", ctypes.c_int32), ("hidden", ctypes.c_int32),
                ("vocab", ctypes.c_int32), ("dtype", ctypes.c_int32)]


class AdamParams(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double), ("step", ctypes.c_int32)]


class LstmShape(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("src_len", ctypes.c_int32),
                ("tgt_len", ctypes.c_int32), ("emb", ctypes.c_int32),
                ("hidden", ctypes.c_int32), ("layers", ctypes.c_int32),
                ("vocab_src", ctypes.c_int32), ("vocab_tgt", ctypes.c_int32)]


class AttnWsViews(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_size_t), ("ctx", ctypes.c_size_t),
                ("hc", ctypes.c_size_t), ("lse", ctypes.c_size_t),
                ("nll", ctypes.c_size_t), ("vocab_chunk", ctypes.c_int64),
                ("alpha_ld", ctypes.c_int64)]


_lib = None
_P = ctypes.c_void_p


def lib() -> ctypes.CDLL:
    """Load libattnsm.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libattnsm.so not built: {LIB_PATH} is missing "
                           "(run __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    S = ctypes.POINTER(AttnShape)
    i32p = ctypes.POINTER(ctypes.c_int32)
    L.attn_softmax_workspace_size.argtypes = [S]
    L.attn_softmax_workspace_size.restype = ctypes.c_size_t
    L.attn_softmax_fwd_bwd.argtypes = [S, _P, _P, i32p, i32p, _P, _P, _P, _P,
                                       ctypes.c_float, _P, _P, _P, _P, _P, _P,
                                       _P, ctypes.c_size_t, _P, _P]
    L.attn_softmax_fwd_bwd.restype = ctypes.c_int
    L.attn_softmax_fwd_bwd_ex.argtypes = [S, _P, _P, i32p, i32p, _P, _P, _P, _P, _P,
                                          ctypes.c_float, _P, _P, _P, _P, _P, _P, _P,
                                          _P, ctypes.c_size_t, _P, _P]
    L.attn_softmax_fwd_bwd_ex.restype = ctypes.c_int
    L.attn_softmax_host_staging_size.argtypes = [S]
    L.attn_softmax_host_staging_size.restype = ctypes.c_size_t
    L.attn_softmax_fwd_bwd_host.argtypes = [S, _P, _P, i32p, i32p, _P, _P, _P,
                                            ctypes.c_float, _P, _P, _P, _P, _P,
                                            _P, ctypes.c_size_t, _P, ctypes.c_size_t,
                                            _P, _P]
    L.attn_softmax_fwd_bwd_host.restype = ctypes.c_int
    L.attn_softmax_prefetch_host.argtypes = [S, _P, _P, _P, _P, ctypes.c_size_t, _P]
    L.attn_softmax_prefetch_host.restype = ctypes.c_int
    L.attn_softmax_fwd_bwd_staged.argtypes = [S, _P, ctypes.c_size_t, i32p, i32p, _P, _P,
                                              ctypes.c_float, _P, _P, _P, _P, _P, _P,
                                              ctypes.c_size_t, _P, _P]
    L.attn_softmax_fwd_bwd_staged.restype = ctypes.c_int
    L.attn_softmax_check_ids.argtypes = [S, i32p, _P, _P]
    L.attn_softmax_check_ids.restype = ctypes.c_int
    L.attn_grad_allreduce.argtypes = [_P, _P, ctypes.c_size_t, _P]
    L.attn_grad_allreduce.restype = ctypes.c_int
    L.attn_comm_get_unique_id.argtypes = [ctypes.c_char_p]
    L.attn_comm_get_unique_id.restype = ctypes.c_int
    L.attn_comm_init.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, ctypes.POINTER(_P)]
    L.attn_comm_init.restype = ctypes.c_int
    L.attn_comm_destroy.argtypes = [_P]
    L.attn_comm_destroy.restype = ctypes.c_int
    L.attn_comm_poll.argtypes = [_P, ctypes.c_int64]
    L.attn_comm_poll.restype = ctypes.c_int
    L.attn_comm_nranks.argtypes = [_P]
    L.attn_comm_nranks.restype = ctypes.c_int
    L.attn_last_error.argtypes = []
    L.attn_last_error.restype = ctypes.c_char_p
    L.attn_version.argtypes = []
    L.attn_version.restype = ctypes.c_char_p
    L.attn_softmax_workspace_views.argtypes = [S, ctypes.POINTER(AttnWsViews)]
    L.attn_softmax_workspace_views.restype = ctypes.c_int
    L.attn_debug_gemm_bf16.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       _P, ctypes.c_int, _P, ctypes.c_int, _P, _P]
    L.attn_debug_gemm_bf16.restype = ctypes.c_int
    L.attn_softmax_set_option.argtypes = [ctypes.c_char_p, ctypes.c_int64]
    L.attn_softmax_set_option.restype = ctypes.c_int
    L.attn_softmax_stage_count.argtypes = []
    L.attn_softmax_stage_count.restype = ctypes.c_int
    L.attn_softmax_stage_time.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_char_p),
                                          ctypes.POINTER(ctypes.c_float)]
    L.attn_softmax_stage_time.restype = ctypes.c_int
    L.attn_softmax_last_launches.argtypes = []
    L.attn_softmax_last_launches.restype = ctypes.c_longlong
    L.attn_softmax_decode_workspace_size.argtypes = [S]
    L.attn_softmax_decode_workspace_size.restype = ctypes.c_size_t
    L.attn_softmax_decode_step.argtypes = [S, _P, _P, i32p, _P, _P, _P, _P, ctypes.c_int, _P, _P,
                                           _P, _P, ctypes.c_size_t, _P]
    L.attn_softmax_decode_step.restype = ctypes.c_int
    A = ctypes.POINTER(AdamParams)
    L.attn_adam_step.argtypes = [A, ctypes.c_size_t, _P, _P, _P, _P, _P, _P]
    L.attn_adam_step.restype = ctypes.c_int
    L.attn_adam_shard_len.argtypes = [_P, ctypes.c_size_t]
    L.attn_adam_shard_len.restype = ctypes.c_size_t
    L.attn_adam_step_sharded.argtypes = [_P, A, ctypes.c_size_t, _P, _P, _P, _P, _P, _P]
    L.attn_adam_step_sharded.restype = ctypes.c_int
    LS = ctypes.POINTER(LstmShape)
    L.attn_lstm_workspace_size.argtypes = [LS]
    L.attn_lstm_workspace_size.restype = ctypes.c_size_t
    L.attn_lstm_packed_bytes.argtypes = [ctypes.c_int, ctypes.c_int]
    L.attn_lstm_packed_bytes.restype = ctypes.c_size_t
    L.attn_lstm_pack_layer.argtypes = [ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, _P, _P]
    L.attn_lstm_pack_layer.restype = ctypes.c_int
    L.attn_encoder_decoder_fwd.argtypes = [LS, _P, _P, i32p, _P, _P, ctypes.POINTER(_P),
                                           ctypes.POINTER(_P), ctypes.POINTER(_P),
                                           ctypes.POINTER(_P), _P, _P, _P, ctypes.c_size_t, _P]
    L.attn_encoder_decoder_fwd.restype = ctypes.c_int
    L.attn_hidden_scatter.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      _P, _P, _P]
    L.attn_lstm_if_workspace_size.argtypes = [LS]
    L.attn_lstm_if_workspace_size.restype = ctypes.c_size_t
    L.attn_encoder_decoder_if_fwd.argtypes = [LS, _P, _P, i32p, _P, _P, ctypes.POINTER(_P),
                                              ctypes.POINTER(_P), ctypes.POINTER(_P),
                                              ctypes.POINTER(_P), _P, _P, _P, _P, _P,
                                              ctypes.c_size_t, _P]
    L.attn_encoder_decoder_if_fwd.restype = ctypes.c_int
    L.attn_lstm_train_workspace_size.argtypes = [LS]
    L.attn_lstm_train_workspace_size.restype = ctypes.c_size_t
    L.attn_encoder_decoder_fwd_train.argtypes = L.attn_encoder_decoder_fwd.argtypes
    L.attn_encoder_decoder_fwd_train.restype = ctypes.c_int
    PP = ctypes.POINTER(_P)
    L.attn_encoder_decoder_bwd.argtypes = [LS, _P, _P, i32p, PP, PP, _P, _P, _P, _P, PP, PP, PP, PP,
                                           _P, _P, _P, ctypes.c_size_t, _P]
    L.attn_encoder_decoder_bwd.restype = ctypes.c_int
    L.attn_hidden_scatter.restype = ctypes.c_int
    _lib = L
    return L


def _check(code: int):
    if code != 0:
        raise AttnError(code, lib().attn_last_error().decode())


def shape(B, N, M, d, V, dtype) -> AttnShape:
    dt = {"f32": ATTN_F32, "bf16": ATTN_BF16, ATTN_F32: ATTN_F32,
          ATTN_BF16: ATTN_BF16}[dtype]
    return AttnShape(B, N, M, d, V, dt)


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _i32(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def attn_softmax_workspace_size(s: AttnShape) -> int:
    n = lib().attn_softmax_workspace_size(ctypes.byref(s))
    if n == 0:
        raise AttnError(2, lib().attn_last_error().decode())
    return n


def attn_softmax_host_staging_size(s: AttnShape) -> int:
    return lib().attn_softmax_host_staging_size(ctypes.byref(s))


def attn_softmax_workspace_views(s: AttnShape) -> AttnWsViews:
    v = AttnWsViews()
    _check(lib().attn_softmax_workspace_views(ctypes.byref(s), ctypes.byref(v)))
    return v


def attn_softmax_fwd_bwd(s, H_dec, H_enc, src_lens, tgt_lens, tgt_ids, W_c,
                         W_out, loss_scale, loss, dH_dec, dH_enc, dW_c, dW_out,
                         workspace, comm=None, stream=None, W_alpha=None,
                         dW_alpha=None):
    src, src_p = _i32(src_lens)
    tgt, tgt_p = _i32(tgt_lens)
    _check(lib().attn_softmax_fwd_bwd(
        ctypes.byref(s), _ptr(H_dec), _ptr(H_enc), src_p, tgt_p, _ptr(tgt_ids),
        _ptr(W_c), _ptr(W_out), _ptr(W_alpha), float(loss_scale), _ptr(loss),
        _ptr(dH_dec), _ptr(dH_enc), _ptr(dW_c), _ptr(dW_out), _ptr(dW_alpha),
        _ptr(workspace), workspace.numel() * workspace.element_size(),
        comm, _stream(stream)))


def attn_softmax_fwd_bwd_ex(s, H_dec, H_enc, src_lens, tgt_lens, tgt_ids, W_c, W_out,
                            loss_scale, loss, dH_dec, dH_enc, dW_c, dW_out, workspace,
                            comm=None, stream=None, W_alpha=None, dW_alpha=None, b_out=None,
                            db_out=None):
    src, src_p = _i32(src_lens)
    tgt, tgt_p = _i32(tgt_lens)
    _check(lib().attn_softmax_fwd_bwd_ex(
        ctypes.byref(s), _ptr(H_dec), _ptr(H_enc), src_p, tgt_p, _ptr(tgt_ids),
        _ptr(W_c), _ptr(W_out), _ptr(W_alpha), _ptr(b_out), float(loss_scale), _ptr(loss),
        _ptr(dH_dec), _ptr(dH_enc), _ptr(dW_c), _ptr(dW_out), _ptr(dW_alpha), _ptr(db_out),
        _ptr(workspace), workspace.numel() * workspace.element_size(),
        comm, _stream(stream)))


def attn_softmax_fwd_bwd_host(s, H_dec_host, H_enc_host, src_lens, tgt_lens,
                              tgt_ids_host, W_c, W_out, loss_scale, loss_host,
                              dH_dec, dH_enc, dW_c, dW_out, staging, workspace,
                              comm=None, stream=None):
    src, src_p = _i32(src_lens)
    tgt, tgt_p = _i32(tgt_lens)
    _check(lib().attn_softmax_fwd_bwd_host(
        ctypes.byref(s), _ptr(H_dec_host), _ptr(H_enc_host), src_p, tgt_p,
        _ptr(tgt_ids_host), _ptr(W_c), _ptr(W_out), float(loss_scale),
        _ptr(loss_host), _ptr(dH_dec), _ptr(dH_enc), _ptr(dW_c), _ptr(dW_out),
        _ptr(staging), staging.numel() * staging.element_size(),
        _ptr(workspace), workspace.numel() * workspace.element_size(),
        comm, _stream(stream)))


def attn_softmax_prefetch_host(s, H_dec_host, H_enc_host, tgt_ids_host, staging, stream=None):
    _check(lib().attn_softmax_prefetch_host(
        ctypes.byref(s), _ptr(H_dec_host), _ptr(H_enc_host), _ptr(tgt_ids_host), _ptr(staging),
        staging.numel() * staging.element_size(), _stream(stream)))


def attn_softmax_fwd_bwd_staged(s, staging, src_lens, tgt_lens, W_c, W_out, loss_scale,
                                loss_host, dH_dec, dH_enc, dW_c, dW_out, workspace,
                                comm=None, stream=None):
    src, src_p = _i32(src_lens)
    tgt, tgt_p = _i32(tgt_lens)
    _check(lib().attn_softmax_fwd_bwd_staged(
        ctypes.byref(s), _ptr(staging), staging.numel() * staging.element_size(), src_p, tgt_p,
        _ptr(W_c), _ptr(W_out), float(loss_scale), _ptr(loss_host), _ptr(dH_dec), _ptr(dH_enc),
        _ptr(dW_c), _ptr(dW_out), _ptr(workspace), workspace.numel() * workspace.element_size(),
        comm, _stream(stream)))


def attn_softmax_check_ids(s, tgt_lens, tgt_ids, stream=None):
    tgt, tgt_p = _i32(tgt_lens)
    _check(lib().attn_softmax_check_ids(ctypes.byref(s), tgt_p, _ptr(tgt_ids),
                                        _stream(stream)))


def attn_grad_allreduce(comm, buf, stream=None):
    _check(lib().attn_grad_allreduce(comm, _ptr(buf), buf.numel(), _stream(stream)))


def attn_comm_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().attn_comm_get_unique_id(buf))
    return buf.raw


def attn_comm_init(uid: bytes, nranks: int, rank: int, device: int):
    out = _P()
    _check(lib().attn_comm_init(uid, nranks, rank, device, ctypes.byref(out)))
    return out


def attn_comm_destroy(comm):
    _check(lib().attn_comm_destroy(comm))


def attn_comm_poll(comm, timeout_ms: int = 0):
    """Wait for the communicator's enqueued collectives, polling NCCL's
    asynchronous error state; raises AttnError (ATTN_ERR_NCCL) on an error or
    after timeout_ms (> 0) -- the communicator is then aborted."""
    _check(lib().attn_comm_poll(comm, int(timeout_ms)))


def attn_comm_nranks(comm) -> int:
    return int(lib().attn_comm_nranks(comm))


def attn_debug_gemm_bf16(M, N, K, A, a_mn, B, b_mn, C, stream=None):
    _check(lib().attn_debug_gemm_bf16(M, N, K, _ptr(A), int(a_mn), _ptr(B),
                                      int(b_mn), _ptr(C), _stream(stream)))


def attn_softmax_set_option(key: str, value: int):
    _check(lib().attn_softmax_set_option(key.encode(), int(value)))


def attn_softmax_stage_times() -> dict:
    """{step name: ms} of the last call (needs option stage_events = 1)."""
    out = {}
    for i in range(lib().attn_softmax_stage_count()):
        name = ctypes.c_char_p()
        ms = ctypes.c_float()
        _check(lib().attn_softmax_stage_time(i, ctypes.byref(name), ctypes.byref(ms)))
        out[name.value.decode()] = ms.value
    return out


def attn_softmax_last_launches() -> int:
    return int(lib().attn_softmax_last_launches())


def attn_last_error() -> str:
    return lib().attn_last_error().decode()


def attn_version() -> str:
    return lib().attn_version().decode()


def adam_params(step, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8) -> AdamParams:
    """Adam hyper-parameters; the defaults are the paper's."""
    return AdamParams(lr, beta1, beta2, eps, int(step))


def attn_adam_step(h: AdamParams, w, m, v, g, w_bf16=None, stream=None):
    _check(lib().attn_adam_step(ctypes.byref(h), w.numel(), _ptr(w), _ptr(m), _ptr(v), _ptr(g),
                                _ptr(w_bf16), _stream(stream)))


def attn_adam_shard_len(comm, n: int) -> int:
    return int(lib().attn_adam_shard_len(comm, n))


def attn_adam_step_sharded(comm, h: AdamParams, n: int, g, w_shard, m_shard, v_shard, w_bf16,
                           stream=None):
    _check(lib().attn_adam_step_sharded(comm, ctypes.byref(h), n, _ptr(g), _ptr(w_shard),
                                        _ptr(m_shard), _ptr(v_shard), _ptr(w_bf16),
                                        _stream(stream)))


def attn_softmax_decode_workspace_size(s: AttnShape) -> int:
    n = lib().attn_softmax_decode_workspace_size(ctypes.byref(s))
    if n == 0:
        raise AttnError(7, "decode step: invalid shape or fp32 (bf16 only)")
    return n


def attn_softmax_decode_step(s, H_dec, H_enc, src_lens, W_c, W_out, k, topk_ids, topk_logp,
                             workspace, lse=None, W_alpha=None, b_out=None, stream=None):
    src, src_p = _i32(src_lens)
    _check(lib().attn_softmax_decode_step(
        ctypes.byref(s), _ptr(H_dec), _ptr(H_enc), src_p, _ptr(W_c), _ptr(W_out), _ptr(W_alpha),
        _ptr(b_out), int(k), _ptr(topk_ids), _ptr(topk_logp), _ptr(lse), _ptr(workspace),
        workspace.numel() * workspace.element_size(), _stream(stream)))


# ---------------------------------------------------------------- NEXT-3
def lstm_shape(B, M, N, emb, hidden, layers, vocab_src, vocab_tgt) -> LstmShape:
    return LstmShape(B, M, N, emb, hidden, layers, vocab_src, vocab_tgt)


def attn_lstm_workspace_size(s: LstmShape) -> int:
    n = lib().attn_lstm_workspace_size(ctypes.byref(s))
    if n == 0:
        raise AttnError(7, lib().attn_last_error().decode())
    return n


def attn_lstm_packed_bytes(in_dim: int, hidden: int) -> int:
    return int(lib().attn_lstm_packed_bytes(int(in_dim), int(hidden)))


def attn_lstm_pack_layer(in_dim, hidden, W_ih, W_hh, b, W_packed, b_packed, stream=None):
    _check(lib().attn_lstm_pack_layer(int(in_dim), int(hidden), _ptr(W_ih), _ptr(W_hh), _ptr(b),
                                      _ptr(W_packed), _ptr(b_packed), _stream(stream)))


def attn_encoder_decoder_fwd(s: LstmShape, src_ids, tgt_ids, src_lens, E_src, E_tgt, enc_W, enc_b,
                             dec_W, dec_b, H_enc, H_dec, workspace, stream=None):
    src, src_p = _i32(src_lens)

    def arr(ts):
        return (_P * len(ts))(*[t.data_ptr() for t in ts])
    eW, eb, dW, db = arr(enc_W), arr(enc_b), arr(dec_W), arr(dec_b)
    _check(lib().attn_encoder_decoder_fwd(
        ctypes.byref(s), _ptr(src_ids), _ptr(tgt_ids), src_p, _ptr(E_src), _ptr(E_tgt), eW, eb,
        dW, db, _ptr(H_enc), _ptr(H_dec), _ptr(workspace),
        workspace.numel() * workspace.element_size(), _stream(stream)))


def attn_hidden_scatter(comm, root, B_global, rows, hidden, full, shard, stream=None):
    _check(lib().attn_hidden_scatter(comm, int(root), int(B_global), int(rows), int(hidden),
                                     _ptr(full), _ptr(shard), _stream(stream)))


def attn_lstm_if_workspace_size(s: LstmShape) -> int:
    n = lib().attn_lstm_if_workspace_size(ctypes.byref(s))
    if n == 0:
        raise AttnError(7, lib().attn_last_error().decode())
    return n


def attn_encoder_decoder_if_fwd(s: LstmShape, src_ids, tgt_ids, src_lens, E_src, E_tgt, enc_W,
                                enc_b, dec_W, dec_b, W_c, H_enc, H_dec, Htilde, workspace,
                                stream=None):
    src, src_p = _i32(src_lens)

    def arr(ts):
        return (_P * len(ts))(*[t.data_ptr() for t in ts])
    eW, eb, dW, db = arr(enc_W), arr(enc_b), arr(dec_W), arr(dec_b)
    _check(lib().attn_encoder_decoder_if_fwd(
        ctypes.byref(s), _ptr(src_ids), _ptr(tgt_ids), src_p, _ptr(E_src), _ptr(E_tgt), eW, eb,
        dW, db, _ptr(W_c), _ptr(H_enc), _ptr(H_dec), _ptr(Htilde), _ptr(workspace),
        workspace.numel() * workspace.element_size(), _stream(stream)))


def attn_lstm_train_workspace_size(s: LstmShape) -> int:
    n = lib().attn_lstm_train_workspace_size(ctypes.byref(s))
    if n == 0:
        raise AttnError(7, lib().attn_last_error().decode())
    return n


def _ptrs(ts):
    return (_P * len(ts))(*[t.data_ptr() for t in ts])


def attn_encoder_decoder_fwd_train(s: LstmShape, src_ids, tgt_ids, src_lens, E_src, E_tgt, enc_W,
                                   enc_b, dec_W, dec_b, H_enc, H_dec, workspace, stream=None):
    src, src_p = _i32(src_lens)
    _check(lib().attn_encoder_decoder_fwd_train(
        ctypes.byref(s), _ptr(src_ids), _ptr(tgt_ids), src_p, _ptr(E_src), _ptr(E_tgt),
        _ptrs(enc_W), _ptrs(enc_b), _ptrs(dec_W), _ptrs(dec_b), _ptr(H_enc), _ptr(H_dec),
        _ptr(workspace), workspace.numel() * workspace.element_size(), _stream(stream)))


def attn_encoder_decoder_bwd(s: LstmShape, src_ids, tgt_ids, src_lens, enc_W, dec_W, H_enc, H_dec,
                             dH_enc, dH_dec, dW_enc, db_enc, dW_dec, db_dec, dE_src, dE_tgt,
                             workspace, stream=None):
    src, src_p = _i32(src_lens)
    _check(lib().attn_encoder_decoder_bwd(
        ctypes.byref(s), _ptr(src_ids), _ptr(tgt_ids), src_p, _ptrs(enc_W), _ptrs(dec_W),
        _ptr(H_enc), _ptr(H_dec), _ptr(dH_enc), _ptr(dH_dec), _ptrs(dW_enc), _ptrs(db_enc),
        _ptrs(dW_dec), _ptrs(db_dec), _ptr(dE_src), _ptr(dE_tgt), _ptr(workspace),
        workspace.numel() * workspace.element_size(), _stream(stream)))
