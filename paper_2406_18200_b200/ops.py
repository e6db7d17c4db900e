"""Single-kernel entry points (include/seed_ops.h) for parity tests: marshalling only."""
import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import check


def _s():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def philox(c0, c1, c2, c3, k0, k1, n):
    """K7: words of Philox4x32-10 for counters (c0 + i, c1, c2, c3), i < n -> uint32 as int64 [n][4]."""
    out = torch.empty((n, 4), dtype=torch.int32, device="cuda")
    check(_lib.load().seed_op_philox(c0, c1, c2, c3, k0, k1, n, _p(out), _s()), None, "seed_op_philox")
    return out.cpu().numpy().view(np.uint32).astype(np.int64)


def gemm(W, X):
    """K2: Y = X W^T, W [N][K] bf16, X [M][K] bf16 (CUDA) -> fp32 [M][N]."""
    N, K = W.shape
    M = X.shape[0]
    Y = torch.empty((M, N), dtype=torch.float32, device="cuda")
    check(_lib.load().seed_op_gemm(_p(W.contiguous()), N, K, _p(X.contiguous()), M, _p(Y), _s()), None,
          "seed_op_gemm")
    return Y


def verify(zt, zd, xs, temperature, seed, sids, rs, bonus=True, want_dbg=True):
    """K4 on given logits. zt [B][g+1][V], zd [B][g][V] fp32 CUDA; xs [B][g] int32 CUDA."""
    B, g1, V = zt.shape
    g = g1 - 1
    dev = zt.device
    sids_t = torch.as_tensor(np.asarray(sids, dtype=np.int64).astype(np.uint32).view(np.int32), device=dev)
    rs_t = torch.as_tensor(np.asarray(rs, dtype=np.int32), device=dev)
    out_tok = torch.empty((B, g + 1), dtype=torch.int32, device=dev)
    out_cnt = torch.empty(B, dtype=torch.int32, device=dev)
    out_acc = torch.empty(B, dtype=torch.int32, device=dev)
    dbg = torch.empty((B, g, 4), dtype=torch.float32, device=dev) if want_dbg else None
    stats = torch.empty((B, 2 * g + 1, 2), dtype=torch.float64, device=dev) if want_dbg else None
    check(_lib.load().seed_op_verify(_p(zt.contiguous()), _p(zd.contiguous()), _p(xs.contiguous()), B, g, V,
                                     float(temperature), int(seed), _p(sids_t), _p(rs_t), int(bool(bonus)),
                                     _p(out_tok), _p(out_cnt), _p(out_acc), _p(dbg), _p(stats), _s()), None,
          "seed_op_verify")
    return {"out_tok": out_tok, "out_cnt": out_cnt, "a": out_acc, "dbg": dbg, "stats": stats}


def draft_sample(z, temperature, seed, sids, rs, j):
    """K1 sampler over rows of z [B][V] fp32 CUDA -> int32 [B]."""
    B, V = z.shape
    dev = z.device
    sids_t = torch.as_tensor(np.asarray(sids, dtype=np.int64).astype(np.uint32).view(np.int32), device=dev)
    rs_t = torch.as_tensor(np.asarray(rs, dtype=np.int32), device=dev)
    out = torch.empty(B, dtype=torch.int32, device=dev)
    check(_lib.load().seed_op_draft_sample(_p(z.contiguous()), V, B, V, float(temperature), int(seed), _p(sids_t),
                                           _p(rs_t), int(j), _p(out), _s()), None, "seed_op_draft_sample")
    return out


def decoder_layer(shape, L, x_in, ctx_len, k_prev=None, v_prev=None):
    """One decoder layer on hidden states x_in [M][d] fp32 CUDA at positions ctx_len..; returns
    (x_out fp32, k_new bf16 [M][Hk][Dh], v_new bf16)."""
    from . import LAYER_KEYS, model_shape
    M, d = x_in.shape
    hk = shape.get("n_kv_heads", 0) or shape["n_heads"]
    dh = d // shape["n_heads"]
    ptrs = (C.c_void_p * 9)(*[L[k].data_ptr() for k in LAYER_KEYS])
    sh = model_shape(shape)
    x_out = torch.empty_like(x_in)
    k_new = torch.empty((M, hk, dh), dtype=torch.bfloat16, device=x_in.device)
    v_new = torch.empty_like(k_new)
    check(_lib.load().seed_op_decoder_layer(C.byref(sh), ptrs, _p(x_in.contiguous()), M, int(ctx_len),
                                            _p(k_prev), _p(v_prev), _p(x_out), _p(k_new), _p(v_new), _s()), None,
          "seed_op_decoder_layer")
    return x_out, k_new, v_new


def decoder_layer_tree(shape, L, x_in, ctx_len, parent, k_prev=None, v_prev=None):
    """One decoder layer over a tree of rows (parent[0] = -1, parent[i] < i): row i at position
    ctx_len + depth(i), attending to the cache and its ancestors; returns (x_out, k_new, v_new)."""
    from . import LAYER_KEYS, model_shape
    M, d = x_in.shape
    hk = shape.get("n_kv_heads", 0) or shape["n_heads"]
    dh = d // shape["n_heads"]
    ptrs = (C.c_void_p * 9)(*[L[k].data_ptr() for k in LAYER_KEYS])
    sh = model_shape(shape)
    par = np.ascontiguousarray(np.asarray(parent, dtype=np.int32))
    x_out = torch.empty_like(x_in)
    k_new = torch.empty((M, hk, dh), dtype=torch.bfloat16, device=x_in.device)
    v_new = torch.empty_like(k_new)
    check(_lib.load().seed_op_decoder_layer_tree(C.byref(sh), ptrs, _p(x_in.contiguous()), M, int(ctx_len),
                                                 par.ctypes.data_as(_lib._I32P), _p(k_prev), _p(v_prev), _p(x_out),
                                                 _p(k_new), _p(v_new), _s()), None, "seed_op_decoder_layer_tree")
    return x_out, k_new, v_new


def draft_topk(z, temperature, seed, sids, rs, node, m):
    """K1T: the m children of `node` for each row of z [B][V] fp32 CUDA -> int32 [B][m] (draw order)."""
    B, V = z.shape
    dev = z.device
    sids_t = torch.as_tensor(np.asarray(sids, dtype=np.int64).astype(np.uint32).view(np.int32), device=dev)
    rs_t = torch.as_tensor(np.asarray(rs, dtype=np.int32), device=dev)
    out = torch.empty((B, m), dtype=torch.int32, device=dev)
    check(_lib.load().seed_op_draft_topk(_p(z.contiguous()), V, B, V, float(temperature), int(seed), _p(sids_t),
                                         _p(rs_t), int(node), int(m), _p(out), int(m), 0, _s()), None,
          "seed_op_draft_topk")
    return out


def verify_tree(zt, zd, tok, counts, temperature, seed, sids, rs, bonus=True):
    """K4T: zt, zd [B][n+1][V] fp32 CUDA, tok [B][n+1] int32 CUDA, counts = k_config."""
    B, nn, V = zt.shape
    K = len(counts)
    dev = zt.device
    sids_t = torch.as_tensor(np.asarray(sids, dtype=np.int64).astype(np.uint32).view(np.int32), device=dev)
    rs_t = torch.as_tensor(np.asarray(rs, dtype=np.int32), device=dev)
    c = np.ascontiguousarray(counts, dtype=np.int32)
    out_tok = torch.empty((B, K + 1), dtype=torch.int32, device=dev)
    out_cnt = torch.empty(B, dtype=torch.int32, device=dev)
    out_node = torch.empty((B, K), dtype=torch.int32, device=dev)
    check(_lib.load().seed_op_verify_tree(_p(zt.contiguous()), _p(zd.contiguous()), _p(tok.contiguous()), B,
                                          c.ctypes.data_as(_lib._I32P), K, V, float(temperature), int(seed),
                                          _p(sids_t), _p(rs_t), int(bool(bonus)), _p(out_tok), _p(out_cnt),
                                          _p(out_node), _s()), None, "seed_op_verify_tree")
    return {"out_tok": out_tok, "out_cnt": out_cnt, "out_node": out_node}
