"""Llama-2 forward pass, written out plainly -- TEST INFRASTRUCTURE ONLY.

The paper names checkpoints only (LLaMA-68M/160M drafts, LLaMA-2-7B/13B
targets) and gives no shapes or equations for them; R15
adopts the textbook Llama-2 definition: RMSNorm (eps 1e-5), rotary position
embedding (theta 1e4, rotate-half, 0-based positions), multi-head causal
attention with a KV cache, SwiGLU MLP, untied LM head, no biases.
Parity for this module is pinned by HF `transformers.LlamaForCausalLM` run in
float64 on the same weights (tests/test_oracle_llama.py), not by the paper.

Two modes:
  "fp64"  -- every step in fp64, no rounding (the definition).
  "bf16"  -- bf16-faithful: fp64 arithmetic, rounded to bf16 (RNE) exactly at the
             points where the CUDA path stores bf16, and to fp32 where it keeps
             fp32:
               B1 RMSNorm operand of the QKV, gate/up and LM-head GEMMs: bf16(x * w);
                  the 1/rms(x) row scale is applied to the fp32 GEMM output
                  (R24; the same linear map, rounded at another point)
               B2 Q and K after RoPE, and V (the KV cache is bf16)
               B3 attention output (operand of the O GEMM)
               B4 SwiGLU product silu(g) * u (operand of the down GEMM)
               F1 residual stream after every add (fp32)
               F2 logits (fp32)
Weights are bf16 values (seedgen) and are used exactly.
"""
from dataclasses import dataclass, field

import numpy as np
import torch


@dataclass(frozen=True)
class LlamaShape:
    vocab: int
    d_model: int
    n_layers: int
    n_heads: int
    d_ff: int
    n_kv_heads: int = 0           # 0 -> n_heads (MHA, R15)
    rms_eps: float = 1e-5
    rope_theta: float = 10000.0

    @property
    def kv_heads(self):
        return self.n_kv_heads or self.n_heads

    @property
    def head_dim(self):
        return self.d_model // self.n_heads


def bf16_round(x):
    """Round-to-nearest-even to bfloat16, returned as fp64 values."""
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    return t.to(torch.bfloat16).to(torch.float64).numpy()


def f32_round(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def _w(t):
    """bf16 torch weight -> fp64 numpy (exact)."""
    return t.to(torch.float64).numpy()


def rmsnorm(x, w, eps):
    """x * rsqrt(mean(x^2) + eps) * w  (RMSNorm, Zhang & Sennrich 2019)."""
    var = np.mean(x * x, axis=-1, keepdims=True)
    return x / np.sqrt(var + eps) * w


def rope_cos_sin(positions, head_dim, theta):
    """Rotary angles pos * theta^(-2i/d), i = 0..d/2-1, duplicated for rotate-half."""
    i = np.arange(head_dim // 2, dtype=np.float64)
    inv_freq = theta ** (-2.0 * i / head_dim)
    ang = np.asarray(positions, dtype=np.float64)[:, None] * inv_freq[None, :]
    ang = np.concatenate([ang, ang], axis=-1)
    return np.cos(ang), np.sin(ang)


def apply_rope(x, cos, sin):
    """x: [q][H][Dh]; rotate-half: x*cos + concat(-x2, x1)*sin."""
    h = x.shape[-1] // 2
    rot = np.concatenate([-x[..., h:], x[..., :h]], axis=-1)
    return x * cos[:, None, :] + rot * sin[:, None, :]


def norm_matmul(x, w, mats, eps, faithful):
    """rmsnorm(x, w) @ M^T for each M in mats.  fp64: the definition.  bf16-faithful (R24):
    (bf16(x * w) @ M^T) * 1/sqrt(mean(x^2) + eps) -- equal in exact arithmetic, since the
    row scale 1/rms(x) commutes with the matrix product."""
    if not faithful:
        h = rmsnorm(x, w, eps)
        return [h @ M.T for M in mats]
    hw = bf16_round(x * w)                                                      # B1
    inv = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return [(hw @ M.T) * inv for M in mats]


def silu(x):
    return x / (1.0 + np.exp(-x))


class KVCache:
    """Per-stream cache: K[l], V[l] arrays [len][H_kv][Dh] (fp64 values)."""

    def __init__(self, shape: LlamaShape):
        self.shape = shape
        self.k = [np.zeros((0, shape.kv_heads, shape.head_dim)) for _ in range(shape.n_layers)]
        self.v = [np.zeros((0, shape.kv_heads, shape.head_dim)) for _ in range(shape.n_layers)]

    def __len__(self):
        return self.k[0].shape[0]

    def truncate(self, n):
        """Rollback: keep the first n entries (Alg. 1 keeps only validated tokens)."""
        for layer in range(self.shape.n_layers):
            self.k[layer] = self.k[layer][:n]
            self.v[layer] = self.v[layer][:n]


def _convert_layer(L):
    return {k: _w(v) for k, v in L.items()}


def _attention(q, K, Vc, positions, grp):
    """Causal softmax attention, one query row and head at a time:
    o = softmax(q k^T / sqrt(Dh)) V over keys 0..pos (Vaswani et al. 2017)."""
    q_len, H, Dh = q.shape
    o = np.zeros((q_len, H, Dh))
    for i in range(q_len):
        n_ctx = int(positions[i]) + 1
        for hh in range(H):
            sc = K[:n_ctx, hh // grp, :] @ q[i, hh] / np.sqrt(Dh)
            sc = sc - np.max(sc)
            pr = np.exp(sc)
            pr = pr / np.sum(pr)
            o[i, hh] = pr @ Vc[:n_ctx, hh // grp, :]
    return o


def _layer(sh, Lc, x, positions, K_prev, V_prev, faithful):
    """One decoder layer (pre-norm): x += Wo attn(rope(Wq h), rope(Wk h), Wv h);
    x += Wd (silu(Wg h2) * Wu h2).  Returns (x, k_new, v_new)."""
    rb = bf16_round if faithful else (lambda a: a)
    rf = f32_round if faithful else (lambda a: a)
    H, Hk, Dh = sh.n_heads, sh.kv_heads, sh.head_dim
    q_len = x.shape[0]
    q, k, v = norm_matmul(x, Lc["attn_norm"], [Lc["wq"], Lc["wk"], Lc["wv"]], sh.rms_eps, faithful)   # B1
    q, k, v = q.reshape(q_len, H, Dh), k.reshape(q_len, Hk, Dh), v.reshape(q_len, Hk, Dh)
    cos, sin = rope_cos_sin(positions, Dh, sh.rope_theta)
    q = rb(apply_rope(q, cos, sin))                                   # B2
    k = rb(apply_rope(k, cos, sin))
    v = rb(v)
    K = np.concatenate([K_prev, k], axis=0)
    Vc = np.concatenate([V_prev, v], axis=0)
    o = rb(_attention(q, K, Vc, positions, H // Hk).reshape(q_len, H * Dh))   # B3
    x = rf(x + o @ Lc["wo"].T)                                        # F1
    g, u = norm_matmul(x, Lc["mlp_norm"], [Lc["w_gate"], Lc["w_up"]], sh.rms_eps, faithful)        # B1
    if faithful:
        g, u = rf(g), rf(u)
    act = rb(silu(g) * u)                                             # B4
    x = rf(x + act @ Lc["w_down"].T)                                  # F1
    return x, k, v


def forward_batch(shape: LlamaShape, W, seqs, mode="bf16", logits_rows=None, capture=None):
    """Forward over several streams, each with its own cache.

    seqs: list of (tokens, cache); the tokens sit at positions len(cache)...
    Appends the new K/V to each cache.  Returns a list of logits arrays
    [q_len][V] (only for rows listed in logits_rows[i] if given).
    capture: optional dict {layer: [x_in per stream]} for layer-level tests.
    Layers are the outer loop so each weight matrix is converted once.
    """
    faithful = mode == "bf16"
    rf = f32_round if faithful else (lambda a: a)
    xs, poss = [], []
    for toks, cache in seqs:
        toks = np.asarray(toks, dtype=np.int64)
        xs.append(W["embed"][torch.from_numpy(toks)].to(torch.float64).numpy())
        p0 = len(cache)
        poss.append(np.arange(p0, p0 + len(toks)))
    for layer in range(shape.n_layers):
        Lc = _convert_layer(W["layers"][layer])
        for s, (toks, cache) in enumerate(seqs):
            if capture is not None:
                capture.setdefault(layer, []).append(xs[s].copy())
            xs[s], k, v = _layer(shape, Lc, xs[s], poss[s], cache.k[layer], cache.v[layer], faithful)
            cache.k[layer] = np.concatenate([cache.k[layer], k], axis=0)
            cache.v[layer] = np.concatenate([cache.v[layer], v], axis=0)
    fn = _w(W["final_norm"])
    head = _w(W["lm_head"])
    out = []
    for s in range(len(seqs)):
        x = xs[s]
        if logits_rows is not None and logits_rows[s] is not None:
            x = x[logits_rows[s]]
        out.append(rf(norm_matmul(x, fn, [head], shape.rms_eps, faithful)[0]))   # B1, F2
    return out


def forward(shape, W, tokens, cache=None, mode="bf16"):
    """Single-stream convenience wrapper; returns logits [q_len][V]."""
    cache = cache if cache is not None else KVCache(shape)
    return forward_batch(shape, W, [(tokens, cache)], mode=mode)[0]


def layer_forward(shape, L, x, positions, k_cache, v_cache, mode="bf16"):
    """One decoder layer on hidden states x [q][d] with prior cache arrays
    [ctx][Hk][Dh]; returns (x_out, k_new, v_new).  For per-layer parity tests."""
    return _layer(shape, _convert_layer(L), np.asarray(x, dtype=np.float64), np.asarray(positions),
                  np.asarray(k_cache, dtype=np.float64), np.asarray(v_cache, dtype=np.float64),
                  mode == "bf16")
