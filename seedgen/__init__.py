"""Seeded synthetic inputs shared by the oracle tests, smoke() and bench.py.

This module holds NO arithmetic of the method: it only draws random weights,
prompts and logits with fixed seeds.  Both the CUDA
path and the oracle receive the same tensors from here; neither imports the
other.

Recipe:
  * model shapes: public HF configs of the checkpoints the paper links
  * weights: N(0, 0.02^2) (HF initializer_range), norm weights 1, stored bf16;
    one torch.Generator per tensor, seeded from (model seed, layer, tensor id)
  * prompts: token ids uniform in [3, V) (0..2 are Llama special tokens)
  * synthetic logits for the verify-only tests: z_t ~ N(0, sigma^2),
    z_d = z_t + N(0, sigma_n^2), fp32
"""
import numpy as np
import torch

# ---- model shapes (vocab, d_model, n_layers, n_heads, d_ff) -----------------
SHAPES = {
    "toy_draft": dict(vocab=32, d_model=64, n_layers=2, n_heads=2, d_ff=256),
    "toy_target": dict(vocab=32, d_model=128, n_layers=2, n_heads=4, d_ff=512),
    "llama_68m": dict(vocab=32000, d_model=768, n_layers=2, n_heads=12, d_ff=3072),
    "llama_160m": dict(vocab=32000, d_model=768, n_layers=12, n_heads=12, d_ff=3072),
    "llama2_7b": dict(vocab=32000, d_model=4096, n_layers=32, n_heads=32, d_ff=11008),
    "llama2_13b": dict(vocab=32000, d_model=5120, n_layers=40, n_heads=40, d_ff=13824),
}

# ---- workload configs (BASELINE.json "configs"; DESIGN.md input recipe) ------
CONFIGS = {
    "toy": dict(draft="toy_draft", target="toy_target", n_streams=3, gamma=4,
                prompt_len=(8, 8), identical_prompts=True, max_new=16),
    "gsm8k": dict(draft="llama_68m", target="llama2_7b", n_streams=3, gamma=4,
                  prompt_len=(150, 450), identical_prompts=True, max_new=64),
    "cw": dict(draft="llama_68m", target="llama2_7b", n_streams=5, gamma=6,
               prompt_len=(120, 200), identical_prompts=True, max_new=256),
    "bw": dict(draft="llama_160m", target="llama2_13b", n_streams=12, gamma=5,
               prompt_len=(900, 1300), identical_prompts=False, max_new=32),
    "sweep": dict(draft="llama_68m", target="llama2_7b", n_streams=24, gamma=4,
                  prompt_len=(300, 500), identical_prompts=False, max_new=64),
}

TARGET_SEED = 1
DRAFT_SEED = 2
PROMPT_SEED = 3
PHILOX_SEED = 0x5EED2406
INIT_STD = 0.02

LAYER_TENSORS = ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down")


def _tensor_seed(model_seed, layer, idx):
    return (int(model_seed) * 1_000_003 + (layer + 1) * 10_007 + idx * 101) & 0x7FFFFFFFFFFFFFFF


def _normal(shape, seed, device, dtype):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    t = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    return (t * INIT_STD).to(dtype)


def layer_weights(shape, model_seed, layer, device="cpu", dtype=torch.bfloat16):
    d, ff = shape["d_model"], shape["d_ff"]
    hk = shape.get("n_kv_heads", 0) or shape["n_heads"]
    dkv = d // shape["n_heads"] * hk
    dims = {"wq": (d, d), "wk": (dkv, d), "wv": (dkv, d), "wo": (d, d),
            "w_gate": (ff, d), "w_up": (ff, d), "w_down": (d, ff)}
    L = {name: _normal(dims[name], _tensor_seed(model_seed, layer, i), device, dtype)
         for i, name in enumerate(LAYER_TENSORS)}
    L["attn_norm"] = torch.ones(d, device=device, dtype=dtype)
    L["mlp_norm"] = torch.ones(d, device=device, dtype=dtype)
    return L


def model_weights(shape, model_seed, device="cpu", dtype=torch.bfloat16, layers=None):
    """Full weight dict {embed, layers[l]{...}, final_norm, lm_head}.

    layers: optional iterable of layer indices to materialise (others None),
    for bounded CPU samples of the big shapes.
    """
    if isinstance(shape, str):
        shape = SHAPES[shape]
    V, d, nl = shape["vocab"], shape["d_model"], shape["n_layers"]
    want = set(range(nl)) if layers is None else set(layers)
    return {
        "embed": _normal((V, d), _tensor_seed(model_seed, -1, 0), device, dtype),
        "layers": [layer_weights(shape, model_seed, l, device, dtype) if l in want else None
                   for l in range(nl)],
        "final_norm": torch.ones(d, device=device, dtype=dtype),
        "lm_head": _normal((V, d), _tensor_seed(model_seed, -1, 1), device, dtype),
    }


def prompts(config, seed=PROMPT_SEED, n_streams=None):
    """Per-stream prompts: ids uniform in [3, V); TG configs share one prompt."""
    cfg = CONFIGS[config] if isinstance(config, str) else config
    V = SHAPES[cfg["target"]]["vocab"]
    n = n_streams or cfg["n_streams"]
    rng = np.random.default_rng(seed)
    lo, hi = cfg["prompt_len"]
    if cfg["identical_prompts"]:
        ln = int(rng.integers(lo, hi + 1))
        p = rng.integers(3, V, size=ln).tolist()
        return [list(p) for _ in range(n)]
    return [rng.integers(3, V, size=int(rng.integers(lo, hi + 1))).tolist() for _ in range(n)]


def synthetic_logits(B, gamma, V, sigma, noise, seed):
    """z_t [B][gamma+1][V], z_d [B][gamma][V] fp32 (verify-only workloads)."""
    rng = np.random.default_rng(seed)
    zt = (rng.standard_normal((B, gamma + 1, V)) * sigma).astype(np.float32)
    zd = (zt[:, :gamma, :] + rng.standard_normal((B, gamma, V)) * noise).astype(np.float32)
    return zt, zd


def hidden_states(M, d, seed, scale=1.0):
    """Residual-stream inputs for layer-level tests, fp32 [M][d]."""
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((M, d)) * scale).astype(np.float32)


def bf16_matrix(rows, cols, seed, std=1.0):
    g = torch.Generator().manual_seed(int(seed))
    return (torch.randn((rows, cols), generator=g) * std).to(torch.bfloat16)
