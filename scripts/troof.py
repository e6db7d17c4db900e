"""Round roofline of SURVEY §8(d): T_roof = sum over phases {GEMM, attention, draft, vocab} of
max(B_phase / BW, F_phase / F_peak), with the measured peaks of MEASURED_PEAKS.json (HBM copy
bandwidth; sustained bf16 for the compute-bound large-N GEMM phase).

    python scripts/troof.py [--config sweep] [--streams N] [--ctx C]

ctx defaults to the config's mean prompt length plus 20 rounds of growth at ~2 emitted tokens per
stream-round (the bench's timed window).  Prints T_roof (ms) and its phases.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seedgen


def params(sh):
    d, ff, L, V = sh["d_model"], sh["d_ff"], sh["n_layers"], sh["vocab"]
    layer = 4 * d * d + 3 * d * ff          # MHA (Hk = H): QKV + O, gate + up + down
    return L * layer + V * d, L * layer      # streamed weights (layers + LM head), layer weights


def troof(cfg_name, n=None, ctx=None, peaks=None, rows=None, draft_steps=None):
    cfg = seedgen.CONFIGS[cfg_name]
    t, dm = seedgen.SHAPES[cfg["target"]], seedgen.SHAPES[cfg["draft"]]
    g = cfg["gamma"]
    n = n or cfg["n_streams"]
    if ctx is None:
        lo, hi = cfg["prompt_len"]
        ctx = (lo + hi) / 2 + 20 * 2
    peaks = peaks or json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                 "MEASURED_PEAKS.json")))
    bw = peaks["hbm_gbs"] * 1e9
    fp = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) * 1e12
    rows = rows or g + 1            # verified positions per stream (a k_config tree: root + nodes)
    g = draft_steps or g
    M = n * rows
    Pt, _ = params(t)
    Pd, _ = params(dm)
    kv_t = 2 * t["n_layers"] * t["d_model"] * 2          # K and V, bf16, every layer, per position
    kv_d = 2 * dm["n_layers"] * dm["d_model"] * 2
    V = t["vocab"]
    gemm = max(2 * Pt / bw, 2 * Pt * M / fp)
    attn_b = n * ctx * kv_t + M * kv_t
    attn_f = 4 * t["n_layers"] * t["d_model"] * M * (ctx + g / 2 + 1)
    attn = max(attn_b / bw, attn_f / fp)
    draft_b = g * 2 * Pd + sum(n * (ctx + j) * kv_d for j in range(g))
    draft = max(draft_b / bw, 2 * Pd * n * g / fp)
    vocab = 2 * 4 * V * (M + n * g) / bw
    total = gemm + attn + draft + vocab
    return {"config": cfg_name, "streams": n, "ctx": ctx, "M": M, "t_roof_ms": total * 1e3,
            "phases_ms": {"gemm": gemm * 1e3, "attention": attn * 1e3, "draft": draft * 1e3, "vocab": vocab * 1e3}}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="sweep")
    ap.add_argument("--streams", type=int, default=0)
    ap.add_argument("--ctx", type=float, default=None)
    a = ap.parse_args()
    print(json.dumps(troof(a.config, a.streams or None, a.ctx)))
