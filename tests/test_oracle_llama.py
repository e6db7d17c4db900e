"""Oracle pins for the Llama-2 forward (DESIGN R15; the paper fixes no shapes).

Pinned by an independent library forward: HF transformers LlamaForCausalLM in
float64 on the same weights.  HF keeps RMSNorm and the rotary table in fp32
even in a float64 model, so the bound is 1e-4 relative -- a dropped term, a
sign or a transposed operand moves logits by O(1).
"""
import numpy as np
import pytest
import torch

import seedgen
from oracle import llama as ll


def _shape(name):
    return ll.LlamaShape(**seedgen.SHAPES[name])


def _hf_model(shape, W):
    from transformers import LlamaConfig, LlamaForCausalLM
    cfg = LlamaConfig(vocab_size=shape.vocab, hidden_size=shape.d_model, intermediate_size=shape.d_ff,
                      num_hidden_layers=shape.n_layers, num_attention_heads=shape.n_heads,
                      num_key_value_heads=shape.kv_heads, rms_norm_eps=shape.rms_eps,
                      rope_theta=shape.rope_theta, max_position_embeddings=256,
                      attention_bias=False, mlp_bias=False, tie_word_embeddings=False,
                      hidden_act="silu")
    cfg._attn_implementation = "eager"
    m = LlamaForCausalLM(cfg).to(torch.float64).eval()
    sd = {"model.embed_tokens.weight": W["embed"], "model.norm.weight": W["final_norm"],
          "lm_head.weight": W["lm_head"]}
    names = {"wq": "self_attn.q_proj", "wk": "self_attn.k_proj", "wv": "self_attn.v_proj",
             "wo": "self_attn.o_proj", "w_gate": "mlp.gate_proj", "w_up": "mlp.up_proj",
             "w_down": "mlp.down_proj", "attn_norm": "input_layernorm",
             "mlp_norm": "post_attention_layernorm"}
    for i, L in enumerate(W["layers"]):
        for k, v in L.items():
            sd[f"model.layers.{i}.{names[k]}.weight"] = v
    sd = {k: v.to(torch.float64) for k, v in sd.items()}
    missing, unexpected = m.load_state_dict(sd, strict=False)
    assert not unexpected and all("rotary" in k for k in missing), (missing, unexpected)
    return m


@pytest.mark.parametrize("name", ["toy_target", "toy_draft"])
def test_fp64_forward_matches_hf_llama(name):
    shape = _shape(name)
    W = seedgen.model_weights(seedgen.SHAPES[name], 11)
    # larger init so the logits are O(1) and any structural error is visible
    for L in W["layers"]:
        for k in ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down"):
            L[k] = (L[k].float() * 10).to(torch.bfloat16)
    W["lm_head"] = (W["lm_head"].float() * 10).to(torch.bfloat16)
    toks = [5, 17, 3, 30, 12, 9, 9, 21, 4, 8, 1, 2]
    ours = ll.forward(shape, W, toks, mode="fp64")
    m = _hf_model(shape, W)
    with torch.no_grad():
        ref = m(torch.tensor([toks])).logits[0].numpy()
    scale = np.max(np.abs(ref))
    assert scale > 0.5
    assert np.max(np.abs(ours - ref)) / scale < 1e-4


def test_cached_decode_equals_full_forward():
    shape = _shape("toy_target")
    W = seedgen.model_weights(seedgen.SHAPES["toy_target"], 12)
    toks = list(range(3, 23))
    full = ll.forward(shape, W, toks, mode="fp64")
    cache = ll.KVCache(shape)
    parts = [toks[:7], toks[7:8], toks[8:13], toks[13:]]
    outs = [ll.forward(shape, W, p, cache=cache, mode="fp64") for p in parts]
    np.testing.assert_allclose(np.concatenate(outs), full, rtol=0, atol=1e-12)
    # rollback then re-feed gives the same rows (KV rollback invariant)
    cache.truncate(10)
    again = ll.forward(shape, W, toks[10:], cache=cache, mode="fp64")
    np.testing.assert_allclose(again, full[10:], rtol=0, atol=1e-12)


def test_bf16_mode_close_to_fp64():
    shape = _shape("toy_target")
    W = seedgen.model_weights(seedgen.SHAPES["toy_target"], 13)
    toks = list(range(3, 15))
    a = ll.forward(shape, W, toks, mode="fp64")
    b = ll.forward(shape, W, toks, mode="bf16")
    rel = np.max(np.abs(a - b), axis=1) / np.max(np.abs(a), axis=1)
    assert np.all(rel < 2e-2) and np.any(rel > 0)


def test_bf16_round_is_rne():
    one = 1.0
    assert ll.bf16_round(np.array([one + 2.0 ** -8]))[0] == 1.0               # tie -> even
    assert ll.bf16_round(np.array([one + 3 * 2.0 ** -8]))[0] == 1.0 + 2.0 ** -6  # tie -> even (up)
    assert ll.bf16_round(np.array([one + 2.0 ** -8 + 2.0 ** -12]))[0] == 1.0 + 2.0 ** -7


def test_layer_forward_matches_forward_batch():
    shape = _shape("toy_target")
    W = seedgen.model_weights(seedgen.SHAPES["toy_target"], 14)
    toks = list(range(3, 12))
    cap = {}
    cache = ll.KVCache(shape)
    ll.forward_batch(shape, W, [(toks[:5], cache)], mode="bf16")
    ll.forward_batch(shape, W, [(toks[5:], cache)], mode="bf16", capture=cap)
    x0 = cap[0][0]
    x1, k, v = ll.layer_forward(shape, W["layers"][0], x0, np.arange(5, 9), cache.k[0][:5], cache.v[0][:5])
    np.testing.assert_array_equal(x1, cap[1][0])
    np.testing.assert_array_equal(k, cache.k[0][5:])
