"""Hugging Face transformers' LlamaForCausalLM loaded with the oracle's synthetic weights.

TEST INFRASTRUCTURE ONLY (tests/ and tests/golden/make_hf_golden.py): an independent, widely used
implementation of the Llama-2 decode math the paper's model family defines, used to pin the CPU
oracle (oracle.c), whose decode arithmetic has no counterpart in /root/reference.

Mapping (oracle tensor -> transformers 5.x LlamaForCausalLM, fp32, eager attention):
  embedding (tid 1) -> model.embed_tokens; classifier (tid 2) -> lm_head;
  layer l, W_q / W_k -> self_attn.q_proj / k_proj with each head's rows reordered from the
  oracle's adjacent-pair RoPE (dims 2i, 2i+1 rotate together, P:125 / Meta's Llama) to
  transformers' half-split RoPE (dims i, i + d_h/2): new row j of a head = old row 2j (j < d_h/2)
  or 2(j - d_h/2) + 1 -- the standard Meta -> HF checkpoint permutation;
  W_v -> v_proj, W_o -> o_proj, W_1 -> mlp.gate_proj, W_3 -> mlp.up_proj, W_2 -> mlp.down_proj;
  every RMSNorm weight 1.0 (the oracle's synthetic norms), eps and rope theta from the spec.
"""
import numpy as np


def _rows_half_split(w, n_heads, dh):
    """Per head, rows (2i, 2i+1) -> (i, i + dh/2)."""
    w = w.reshape(n_heads, dh // 2, 2, -1)
    return np.ascontiguousarray(w.transpose(0, 2, 1, 3).reshape(n_heads * dh, -1))


def build_hf_llama(spec, seed: int = 1234):
    """LlamaForCausalLM (fp32, eager) holding the oracle's synthetic weights for `spec`."""
    import torch
    from transformers import LlamaConfig, LlamaForCausalLM

    from oracle import randn
    D, Dkv, Dh, H, Hkv, V = spec.d_model, spec.d_kv, spec.d_hidden, spec.n_heads, spec.n_kv_heads, spec.vocab_size
    dh = D // H
    if spec.dtype_bytes != 4:
        raise ValueError("the transformers cross-check is fp32 (the oracle rounds bf16 stage outputs, P:514)")
    cfg = LlamaConfig(vocab_size=V, hidden_size=D, intermediate_size=Dh, num_hidden_layers=spec.n_layers,
                      num_attention_heads=H, num_key_value_heads=Hkv, head_dim=dh, hidden_act="silu",
                      max_position_embeddings=spec.max_seq_len, rms_norm_eps=spec.norm_eps,
                      rope_parameters={"rope_type": "default", "rope_theta": float(spec.rope_theta)},
                      tie_word_embeddings=False, attention_bias=False, mlp_bias=False)
    cfg._attn_implementation = "eager"
    model = LlamaForCausalLM(cfg).eval().to(torch.float32)

    def w(tid, rows, cols, std):
        return randn(seed, tid, 0, rows * cols, std).reshape(rows, cols)

    sD, sH = 1.0 / np.sqrt(D), 1.0 / np.sqrt(Dh)
    sd = {"model.embed_tokens.weight": w(1, V, D, 1.0), "lm_head.weight": w(2, V, D, sD),
          "model.norm.weight": np.ones(D, np.float32)}
    for l in range(spec.n_layers):
        t = lambda k: 64 + 16 * l + k  # noqa: E731  (oracle.c tid_layer)
        p = f"model.layers.{l}."
        sd[p + "self_attn.q_proj.weight"] = _rows_half_split(w(t(0), D, D, sD), H, dh)
        sd[p + "self_attn.k_proj.weight"] = _rows_half_split(w(t(1), Dkv, D, sD), Hkv, dh)
        sd[p + "self_attn.v_proj.weight"] = w(t(2), Dkv, D, sD)
        sd[p + "self_attn.o_proj.weight"] = w(t(3), D, D, sD)
        sd[p + "mlp.gate_proj.weight"] = w(t(4), Dh, D, sD)
        sd[p + "mlp.up_proj.weight"] = w(t(5), Dh, D, sD)
        sd[p + "mlp.down_proj.weight"] = w(t(6), D, Dh, sH)
        sd[p + "input_layernorm.weight"] = np.ones(D, np.float32)
        sd[p + "post_attention_layernorm.weight"] = np.ones(D, np.float32)
    missing, unexpected = model.load_state_dict({k: torch.from_numpy(np.asarray(v, np.float32)) for k, v in sd.items()},
                                                strict=False)
    missing = [k for k in missing if "rotary_emb" not in k]
    if missing or unexpected:
        raise RuntimeError(f"state dict mismatch: missing {missing}, unexpected {unexpected}")
    return model


def hf_greedy(model, prompts, max_new):
    """Greedy decode with transformers' KV cache, token by token (the decode step the oracle
    restates).  Returns (tokens [n, max_new], logits [n, max_new, V]) for each prompt alone."""
    import torch
    toks, lgs = [], []
    with torch.no_grad():
        for p in prompts:
            ids = torch.tensor(np.asarray(p, np.int64)[None, :])
            out = model(input_ids=ids, use_cache=True)
            past, lg = out.past_key_values, out.logits[0, -1]
            t_seq, l_seq = [], []
            for i in range(max_new):
                nxt = int(torch.argmax(lg))
                t_seq.append(nxt)
                l_seq.append(lg.numpy().copy())
                if i + 1 < max_new:
                    out = model(input_ids=torch.tensor([[nxt]]), past_key_values=past, use_cache=True)
                    past, lg = out.past_key_values, out.logits[0, -1]
            toks.append(t_seq)
            lgs.append(np.stack(l_seq))
    return np.array(toks, np.int32), np.stack(lgs)
