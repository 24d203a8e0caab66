"""Pinning the CPU oracle's decode math against an independent implementation: Hugging Face
transformers' LlamaForCausalLM (transformers 5.5.0, fp32, eager attention, KV-cache greedy decode)
holding the oracle's synthetic weights (oracle/hf_llama.py).  The reference repository has no
decode code; Llama-2 is the model family the paper evaluates (Table 8), and
transformers' Llama is its de-facto public definition.

* the committed fixture tests/golden/hf_llama_c1.npz (tests/golden/make_hf_golden.py): C1 (tiny
  288x6 fp32, 4 prompts x 128 greedy tokens) -- the 512 token ids must equal the oracle's C1
  golden tokens (which the GPU engine reproduces bit-exactly, tests/test_gpu_engine.py);
* live, where transformers is importable: MHA and GQA fp32 shapes, tokens equal and logits
  within 2e-5 x max|logit| (fp32, different summation order)."""
from pathlib import Path

import numpy as np
import pytest

import paper_2501_11779_b200 as gh
from oracle import Oracle

GOLD = Path(__file__).resolve().parent / "golden"


def test_hf_golden_tokens_equal_oracle_c1():
    hf = np.load(GOLD / "hf_llama_c1.npz")
    c1 = np.load(GOLD / "oracle_c1.npz")
    assert np.array_equal(hf["prompts"], c1["prompts"])
    assert hf["tokens"].shape == (4, 128)
    assert np.array_equal(hf["tokens"], c1["tokens"])
    lg_o, lg_h = c1["logits_p0_s0"], hf["logits_p0_s0"]
    assert np.abs(lg_o - lg_h).max() <= 2e-5 * np.abs(lg_o).max()


def test_oracle_c1_first_steps_equal_hf_golden():
    """The live oracle (not only its committed fixture) against the transformers tokens."""
    hf = np.load(GOLD / "hf_llama_c1.npz")
    ora = Oracle(gh.TINY, n_slots=4)
    toks, lg = ora.generate(hf["prompts"], 16)
    ora.close()
    assert np.array_equal(toks, hf["tokens"][:, :16])
    assert np.abs(lg[0, 0] - hf["logits_p0_s0"]).max() <= 2e-5 * np.abs(hf["logits_p0_s0"]).max()


@pytest.mark.parametrize("spec", [
    gh.TINY.with_(n_layers=2, max_seq_len=64),
    gh.ModelSpec("gqa-fp32", 2, 256, 64, 512, 8, 2, 64, 4, 1000),
])
def test_oracle_matches_transformers_llama(spec):
    pytest.importorskip("transformers")
    from oracle.hf_llama import build_hf_llama, hf_greedy
    prompts = np.random.default_rng(1).integers(0, spec.vocab_size, size=(3, 5)).astype(np.int32)
    ht, hl = hf_greedy(build_hf_llama(spec), prompts, 12)
    ora = Oracle(spec, n_slots=1)
    for i, p in enumerate(prompts):
        t, lg = ora.generate(p[None, :], 12)
        assert np.array_equal(t[0], ht[i])
        assert np.abs(lg[0] - hl[i]).max() <= 2e-5 * np.abs(lg[0]).max()
    ora.close()
