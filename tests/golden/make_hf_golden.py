"""Regenerate tests/golden/hf_llama_c1.npz: Hugging Face transformers' LlamaForCausalLM
(transformers 5.5.0, fp32, eager attention) holding the oracle's synthetic C1 weights
(oracle/hf_llama.py), greedy-decoding the C1 prompts (tiny 288x6, 4 prompts of length 8 from
tests/golden/oracle_c1.npz, 128 new tokens each, KV cache).

  python tests/golden/make_hf_golden.py

Records the token ids, the per-step maximum logit, and the full logits of prompt 0 at the first
generated step.  tests/test_oracle_hf.py compares the oracle against these (and, where
transformers is importable, against a live transformers run)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_2501_11779_b200 as gh  # noqa: E402
from oracle.hf_llama import build_hf_llama, hf_greedy  # noqa: E402

HERE = Path(__file__).resolve().parent

if __name__ == "__main__":
    import transformers
    c1 = np.load(HERE / "oracle_c1.npz")
    model = build_hf_llama(gh.TINY, seed=1234)
    toks, lgs = hf_greedy(model, c1["prompts"], c1["tokens"].shape[1])
    np.savez_compressed(HERE / "hf_llama_c1.npz", prompts=c1["prompts"], tokens=toks,
                        logit_max=lgs.max(-1).astype(np.float32), logits_p0_s0=lgs[0, 0].astype(np.float32),
                        transformers_version=np.array(transformers.__version__))
    same = np.array_equal(toks, c1["tokens"])
    print(f"transformers {transformers.__version__}: tokens {toks.shape}, equal to the oracle's C1 tokens: {same}; "
          f"max |logit diff| at prompt 0 step 0: {np.abs(lgs[0, 0] - c1['logits_p0_s0']).max():.3e}")
