"""Regenerate the committed golden fixtures (run in the build container, which has
/root/reference):

  python tests/golden/make_golden.py

* reference_accounting.json — values returned by the UNMODIFIED reference library
  (oracle/_ref/libtierplan_ref.so, compiled from /root/reference/proj/src) for the hot-path
  contract functions at the BASELINE configs and the reference's own test fixtures.  The CPU
  tests compare include/gh/gh.h accounting against these even where /root/reference is absent.
* rng.json — values of the synthetic generator (oracle restatement) at fixed indices.
* oracle_c1.npz — the oracle's C1 run (tiny 288x6 fp32, 4 prompts of length 8, 128 greedy
  tokens, weight seed 1234, prompt seed 5678): tokens, per-step logit statistics, and the full
  logits of prompt 0 at the first generated step.
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_2501_11779_b200 as gh  # noqa: E402
from oracle import Oracle, Ref, randn  # noqa: E402

HERE = Path(__file__).resolve().parent
GiB = 1 << 30

SPECS = {
    "tiny": gh.TINY, "llama2-7b": gh.LLAMA2_7B, "llama2-13b": gh.LLAMA2_13B, "llama2-70b": gh.LLAMA2_70B,
    "C2": gh.CONFIGS["C2"]["spec"], "C3": gh.CONFIGS["C3"]["spec"],
    "llama70b_like": gh.ModelSpec("llama2-70b-like", 80, 8192, 1024, 28672, 64, 8, 2048, 2, 32000),
    "tiny_spec": gh.ModelSpec("tiny", 1, 2, 2, 2, 1, 1, 16, 2, 0),
}


def accounting():
    out = []

    def add(fn, spec_name, args, rc_val):
        rc, val = rc_val
        out.append({"fn": fn, "spec": spec_name, "args": list(args), "rc": rc,
                    "value": list(val) if isinstance(val, (list, tuple)) else val})

    for name, s in SPECS.items():
        for seq in sorted({0, 1, min(17, s.max_seq_len), s.max_seq_len, s.max_seq_len + 1}):
            add("kv_bytes_per_prompt", name, [seq], Ref.kv_bytes_per_prompt(s, seq))
        for b in (0, 1, 64, 1190, 4096):
            add("nonattention_footprint", name, [b], Ref.nonattention_footprint(s, b))
            add("attention_footprint", name, [b, min(512, s.max_seq_len)], Ref.attention_footprint(s, b, min(512, s.max_seq_len)))
        add("weights_bytes", name, [], Ref.weights_bytes(s))
        add("payload", name, [], Ref.payload(s))
        for k in range(1, min(s.n_layers, 4) + 1):
            add("node_weight_bytes", name, [k], Ref.node_weight_bytes(s, k))
            for k2 in (1, 3, 7):
                for mem in (16 * GiB, 179 * GiB):
                    add("two_tier_context_slots", name, [k, k2, mem, s.max_seq_len],
                        Ref.two_tier_context_slots(s, k, k2, mem, s.max_seq_len))
    for n, k in ((32, 1), (32, 3), (80, 2), (6, 7), (40, 8)):
        add("layer_spans", None, [n, k], Ref.layer_spans(n, k))
    for m in (1, 2, 5, 1190, 4096):
        add("batch_grid", None, [m], Ref.batch_grid(m))
    (HERE / "reference_accounting.json").write_text(json.dumps(out, indent=1))
    print("reference_accounting.json:", len(out), "entries")


def rng():
    cases = []
    for seed, tid, start, std in ((1234, 64, 0, 1 / 64.0), (1234, 1, 12345, 1.0), (7, (1 << 40) | 5, 999, 1.0)):
        v = randn(seed, tid, start, 8, std)
        cases.append({"seed": seed, "tid": tid, "start": start, "std": std,
                      "f32_hex": [float(x).hex() for x in v]})
    (HERE / "rng.json").write_text(json.dumps(cases, indent=1))
    print("rng.json:", len(cases), "cases")


def c1():
    c = gh.CONFIGS["C1"]
    spec = c["spec"]
    prompts = np.random.default_rng(5678).integers(0, spec.vocab_size, size=(c["batch"], c["prompt_len"]),
                                                   dtype=np.int32)
    ora = Oracle(spec, seed=1234, n_slots=c["batch"])
    gen, lg = ora.generate(prompts, c["steps"])
    top2 = np.sort(lg, axis=-1)[..., -2:]
    np.savez_compressed(HERE / "oracle_c1.npz", prompts=prompts, tokens=gen,
                        logit_sum=lg.sum(-1, dtype=np.float64), logit_max=lg.max(-1),
                        margin=top2[..., 1] - top2[..., 0], logits_p0_s0=lg[0, 0])
    print("oracle_c1.npz: tokens", gen.shape, "min margin", float((top2[..., 1] - top2[..., 0]).min()))


if __name__ == "__main__":
    accounting()
    rng()
    c1()
