"""Accounting restatements (include/gh/gh.h) vs the reference's own library compiled from
/root/reference (oracle/_ref) and vs the reference test-suite goldens."""
import itertools

import pytest

import paper_2501_11779_b200 as gh
from oracle import Ref, ref_available

GiB = 1 << 30
MiB = 1 << 20

LLAMA70B_LIKE = gh.ModelSpec("llama2-70b-like", 80, 8192, 1024, 28672, 64, 8, 2048, 2, 32000)  # fixtures.hpp:19-33
TINY_REF = gh.ModelSpec("tiny", 1, 2, 2, 2, 1, 1, 16, 2, 0)                                     # fixtures.hpp:35-48
SPECS = [gh.TINY, gh.LLAMA2_7B, gh.LLAMA2_13B, gh.LLAMA2_70B, LLAMA70B_LIKE, TINY_REF,
         gh.CONFIGS["C2"]["spec"], gh.CONFIGS["C3"]["spec"]]

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")


# ---------------------------------------------------------------- reference goldens
def test_kv_640MiB_anchor():           # test_model.cpp:19-23
    assert gh.kv_bytes_per_prompt(LLAMA70B_LIKE, 2048) == 640 * MiB
    assert 128 * gh.kv_bytes_per_prompt(LLAMA70B_LIKE, 2048) == 80 * GiB


def test_intra_tier_payload_16KiB():   # test_netmodel.cpp:68-76
    assert gh.payload(LLAMA70B_LIKE).intra_tier1_per_token == 16 * 1024


def test_round_trip_payload():         # test_netmodel.cpp:57-66: 2BK'(4D + 2D_kv)
    p = gh.payload(LLAMA70B_LIKE)
    B, K2 = 7, 3
    assert B * K2 * (p.tier1_to_tier2_per_token + p.tier2_to_tier1_per_token) == 2 * B * K2 * (4 * 8192 + 2 * 1024)


def test_batch_grid_to_4096():         # test_profiles.cpp:149-155
    g = gh.batch_grid(4096)
    assert g[:10] == [1, 2, 3, 4, 6, 8, 11, 16, 23, 32]
    assert g[-2:] == [2896, 4096]


def test_context_slots_linear_in_kprime():   # test_optimizer.cpp:68-72
    base = gh.two_tier_context_slots(LLAMA70B_LIKE, 2, 1, 110 * GiB, 2048)
    assert gh.two_tier_context_slots(LLAMA70B_LIKE, 2, 3, 110 * GiB, 2048) == 3 * base


def test_survey_capacity_numbers():    # SURVEY.md §0.5 [computed] at 179 GiB per B200
    c3 = gh.CONFIGS["C3"]["spec"]
    assert [gh.two_tier_context_slots(c3, 1, k, 179 * GiB, 2048) for k in (1, 3, 7)] == [170, 510, 1190]


def test_nonattention_row_oracle_discrepancy():  # footprint_oracle.hpp:7-10 / test_model.cpp:60-71
    s = LLAMA70B_LIKE
    D, Dkv, Dh = s.d_model, s.d_kv, s.d_hidden
    for B in (1, 2, 7, 64, 999):
        rows_mem = (2 * B * D + D * D) + (B * D + 2 * D * Dkv + 2 * B * Dkv) + (2 * B * D + D * D) + \
                   (B * D + 2 * D * Dh + 2 * B * Dh) + (B * Dh + Dh * D + B * D)
        assert gh.nonattention_footprint(s, B).mem_accesses == rows_mem + B * D


def test_throughput_identity():
    ts = [0, 1_000_000, 2_000_000, 3_000_000]  # 1 ms TBT
    assert gh.throughput_from(ts, 64, 2) == pytest.approx(128_000.0)


# ---------------------------------------------------------------- vs the compiled reference
@needs_ref
@pytest.mark.parametrize("spec", SPECS, ids=lambda s: s.name)
def test_against_reference_library(spec):
    assert Ref.validate(spec) == 0
    for seq in sorted({0, 1, min(17, spec.max_seq_len), spec.max_seq_len}):
        rc, v = Ref.kv_bytes_per_prompt(spec, seq)
        assert rc == 0 and v == gh.kv_bytes_per_prompt(spec, seq)
    rc, v = Ref.kv_bytes_per_prompt(spec, spec.max_seq_len + 1)
    assert rc == 2
    with pytest.raises(gh.ValidationError):
        gh.kv_bytes_per_prompt(spec, spec.max_seq_len + 1)
    for b in (0, 1, 3, 64, 1190, 4096):
        assert Ref.nonattention_footprint(spec, b) == (0, tuple(gh.nonattention_footprint(spec, b)))
        for s in (1, min(512, spec.max_seq_len), spec.max_seq_len):
            assert Ref.attention_footprint(spec, b, s) == (0, tuple(gh.attention_footprint(spec, b, s)))
    assert Ref.weights_bytes(spec) == (0, gh.weights_bytes(spec))
    assert Ref.payload(spec) == (0, tuple(gh.payload(spec)))
    for k in range(1, min(spec.n_layers, 9) + 1):
        assert Ref.node_weight_bytes(spec, k) == (0, gh.node_weight_bytes(spec, k))
        for k2, mem, seq in itertools.product((1, 3, 7), (16 * GiB, 179 * GiB), (1, spec.max_seq_len)):
            assert Ref.two_tier_context_slots(spec, k, k2, mem, seq) == \
                (0, gh.two_tier_context_slots(spec, k, k2, mem, seq))


@needs_ref
def test_layer_spans_and_grid_against_reference():
    for n, k in itertools.product((1, 6, 32, 40, 80), (1, 2, 3, 5, 7, 8)):
        if k > n:
            assert Ref.layer_spans(n, k)[0] == 2
            with pytest.raises(gh.ValidationError):
                gh.layer_spans(n, k)
        else:
            assert Ref.layer_spans(n, k) == (0, gh.layer_spans(n, k))
    for m in (1, 2, 3, 5, 100, 1024, 1190, 4096):
        assert Ref.batch_grid(m) == (0, gh.batch_grid(m))


@needs_ref
def test_error_codes_against_reference():
    assert Ref.two_tier_context_slots(gh.TINY, 1, 0, GiB, 8)[0] == 2
    with pytest.raises(gh.ValidationError):
        gh.two_tier_context_slots(gh.TINY, 1, 0, GiB, 8)
    assert Ref.two_tier_context_slots(gh.TINY, 1, 1, GiB, 0)[0] == 2
    with pytest.raises(gh.ValidationError):
        gh.two_tier_context_slots(gh.TINY, 1, 1, GiB, 0)
    assert Ref.validate(gh.TINY.with_(dtype_bytes=3)) == 2
    with pytest.raises(gh.ValidationError):
        gh.TINY.with_(dtype_bytes=3).validate()


@needs_ref
def test_throughput_identity_against_reference():
    ts = [5, 1_000_017, 2_000_001, 2_999_999, 4_100_000]
    rc, v = Ref.throughput_from(ts, 1190, 3)
    assert rc == 0 and v == gh.throughput_from(ts, 1190, 3)
