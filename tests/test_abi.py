"""The C-ABI library loads on a GPU-less host and exports every symbol include/gh/gh.h declares
(no compute calls here); host-side status behaviour mirrors the reference's error taxonomy."""
import ctypes as C
import re
from pathlib import Path

import pytest

import paper_2501_11779_b200 as gh
from paper_2501_11779_b200 import _lib as L

HEADER = Path(__file__).resolve().parents[1] / "include" / "gh" / "gh.h"


def declared_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(gh_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_symbols():
    syms = declared_symbols()
    assert "gh_tier2_attend" in syms and "gh_tier1_pre" in syms and len(syms) > 30


def test_every_declared_symbol_is_exported_and_bound():
    lib = gh.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} declared in gh.h but not exported by libgh.so"
        assert s in L.PROTOTYPES, f"{s} has no ctypes prototype"
    assert set(L.PROTOTYPES) <= set(declared_symbols())


def test_abi_version_and_status_names():
    lib = gh.lib()
    assert lib.gh_abi_version() == 1
    assert lib.gh_status_name(3) == b"GH_EINFEASIBLE"
    assert lib.gh_status_name(2) == b"GH_EINVAL"


def test_validation_errors_map_to_exit_code_2():
    bad = gh.TINY.with_(d_model=290)  # not divisible by n_heads
    with pytest.raises(gh.ValidationError):
        bad.validate()
    with pytest.raises(gh.ValidationError):
        gh.kv_bytes_per_prompt(gh.TINY, gh.TINY.max_seq_len + 1)


def test_unknown_model_field_rejected():
    txt = gh.TINY.to_reference_json().replace('"name"', '"rope_theta": 1.0, "name"')
    with pytest.raises(gh.ValidationError):
        gh.ModelSpec.from_json(txt)
    back = gh.ModelSpec.from_json(gh.TINY.to_reference_json(), gh.TINY.sidecar_json())
    assert back == gh.TINY


def test_create_without_device_fails_loudly():
    if gh.lib().gh_device_count() > 0:
        pytest.skip("a GPU is visible")
    from paper_2501_11779_b200.stages import Tier1
    with pytest.raises(gh.CudaError):
        Tier1(gh.TINY, max_batch=4)
