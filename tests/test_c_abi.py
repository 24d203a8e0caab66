"""A compiled C11 consumer of include/gh/gh.h (tests/c_abi/smoke.c) linked against libgh.so: the
binding a reference-side (C / C++) maintainer would write, exercised without Python in between.

CPU: accounting + profile-CSV calls, checked against the reference's own values (recorded from
the unmodified reference library, tests/golden/reference_accounting.json) and the reference
parser's format.  GPU: the INTEGRATION.md per-layer stage sequence for BASELINE configs[0] (C1)
must reproduce the oracle's committed greedy tokens bit-exactly (tests/golden/oracle_c1.npz)."""
import json
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "c_abi" / "smoke.c"
CUDA = Path("/usr/local/cuda")


@pytest.fixture(scope="module")
def smoke_bin(tmp_path_factory):
    cc = shutil.which("cc") or shutil.which("gcc")
    if cc is None:
        pytest.skip("no C compiler")
    out = tmp_path_factory.mktemp("c_abi") / "smoke"
    libdir = ROOT / "paper_2501_11779_b200"
    cmd = [cc, "-std=c11", "-O2", "-Wall", "-Werror", "-I", str(ROOT / "include"), "-I", str(CUDA / "include"),
           str(SRC), "-o", str(out), "-L", str(libdir), "-lgh", f"-Wl,-rpath,{libdir}",
           "-L", str(CUDA / "lib64"), "-lcudart", f"-Wl,-rpath,{CUDA / 'lib64'}"]
    subprocess.run(cmd, check=True)
    return out


def test_c_consumer_accounting_and_csv(smoke_bin, tmp_path):
    import paper_2501_11779_b200 as gh
    csv = tmp_path / "b200.csv"
    r = subprocess.run([str(smoke_bin), "cpu", str(csv)], capture_output=True, text=True, check=True)
    d = json.loads(r.stdout)
    spec = gh.CONFIGS["C2"]["spec"]
    assert d["abi"] == 1
    assert d["kv_bytes_per_prompt"] == 256 << 20                       # 2*2*32*512*4096 (model.cpp:40-46)
    assert d["payload"] == [32768, 16384, 8192]                         # netmodel.cpp:18-24 at 7B
    assert (d["nonattention_mem"], d["nonattention_flops"]) == gh.nonattention_footprint(spec, 64)
    assert d["weights_bytes"] == gh.weights_bytes(spec)
    assert d["two_tier_context_slots"] == gh.two_tier_context_slots(spec, 1, 3, 179 << 30, 512)
    assert d["layer_spans"] == [40, 40]
    assert d["invalid_spec_status"] == 2                                # ValidationError, exit code 2
    golden = json.loads((ROOT / "tests" / "golden" / "reference_accounting.json").read_text())
    ref = {(e["fn"], e["spec"], tuple(e["args"])): e["value"] for e in golden}
    assert ref[("kv_bytes_per_prompt", "C2", (512,))] == d["kv_bytes_per_prompt"]
    lines = csv.read_text().splitlines()
    assert lines[0] == "device,stage,seq_len,batch_size,latency_us"     # profiles.hpp:66-69
    assert len(lines) == 7 and lines[1].startswith("b200,nonattention,512,1,")


def test_c_consumer_sched_chunked_prefill(smoke_bin):
    """gh_sched_* from C: every request equals decoding it alone, with and without chunked
    prefill, and chunking takes fewer steps when lanes are idle."""
    r = subprocess.run([str(smoke_bin), "sched"], capture_output=True, text=True, check=True)
    d = json.loads(r.stdout)
    assert d["equal"] == 1
    assert d["steps"][1] < d["steps"][0], d


@pytest.mark.gpu
def test_c_consumer_c1_tokens_bit_exact(smoke_bin, tmp_path, need_gpu):
    g = np.load(ROOT / "tests" / "golden" / "oracle_c1.npz")
    p = tmp_path / "prompts.txt"
    p.write_text("\n".join(" ".join(str(int(t)) for t in row) for row in g["prompts"]))
    r = subprocess.run([str(smoke_bin), "gpu", str(p)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    got = np.array([[int(t) for t in ln.split()] for ln in r.stdout.strip().splitlines()], np.int32)
    assert got.shape == g["tokens"].shape
    assert np.array_equal(got, g["tokens"]), np.argwhere(got != g["tokens"])[:4]
