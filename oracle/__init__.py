"""CPU oracle and compiled reference — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl reference) may
import this package, and only as the checker / the CPU baseline, never as the measured product.

* ``Oracle`` wraps liboracle.so (oracle.c): the CPU fp32 restatement of the decode step.
  The reference has no decode code to pin against (see oracle.c header); the restatement is
  pinned on the reference accounting goldens, on transformers' LlamaForCausalLM holding the same
  weights (hf_llama.py: identical C1 greedy tokens), and on tests/golden/.
* ``Ref`` wraps _ref/libtierplan_ref.so: the unmodified reference library compiled from
  /root/reference/proj/src by oracle/Makefile, plus the extern "C" shim ref_shim.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libtierplan_ref.so"
REFERENCE_ROOT = Path("/root/reference/proj")


class OrSpec(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("n_layers", "d_model", "d_kv", "d_hidden", "n_heads",
                                           "n_kv_heads", "max_seq_len", "dtype_bytes", "vocab_size")]
    _fields_ += [("rope_theta", C.c_float), ("norm_eps", C.c_float)]


def _spec(s) -> OrSpec:
    return OrSpec(s.n_layers, s.d_model, s.d_kv, s.d_hidden, s.n_heads, s.n_kv_heads, s.max_seq_len,
                  s.dtype_bytes, s.vocab_size, s.rope_theta, s.norm_eps)


def build(ref: bool | None = None) -> None:
    """Build liboracle.so (always) and _ref (when /root/reference is present)."""
    targets = ["liboracle.so"]
    if ref or (ref is None and REFERENCE_ROOT.exists()):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE)] + targets, check=True)


_olib = None


def olib() -> C.CDLL:
    global _olib
    if _olib is None:
        if not ORACLE_SO.exists():
            build(ref=False)
        L = C.CDLL(str(ORACLE_SO))
        vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
        sig = {
            "or_model_create": (vp, [C.POINTER(OrSpec), u64, u32, u32]),
            "or_model_destroy": (None, [vp]),
            "or_model_weight": (C.c_float, [vp, u32, i32, u64]),
            "or_kv_create": (vp, [C.POINTER(OrSpec), u32, u32, u32]),
            "or_kv_destroy": (None, [vp]),
            "or_kv_fill_synthetic": (None, [vp, u64, u32, u32]),
            "or_kv_read": (None, [vp, u32, u32, i32, i32, i32, vp]),
            "or_embed": (i32, [vp, i32, vp, vp]),
            "or_pre": (i32, [vp, u32, i32, vp, vp, vp]),
            "or_attend": (i32, [vp, u32, i32, vp, vp, vp, vp]),
            "or_post": (i32, [vp, u32, i32, vp, vp]),
            "or_classify": (i32, [vp, i32, vp, vp, vp]),
            "or_decode_step": (i32, [vp, vp, i32, vp, vp, vp, vp, vp]),
            "or_set_threads": (None, [i32]),
            "or_set_sum_order": (None, [i32]),
            "or_max_threads": (i32, []),
            "or_randn": (None, [u64, u64, u64, u64, C.c_double, vp]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _olib = L
    return _olib


def np_dtype(spec):
    return np.float32 if spec.dtype_bytes == 4 else np.uint16


def to_f32(a: np.ndarray) -> np.ndarray:
    """native-dtype array (fp32 or bf16 bits as uint16) -> float32"""
    if a.dtype == np.uint16:
        return (a.astype(np.uint32) << 16).view(np.float32)
    return a.astype(np.float32)


class Oracle:
    """CPU restatement of one model (layers [l0, l1)) plus its KV context."""

    def __init__(self, spec, seed: int = 1234, n_slots: int = 4, l0: int = 0, l1: int | None = None,
                 threads: int = 0):
        self.spec = spec
        self.l0, self.l1 = l0, spec.n_layers if l1 is None else l1
        L = olib()
        if threads:
            L.or_set_threads(threads)
        self.m = L.or_model_create(C.byref(_spec(spec)), seed, self.l0, self.l1)
        self.kv = L.or_kv_create(C.byref(_spec(spec)), self.l0, self.l1, n_slots)
        if not self.kv:
            raise MemoryError("oracle KV arena allocation failed")

    def close(self):
        L = olib()
        if getattr(self, "m", None):
            L.or_model_destroy(self.m)
            self.m = None
        if getattr(self, "kv", None):
            L.or_kv_destroy(self.kv)
            self.kv = None

    __del__ = close

    # native-dtype numpy buffers in the message layouts
    def buffers(self, B):
        s, dt = self.spec, np_dtype(self.spec)
        return (np.zeros((B, s.d_model), dt), np.zeros((B, 2 * s.d_model + 2 * s.d_kv), dt),
                np.zeros((B, 2 * s.d_model), dt))

    def embed(self, tok, x):
        self._rc(olib().or_embed(self.m, len(tok), _p(tok, np.int32), x.ctypes.data))

    def pre(self, layer, x, pos, fwd):
        self._rc(olib().or_pre(self.m, layer, x.shape[0], x.ctypes.data, _p(pos, np.int32), fwd.ctypes.data))

    def attend(self, layer, slot, pos, fwd, bwd):
        self._rc(olib().or_attend(self.kv, layer, fwd.shape[0], _p(slot, np.uint32), _p(pos, np.int32),
                                  fwd.ctypes.data, bwd.ctypes.data))

    def post(self, layer, bwd, x_next):
        self._rc(olib().or_post(self.m, layer, bwd.shape[0], bwd.ctypes.data, x_next.ctypes.data))

    def classify(self, x, want_logits=True):
        B = x.shape[0]
        nxt = np.zeros(B, np.int32)
        lg = np.zeros((B, self.spec.vocab_size), np.float32) if want_logits else None
        self._rc(olib().or_classify(self.m, B, x.ctypes.data, None if lg is None else lg.ctypes.data,
                                    nxt.ctypes.data))
        return nxt, lg

    def fill_synthetic(self, seed, n_fill, npos):
        olib().or_kv_fill_synthetic(self.kv, seed, n_fill, npos)

    def read_kv(self, layer, slot, kv, head, n):
        out = np.zeros((n, self.spec.d_head), np.float32)
        olib().or_kv_read(self.kv, layer, slot, kv, head, n, out.ctypes.data)
        return out

    def step(self, tok, pos, slot, want_logits=True):
        B = len(tok)
        nxt = np.zeros(B, np.int32)
        lg = np.zeros((B, self.spec.vocab_size), np.float32) if want_logits else None
        self._rc(olib().or_decode_step(self.m, self.kv, B, _p(tok, np.int32), _p(pos, np.int32),
                                       _p(slot, np.uint32), nxt.ctypes.data,
                                       None if lg is None else lg.ctypes.data))
        return nxt, lg

    def generate(self, prompts, max_new, want_logits=True):
        """Greedy decode with the same dispatcher convention as stages.Dispatcher."""
        prompts = np.asarray(prompts, np.int32)
        B, plen = prompts.shape
        slot = np.arange(B, dtype=np.uint32)
        tok = prompts[:, 0].copy()
        out, logits = [], []
        for t in range(plen - 1 + max_new):
            nxt, lg = self.step(tok, np.full(B, t, np.int32), slot, want_logits)
            if t + 1 < plen:
                tok = prompts[:, t + 1].copy()
            else:
                out.append(nxt.copy())
                if want_logits:
                    logits.append(lg)
                tok = nxt
        return np.stack(out, 1), (np.stack(logits, 1) if want_logits else None)

    @staticmethod
    def _rc(rc):
        if rc != 0:
            raise RuntimeError(f"oracle call failed with code {rc}")


def set_sum_order(order: int) -> None:
    """0 = the restatement's summation order; 1 = every fp32 reduction reversed (noise-floor
    calibration of bf16 parity tolerances, see oracle.c)."""
    olib().or_set_sum_order(order)


def randn(seed, tid, start, n, std):
    out = np.zeros(n, np.float32)
    olib().or_randn(seed, tid, start, n, std, out.ctypes.data)
    return out


def _p(a, dt):
    a = np.ascontiguousarray(a, dtype=dt)
    _keep.append(a)
    if len(_keep) > 64:
        del _keep[:32]
    return a.ctypes.data


_keep: list = []


# ------------------------------------------------------------------ compiled reference
class RefSpec(OrSpec):
    pass


_rlib = None


def ref_available() -> bool:
    return REF_SO.exists()


def rlib() -> C.CDLL:
    global _rlib
    if _rlib is None:
        if not REF_SO.exists():
            if REFERENCE_ROOT.exists():
                build(ref=True)
            else:
                raise FileNotFoundError("oracle/_ref/libtierplan_ref.so not built and /root/reference absent")
        L = C.CDLL(str(REF_SO))
        u64, vp = C.c_uint64, C.c_void_p
        P = C.POINTER
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_validate": (C.c_int, [P(OrSpec)]),
            "ref_kv_bytes_per_prompt": (C.c_int, [P(OrSpec), u64, P(u64)]),
            "ref_nonattention_footprint": (C.c_int, [P(OrSpec), u64, P(u64), P(u64)]),
            "ref_attention_footprint": (C.c_int, [P(OrSpec), u64, u64, P(u64), P(u64)]),
            "ref_weights_bytes": (C.c_int, [P(OrSpec), P(u64)]),
            "ref_payload": (C.c_int, [P(OrSpec), P(u64)]),
            "ref_layer_spans": (C.c_int, [u64, u64, P(u64)]),
            "ref_node_weight_bytes": (C.c_int, [P(OrSpec), u64, P(u64)]),
            "ref_two_tier_context_slots": (C.c_int, [P(OrSpec), u64, u64, u64, u64, P(u64)]),
            "ref_batch_grid": (C.c_int, [u64, P(u64), u64, P(u64)]),
            "ref_throughput_from": (C.c_int, [P(C.c_int64), u64, u64, u64, P(C.c_double)]),
            "ref_profile_check": (C.c_int, [C.c_char_p, P(C.c_int)]),
            "ref_profile_latency": (C.c_int, [C.c_char_p, C.c_int, u64, u64, P(C.c_int64)]),
            "ref_cmd_simulate": (C.c_int, [C.c_char_p] * 4 + [u64, u64, u64, u64, u64, C.c_char_p, u64]),
            "ref_cmd_optimize": (C.c_int, [C.c_char_p] * 4 + [u64, u64, C.c_char_p, u64]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _rlib = L
    return _rlib


class Ref:
    """Calls into the unmodified reference library; every method returns (rc, value)."""

    @staticmethod
    def err() -> str:
        return rlib().ref_last_error().decode()

    @staticmethod
    def validate(spec):
        return rlib().ref_validate(C.byref(_spec(spec)))

    @staticmethod
    def kv_bytes_per_prompt(spec, seq):
        o = C.c_uint64()
        return rlib().ref_kv_bytes_per_prompt(C.byref(_spec(spec)), seq, C.byref(o)), o.value

    @staticmethod
    def nonattention_footprint(spec, b):
        m, f = C.c_uint64(), C.c_uint64()
        return rlib().ref_nonattention_footprint(C.byref(_spec(spec)), b, C.byref(m), C.byref(f)), (m.value, f.value)

    @staticmethod
    def attention_footprint(spec, b, s):
        m, f = C.c_uint64(), C.c_uint64()
        return rlib().ref_attention_footprint(C.byref(_spec(spec)), b, s, C.byref(m), C.byref(f)), (m.value, f.value)

    @staticmethod
    def weights_bytes(spec):
        o = C.c_uint64()
        return rlib().ref_weights_bytes(C.byref(_spec(spec)), C.byref(o)), o.value

    @staticmethod
    def payload(spec):
        o = (C.c_uint64 * 3)()
        return rlib().ref_payload(C.byref(_spec(spec)), o), tuple(o)

    @staticmethod
    def layer_spans(n, k):
        o = (C.c_uint64 * max(k, 1))()
        return rlib().ref_layer_spans(n, k, o), list(o)

    @staticmethod
    def node_weight_bytes(spec, k):
        o = (C.c_uint64 * max(k, 1))()
        return rlib().ref_node_weight_bytes(C.byref(_spec(spec)), k, o), list(o)

    @staticmethod
    def two_tier_context_slots(spec, k1, k2, mem, seq):
        o = C.c_uint64()
        return rlib().ref_two_tier_context_slots(C.byref(_spec(spec)), k1, k2, mem, seq, C.byref(o)), o.value

    @staticmethod
    def batch_grid(mx):
        n = C.c_uint64()
        o = (C.c_uint64 * 64)()
        rc = rlib().ref_batch_grid(mx, o, 64, C.byref(n))
        return rc, list(o)[: n.value]

    @staticmethod
    def throughput_from(ts, batch, inflight):
        a = (C.c_int64 * len(ts))(*ts)
        o = C.c_double()
        return rlib().ref_throughput_from(a, len(ts), batch, inflight, C.byref(o)), o.value

    @staticmethod
    def profile_check(path):
        w = C.c_int()
        return rlib().ref_profile_check(str(path).encode(), C.byref(w)), w.value

    @staticmethod
    def profile_latency(path, stage, batch, seq=0):
        o = C.c_int64()
        return rlib().ref_profile_latency(str(path).encode(), stage, batch, seq, C.byref(o)), o.value

    @staticmethod
    def optimize(model, cluster, t1, t2, seq=0, max_nodes=0):
        buf = C.create_string_buffer(1 << 20)
        rc = rlib().ref_cmd_optimize(*(str(p).encode() for p in (model, cluster, t1, t2)), seq, max_nodes,
                                     buf, 1 << 20)
        return rc, buf.value.decode()

    @staticmethod
    def simulate(model, cluster, t1, t2, k1, k2, batch, seq=0, inflight=0):
        buf = C.create_string_buffer(1 << 20)
        rc = rlib().ref_cmd_simulate(*(str(p).encode() for p in (model, cluster, t1, t2)), k1, k2, batch, seq,
                                     inflight, buf, 1 << 20)
        return rc, buf.value.decode()
