"""ctypes wrapper of the CPU oracle (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / reference arm, always as the checker or the CPU
baseline, never on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"
REF_LIB = HERE / "_ref" / "libeeref.so"


class _Desc(C.Structure):
    _fields_ = [
        ("num_layers", C.c_int), ("d_model", C.c_int), ("n_heads", C.c_int), ("n_kv_heads", C.c_int),
        ("d_ffn", C.c_int), ("vocab", C.c_int), ("n_exits", C.c_int), ("exit_layers", C.c_int * 64),
        ("exit_coverage", C.c_float * 64), ("design_th", C.c_float), ("dtype", C.c_int),
        ("mlp_kind", C.c_int), ("max_slots", C.c_int), ("max_seq_len", C.c_int), ("seed", C.c_uint64),
        ("rope_theta", C.c_float), ("norm_eps", C.c_float),
    ]


class _Out(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "exit_layer", "token_id", "confidence", "logprob", "breached", "unchanged", "hist",
        "n_breached", "sum_logprob", "head_token", "head_confidence", "head_logprob", "logits_out")]


class _Decision(C.Structure):
    _fields_ = [("index", C.c_int), ("exit_layer", C.c_int), ("breached", C.c_int), ("unchanged", C.c_int)]


def decide(policy: int, layers, tokens, confidences, th: float, depth: int = 0, num_layers: int | None = None):
    """The reference's per-token exit rule over one complete record (orc_decide).

    Returns (index of the observation used, exit_layer, breached, unchanged);
    raises ValueError where the reference throws DomainError."""
    layers = np.ascontiguousarray(layers, np.int32)
    tokens = np.ascontiguousarray(tokens, np.int32)
    confs = np.ascontiguousarray(confidences, np.float32)
    d = _Decision()
    rc = lib().orc_decide(policy, len(layers), layers.ctypes.data, tokens.ctypes.data, confs.ctypes.data,
                          float(th), depth, int(num_layers if num_layers is not None else layers[-1]), C.byref(d))
    if rc < 0:
        raise ValueError(lib().orc_last_error().decode())
    return d.index, d.exit_layer, bool(d.breached), bool(d.unchanged)


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.POINTER(_Desc), C.c_int]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_load.argtypes = [C.c_void_p, C.c_int]
        L.orc_alpha.restype = C.c_float
        L.orc_alpha.argtypes = [C.c_void_p, C.c_int]
        L.orc_weight.restype = C.c_float
        L.orc_weight.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int64]
        L.orc_decode_step.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_float, C.c_int, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.POINTER(_Out)]
        L.orc_read_kv.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_tensor_get.restype = C.c_int64
        L.orc_tensor_get.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64]
        L.orc_tensor_set.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64]
        L.orc_write_kv.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_fill_kv_synthetic.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64]
        L.orc_last_error.restype = C.c_char_p
        L.orc_decide.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_float, C.c_int,
                                 C.c_int, C.POINTER(_Decision)]
        _lib = L
    return _lib


class OracleModel:
    """CPU restatement of one registered model (weights, KV pool, step)."""

    def __init__(self, desc, threads: int | None = None):
        self.desc = desc
        d = _Desc()
        d.num_layers, d.d_model, d.n_heads = desc.num_layers, desc.d_model, desc.n_heads
        d.n_kv_heads, d.d_ffn, d.vocab = desc.n_kv_heads, desc.d_ffn, desc.vocab
        d.n_exits = len(desc.exit_layers)
        for i, (l, c) in enumerate(zip(desc.exit_layers, desc.coverage())):
            d.exit_layers[i] = l
            d.exit_coverage[i] = c
        d.design_th, d.dtype, d.mlp_kind = desc.design_th, desc.dtype, desc.mlp_kind
        d.max_slots, d.max_seq_len, d.seed = desc.max_slots, desc.max_seq_len, desc.seed
        d.rope_theta, d.norm_eps = desc.rope_theta, desc.norm_eps
        self.threads = threads or os.cpu_count() or 1
        self.h = lib().orc_create(C.byref(d), self.threads)
        if not self.h:
            raise MemoryError("oracle model allocation failed")

    def close(self):
        if self.h:
            lib().orc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load(self, depth: int) -> None:
        if lib().orc_load(self.h, depth) != 0:
            raise RuntimeError(lib().orc_last_error().decode())

    def alpha(self, e: int) -> float:
        return lib().orc_alpha(self.h, e)

    def weight(self, tensor: int, layer: int, index: int) -> float:
        return lib().orc_weight(self.h, tensor, layer, index)

    def decode_step(self, depth: int, policy: int, th: float, slots, tokens, positions,
                    want_logits: bool = False) -> dict:
        slots = np.ascontiguousarray(slots, np.int32)
        tokens = np.ascontiguousarray(tokens, np.int32)
        positions = np.ascontiguousarray(positions, np.int32)
        b = len(tokens)
        ne = len(self.desc.exit_layers)
        r = dict(exit_layer=np.zeros(b, np.int32), token_id=np.zeros(b, np.int32),
                 confidence=np.zeros(b, np.float32), logprob=np.zeros(b, np.float32),
                 breached=np.zeros(b, np.uint8), unchanged=np.zeros(b, np.uint8),
                 hist=np.zeros(ne, np.int64), n_breached=np.zeros(1, np.int64),
                 sum_logprob=np.zeros(1, np.float64), head_token=np.zeros((b, ne), np.int32),
                 head_confidence=np.zeros((b, ne), np.float32), head_logprob=np.zeros((b, ne), np.float32))
        if want_logits:
            r["logits_out"] = np.full((ne, b, self.desc.vocab), np.nan, np.float32)
        out = _Out(*[r[n].ctypes.data if n in r else None for n, _ in _Out._fields_])
        rc = lib().orc_decode_step(self.h, depth, policy, float(th), b, slots.ctypes.data,
                                   tokens.ctypes.data, positions.ctypes.data, C.byref(out))
        if rc != 0:
            raise RuntimeError(lib().orc_last_error().decode())
        if want_logits:
            r["logits"] = r.pop("logits_out")
        return r

    def read_kv(self, layer: int, slot: int, pos: int):
        n = self.desc.n_kv_heads * self.desc.head_dim
        k = np.zeros(n, np.float32)
        v = np.zeros(n, np.float32)
        lib().orc_read_kv(self.h, layer, slot, pos, k.ctypes.data, v.ctypes.data)
        return k, v

    def write_kv(self, layer: int, slot: int, pos0: int, k, v) -> None:
        """Import K/V rows [n, Hkv*hd] at positions pos0.. of a slot (test hook)."""
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        if lib().orc_write_kv(self.h, layer, slot, pos0, len(k), k.ctypes.data, v.ctypes.data) != 0:
            raise RuntimeError(lib().orc_last_error().decode())

    def fill_kv_synthetic(self, slot: int, n: int, seed: int = 1) -> None:
        """Synthetic full-depth KV for positions [0, n) of a slot (CPU-baseline context)."""
        if lib().orc_fill_kv_synthetic(self.h, slot, n, seed) != 0:
            raise RuntimeError(lib().orc_last_error().decode())

    def tensor(self, tensor: int, layer: int = 0) -> np.ndarray:
        """A whole weight tensor (f32 values, already on the dtype's grid)."""
        n = lib().orc_tensor_get(self.h, tensor, layer, None, 0)
        if n < 0:
            raise RuntimeError(lib().orc_last_error().decode())
        out = np.empty(n, np.float32)
        lib().orc_tensor_get(self.h, tensor, layer, out.ctypes.data, n)
        return out

    def set_tensor(self, tensor: int, layer: int, values) -> None:
        v = np.ascontiguousarray(values, np.float32).ravel()
        if lib().orc_tensor_set(self.h, tensor, layer, v.ctypes.data, v.size) != 0:
            raise RuntimeError(lib().orc_last_error().decode())
