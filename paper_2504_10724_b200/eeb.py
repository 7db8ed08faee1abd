"""ctypes binding of the C ABI in include/eeb/eeb.h (libeeb.so).

This is thin plumbing for tests and the benchmark; the product is the native
library.  There is no CPU fallback: if libeeb.so is missing or no sm_100 GPU is
present, constructing a :class:`Context` raises.

Model presets mirror BASELINE.json's configs (C1–C5) with the public
architecture dimensions listed in SURVEY.md §8; exit ladders follow the
reference fixtures (fixtures/repo_opt.json:6, fixtures/repo_large.json:6,23).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / os.environ.get("EEB_LIB", "libeeb.so")

FLAT, INTROSPECTIVE, FULL_DEPTH, PROFILE = 0, 1, 2, 3
F32, BF16 = 0, 1
MLP_RELU, MLP_SWIGLU = 0, 1

STATUS = {0: "ok", 1: "ValidationError", 2: "CapacityError", 3: "DomainError", 4: "StalenessError",
          5: "CudaError"}


class EebError(RuntimeError):
    """Raised for a non-zero eeb_status; ``kind`` names the reference exception
    type (errors.hpp:9-30) the status maps to."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS.get(code, "unknown")


class _Desc(C.Structure):
    _fields_ = [
        ("num_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
        ("n_kv_heads", C.c_int32), ("d_ffn", C.c_int32), ("vocab", C.c_int32),
        ("n_exits", C.c_int32), ("exit_layers", C.POINTER(C.c_int32)),
        ("exit_coverage", C.POINTER(C.c_float)), ("design_th", C.c_float),
        ("dtype", C.c_int32), ("mlp_kind", C.c_int32), ("max_slots", C.c_int32),
        ("max_seq_len", C.c_int32), ("seed", C.c_uint64), ("rope_theta", C.c_float),
        ("norm_eps", C.c_float), ("tp_size", C.c_int32), ("tp_rank", C.c_int32),
    ]


class _Out(C.Structure):
    _fields_ = [
        ("exit_layer", C.c_void_p), ("token_id", C.c_void_p), ("confidence", C.c_void_p),
        ("logprob", C.c_void_p), ("breached", C.c_void_p), ("unchanged", C.c_void_p),
        ("hist", C.c_void_p), ("n_breached", C.c_void_p), ("sum_logprob", C.c_void_p),
        ("head_token", C.c_void_p), ("head_confidence", C.c_void_p), ("head_logprob", C.c_void_p),
    ]


EXPORTED = [
    "eeb_abi_version", "eeb_last_error", "eeb_create", "eeb_destroy", "eeb_model_register",
    "eeb_load_layers", "eeb_evict", "eeb_loaded_depth", "eeb_weight_bytes", "eeb_reset_slots",
    "eeb_decode_step", "eeb_decode_step_device", "eeb_synchronize", "eeb_set_graphs",
    "eeb_set_gemm_tier", "eeb_debug_last_logits", "eeb_debug_retain_logits", "eeb_debug_read_weight",
    "eeb_debug_read_kv", "eeb_profile_enable", "eeb_profile_read", "eeb_stream",
    "eeb_nccl_unique_id", "eeb_nccl_init", "eeb_profile_allreduce", "eeb_debug_gemm", "eeb_debug_bench_gemm",
    "eeb_prefill", "eeb_host_stage", "eeb_load_layers_async", "eeb_load_wait",
    "eeb_kv_configure_pages", "eeb_kv_reserve", "eeb_kv_release", "eeb_kv_pages",
    "eeb_debug_stamps", "eeb_debug_stamps_read", "eeb_debug_read_kv_span",
    "eeb_weight_layout", "eeb_host_stage_layer", "eeb_host_stage_base", "eeb_load_layers_from",
    "eeb_tp_px_alloc", "eeb_tp_px_attach", "eeb_weight_reserve",
    "eeb_debug_stamps_cta",
]


class _Layout(C.Structure):
    _fields_ = [("layer_bytes", C.c_int64), ("base_bytes", C.c_int64), ("layer_off", C.c_int64 * 6),
                ("base_off", C.c_int64 * 129)]

_lib = None


def load_library() -> C.CDLL:
    """Load libeeb.so (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() first")
        lib = C.CDLL(str(LIB_PATH))
        lib.eeb_last_error.restype = C.c_char_p
        lib.eeb_stream.restype = C.c_void_p
        lib.eeb_stream.argtypes = [C.c_void_p]
        lib.eeb_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        lib.eeb_destroy.argtypes = [C.c_void_p]
        lib.eeb_model_register.argtypes = [C.c_void_p, C.POINTER(_Desc), C.POINTER(C.c_int)]
        lib.eeb_load_layers.argtypes = [C.c_void_p, C.c_int, C.c_int]
        lib.eeb_evict.argtypes = [C.c_void_p, C.c_int]
        lib.eeb_loaded_depth.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int)]
        lib.eeb_weight_bytes.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int64)]
        lib.eeb_reset_slots.argtypes = [C.c_void_p, C.c_int, C.c_int32, C.c_void_p]
        step_args = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_float, C.c_int32,
                     C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(_Out)]
        lib.eeb_decode_step.argtypes = step_args
        lib.eeb_decode_step_device.argtypes = step_args
        lib.eeb_synchronize.argtypes = [C.c_void_p]
        lib.eeb_host_stage.argtypes = [C.c_void_p, C.c_int, C.c_int]
        lib.eeb_load_layers_async.argtypes = [C.c_void_p, C.c_int, C.c_int]
        lib.eeb_load_wait.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        lib.eeb_prefill.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p]
        lib.eeb_set_graphs.argtypes = [C.c_void_p, C.c_int]
        lib.eeb_set_gemm_tier.argtypes = [C.c_void_p, C.c_int]
        lib.eeb_debug_last_logits.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
        lib.eeb_debug_retain_logits.argtypes = [C.c_void_p, C.c_int]
        lib.eeb_debug_read_weight.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int64,
                                              C.c_int64, C.c_void_p]
        lib.eeb_debug_read_kv.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_void_p, C.c_void_p]
        lib.eeb_debug_read_kv_span.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                               C.c_void_p, C.c_void_p]
        lib.eeb_debug_gemm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_void_p, C.c_void_p, C.c_void_p]
        lib.eeb_debug_bench_gemm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.POINTER(C.c_double)]
        lib.eeb_weight_layout.argtypes = [C.c_void_p, C.c_int, C.POINTER(_Layout)]
        lib.eeb_host_stage_layer.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64]
        lib.eeb_host_stage_base.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
        lib.eeb_load_layers_from.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int64]
        lib.eeb_debug_stamps_cta.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        lib.eeb_debug_stamps.argtypes = [C.c_void_p, C.c_int]
        lib.eeb_debug_stamps_read.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        lib.eeb_profile_enable.argtypes = [C.c_void_p, C.c_int]
        lib.eeb_profile_read.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        lib.eeb_nccl_unique_id.argtypes = [C.c_void_p]
        lib.eeb_nccl_init.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        lib.eeb_profile_allreduce.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
        _lib = lib
    return _lib


def _check(code: int) -> None:
    if code != 0:
        raise EebError(code, load_library().eeb_last_error().decode())


@dataclasses.dataclass
class ModelDesc:
    """↔ ModelSpec (model_spec.hpp:15-37) plus architecture dimensions."""

    name: str
    num_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    d_ffn: int
    vocab: int
    exit_layers: tuple
    exit_coverage: tuple | None = None
    design_th: float = 0.7
    dtype: int = BF16
    mlp_kind: int = MLP_RELU
    max_slots: int = 64
    max_seq_len: int = 256
    seed: int = 20260819           # fixtures/gen_calibration.json:2
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5
    tp_size: int = 1               # tensor parallelism (C5); 1 = none
    tp_rank: int = 0               # this context's shard; -1 = all shards in one context

    def replace(self, **kw) -> "ModelDesc":
        return dataclasses.replace(self, **kw)

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    def coverage(self) -> list[float]:
        if self.exit_coverage is not None:
            return list(self.exit_coverage)
        n = len(self.exit_layers)
        out = []
        for i in range(n):
            if i == n - 1:
                out.append(1.0)
            elif n <= 2 or i == 0:
                out.append(0.73)
            else:
                out.append(0.73 + 0.047 * i / (n - 2))
        return [float(np.float32(c)) for c in out]

    def to_c(self):
        layers = (C.c_int32 * len(self.exit_layers))(*self.exit_layers)
        cov = (C.c_float * len(self.exit_layers))(*self.coverage())
        d = _Desc(self.num_layers, self.d_model, self.n_heads, self.n_kv_heads, self.d_ffn, self.vocab,
                  len(self.exit_layers), C.cast(layers, C.POINTER(C.c_int32)),
                  C.cast(cov, C.POINTER(C.c_float)), self.design_th, self.dtype, self.mlp_kind,
                  self.max_slots, self.max_seq_len, self.seed, self.rope_theta, self.norm_eps,
                  self.tp_size, self.tp_rank)
        return d, (layers, cov)

    def layer_weight_elems(self) -> int:
        hd = self.head_dim
        dq, dkv = self.n_heads * hd, self.n_kv_heads * hd
        up = 2 * self.d_ffn if self.mlp_kind == MLP_SWIGLU else self.d_ffn
        return (dq + 2 * dkv) * self.d_model + self.d_model * dq + up * self.d_model + self.d_model * self.d_ffn

    @property
    def bytes_per_el(self) -> int:
        return 2 if self.dtype == BF16 else 4


PRESETS = {
    # C1: tiny decoder mirroring tiny_spec (test_model_spec.cpp:11-22): L12, exits {6, 12}.
    "tiny": ModelDesc("tiny", 12, 256, 4, 4, 1024, 512, (6, 12), dtype=F32, max_slots=8, max_seq_len=64),
    # C2: OPT-1.3B shape (d2048, 32 heads, ffn 8192, V 50272); reference exits 6/12/24.
    "opt-1.3b": ModelDesc("opt-1.3b", 24, 2048, 32, 32, 8192, 50272, (6, 12, 24)),
    # BASELINE C2 ladder 6/12/18(/24): the final layer must be an exit (model_spec.hpp:73-74).
    "opt-1.3b-4x": ModelDesc("opt-1.3b-4x", 24, 2048, 32, 32, 8192, 50272, (6, 12, 18, 24)),
    # C3 partner: OPT-2.7B shape.
    "opt-2.7b": ModelDesc("opt-2.7b", 32, 2560, 32, 32, 10240, 50272, (8, 16, 32), seed=20260820),
    # reference partner of OPT-1.3B (fixtures/repo_opt.json:21-36): exits 9/17/32.
    "opt-6.7b": ModelDesc("opt-6.7b", 32, 4096, 32, 32, 16384, 50272, (9, 17, 32), seed=20260821),
    # C4: CodeLlama-34B shape, exits 12/16/24/48 (fixtures/repo_large.json:6).
    "codellama-34b": ModelDesc("codellama-34b", 48, 8192, 64, 8, 22016, 32000, (12, 16, 24, 48),
                               mlp_kind=MLP_SWIGLU, seed=20260822),
    # C5: Llama2-70B shape, exits 8/10/20/40/80 (fixtures/repo_large.json:23).
    "llama2-70b": ModelDesc("llama2-70b", 80, 8192, 64, 8, 28672, 32000, (8, 10, 20, 40, 80),
                            mlp_kind=MLP_SWIGLU, seed=20260823),
}


def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even f32 -> bf16 bit patterns (uint16)."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def _as_dtype_bytes(t, dtype: int) -> np.ndarray:
    """f32 values -> raw bytes of the model dtype (bf16: round to nearest even)."""
    a = np.ascontiguousarray(t, np.float32).ravel()
    return (to_bf16_bits(a) if dtype == BF16 else a).view(np.uint8)


def bf16_round(a: np.ndarray) -> np.ndarray:
    return (to_bf16_bits(a).astype(np.uint32) << 16).view(np.float32)


def _i32(a) -> np.ndarray:
    if isinstance(a, np.ndarray) and a.dtype == np.int32 and a.flags.c_contiguous:
        return a
    return np.ascontiguousarray(a, dtype=np.int32)


def _addr(a: np.ndarray) -> int:
    return a.__array_interface__["data"][0]


_OUT_CACHE: dict = {}


def _out_layout(b: int, ne: int, profile: bool):
    """(field, dtype, shape, byte offset) of eeb_step_out's arrays packed into
    one buffer (8-byte aligned), in _Out field order, and the total bytes."""
    key = (b, ne, profile)
    hit = _OUT_CACHE.get(key)
    if hit is not None:
        return hit
    fields = [("exit_layer", np.int32, (b,)), ("token_id", np.int32, (b,)), ("confidence", np.float32, (b,)),
              ("logprob", np.float32, (b,)), ("breached", np.uint8, (b,)), ("unchanged", np.uint8, (b,)),
              ("hist", np.int64, (ne,)), ("n_breached", np.int64, (1,)), ("sum_logprob", np.float64, (1,))]
    if profile:
        fields += [("head_token", np.int32, (b, ne)), ("head_confidence", np.float32, (b, ne)),
                   ("head_logprob", np.float32, (b, ne))]
    spec, off = [], 0
    for name, dt, shape in fields:
        off = (off + 7) & ~7
        spec.append((name, dt, shape, off))
        off += int(np.prod(shape)) * np.dtype(dt).itemsize
    _OUT_CACHE[key] = (spec, max(off, 8))
    return _OUT_CACHE[key]


class StepResult(dict):
    """Per-row outputs of one decode step (numpy arrays)."""

    def __getattr__(self, k):
        try:
            return self[k]
        except KeyError as e:
            raise AttributeError(k) from e


class Context:
    """One eeb context (one GPU, one stream) — eeb_create / eeb_destroy."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        _check(self.lib.eeb_create(device, C.byref(h)))
        self.h = h
        self.models: dict[int, ModelDesc] = {}

    def close(self) -> None:
        if self.h:
            self.lib.eeb_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- models ---------------------------------------------------------------
    def register(self, desc: ModelDesc) -> int:
        cd, keep = desc.to_c()
        m = C.c_int()
        _check(self.lib.eeb_model_register(self.h, C.byref(cd), C.byref(m)))
        del keep
        self.models[m.value] = desc
        return m.value

    def load_layers(self, model: int, depth: int) -> None:
        _check(self.lib.eeb_load_layers(self.h, model, depth))

    def evict(self, model: int) -> None:
        _check(self.lib.eeb_evict(self.h, model))

    def loaded_depth(self, model: int) -> int:
        d = C.c_int()
        _check(self.lib.eeb_loaded_depth(self.h, model, C.byref(d)))
        return d.value

    def weight_bytes(self, model: int, depth: int) -> int:
        b = C.c_int64()
        _check(self.lib.eeb_weight_bytes(self.h, model, depth, C.byref(b)))
        return b.value

    def reset_slots(self, model: int, slots) -> None:
        s = np.ascontiguousarray(slots, dtype=np.int32)
        _check(self.lib.eeb_reset_slots(self.h, model, len(s), s.ctypes.data))

    # ---- paged KV pool (eeb_kv_configure_pages & co.) -------------------------
    def kv_configure_pages(self, model: int, page_size: int, n_pages: int) -> None:
        _check(self.lib.eeb_kv_configure_pages(self.h, model, page_size, n_pages))

    def kv_reserve(self, model: int, slot: int, n_positions: int) -> None:
        _check(self.lib.eeb_kv_reserve(self.h, model, slot, n_positions))

    def kv_release(self, model: int, slot: int) -> None:
        _check(self.lib.eeb_kv_release(self.h, model, slot))

    def kv_pages(self, model: int) -> tuple[int, int, int]:
        """(page_size, n_pages, n_free)."""
        ps, n, f = C.c_int32(), C.c_int32(), C.c_int32()
        _check(self.lib.eeb_kv_pages(self.h, model, C.byref(ps), C.byref(n), C.byref(f)))
        return ps.value, n.value, f.value

    def host_stage(self, model: int, depth: int) -> None:
        _check(self.lib.eeb_host_stage(self.h, model, depth))

    def load_layers_async(self, model: int, depth: int) -> None:
        _check(self.lib.eeb_load_layers_async(self.h, model, depth))

    def load_wait(self, model: int) -> tuple[float, int]:
        sec, nb = C.c_double(), C.c_int64()
        _check(self.lib.eeb_load_wait(self.h, model, C.byref(sec), C.byref(nb)))
        return sec.value, nb.value

    def prefill(self, model: int, depth: int, slots, prompts, start_pos=None) -> None:
        """Run each prompt (list of token arrays) through layers 1..depth into its
        KV slot (eeb_prefill); start_pos defaults to 0 per sequence."""
        sl = np.ascontiguousarray(slots, dtype=np.int32)
        lens = np.ascontiguousarray([len(p) for p in prompts], dtype=np.int32)
        sp = np.zeros(len(sl), np.int32) if start_pos is None else np.ascontiguousarray(start_pos, dtype=np.int32)
        toks = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int32) for p in prompts])
                                    if len(prompts) else np.zeros(0, np.int32), dtype=np.int32)
        if len(toks) == 0:
            toks = np.zeros(1, np.int32)
        _check(self.lib.eeb_prefill(self.h, model, depth, len(sl), sl.ctypes.data, sp.ctypes.data, lens.ctypes.data,
                                    toks.ctypes.data))

    def set_graphs(self, on: bool) -> None:
        _check(self.lib.eeb_set_graphs(self.h, 1 if on else 0))

    def set_gemm_tier(self, tier: int) -> None:
        _check(self.lib.eeb_set_gemm_tier(self.h, tier))

    # -- the step ---------------------------------------------------------------
    def decode_step(self, model: int, depth: int, policy: int, th: float, slots, tokens, positions,
                    ) -> StepResult:
        """eeb_decode_step with host buffers (H2D/D2H inside the call)."""
        desc = self.models[model]
        slots, tokens, positions = _i32(slots), _i32(tokens), _i32(positions)
        b = len(tokens)
        # every output array is a view of one fresh buffer (the library writes
        # each field it is given a pointer for): one allocation per step
        spec, total = _out_layout(b, len(desc.exit_layers), policy == PROFILE)
        buf = np.empty(total, np.uint8)
        base = buf.__array_interface__["data"][0]
        out = _Out(*[base + o for _, _, _, o in spec])
        _check(self.lib.eeb_decode_step(self.h, model, depth, policy, float(th), b, _addr(slots),
                                        _addr(tokens), _addr(positions), C.byref(out)))
        return StepResult({k: np.ndarray(shape, dt, buf, o) for k, dt, shape, o in spec})

    def decode_step_device(self, model: int, depth: int, policy: int, th: float, batch: int,
                             d_slots: int, d_tokens: int, d_positions: int, out_ptrs: dict | None = None):
        out = _Out(*[(out_ptrs or {}).get(k) for k, _ in _Out._fields_])
        _check(self.lib.eeb_decode_step_device(self.h, model, depth, policy, float(th), batch, d_slots,
                                               d_tokens, d_positions, C.byref(out)))

    def synchronize(self) -> None:
        _check(self.lib.eeb_synchronize(self.h))

    def stream(self) -> int:
        return self.lib.eeb_stream(self.h)

    # -- diagnostics ----------------------------------------------------------------
    def retain_logits(self, on: bool) -> None:
        _check(self.lib.eeb_debug_retain_logits(self.h, 1 if on else 0))

    def last_logits(self, head: int, batch: int, vocab: int) -> np.ndarray:
        a = np.zeros((batch, vocab), np.float32)
        _check(self.lib.eeb_debug_last_logits(self.h, head, a.ctypes.data, a.size))
        return a

    def read_weight(self, model: int, tensor: int, layer: int, offset: int, n: int) -> np.ndarray:
        a = np.zeros(n, np.float32)
        _check(self.lib.eeb_debug_read_weight(self.h, model, tensor, layer, offset, n, a.ctypes.data))
        return a

    def read_kv(self, model: int, layer: int, slot: int, pos: int):
        desc = self.models[model]
        k = np.zeros(desc.n_kv_heads * desc.head_dim, np.float32)
        v = np.zeros_like(k)
        _check(self.lib.eeb_debug_read_kv(self.h, model, layer, slot, pos, k.ctypes.data, v.ctypes.data))
        return k, v

    def read_kv_span(self, model: int, layer: int, slot: int, pos0: int, n_pos: int):
        """K, V of positions [pos0, pos0 + n_pos) of a slot at a layer: f32 [n_pos, Hkv * hd]."""
        desc = self.models[model]
        k = np.zeros((n_pos, desc.n_kv_heads * desc.head_dim), np.float32)
        v = np.zeros_like(k)
        _check(self.lib.eeb_debug_read_kv_span(self.h, model, layer, slot, pos0, n_pos, k.ctypes.data,
                                               v.ctypes.data))
        return k, v

    def debug_gemm(self, tier: int, w: np.ndarray, x: np.ndarray, mode: int = 0, dtype: int = BF16) -> np.ndarray:
        """One decode GEMM through a chosen tier; w [n,k], x [b,k] given as f32
        values (rounded to bf16 bit patterns when dtype is bf16)."""
        n, k = w.shape
        b = x.shape[0]
        if dtype == BF16:
            wb, xb = to_bf16_bits(w), to_bf16_bits(x)
        else:
            wb, xb = np.ascontiguousarray(w, np.float32), np.ascontiguousarray(x, np.float32)
        n_out = n // 2 if mode == 3 else n
        y = np.zeros((b, n_out), np.float32)
        _check(self.lib.eeb_debug_gemm(self.h, tier, dtype, n, k, b, mode, wb.ctypes.data, xb.ctypes.data,
                                       y.ctypes.data))
        return y

    def bench_gemm(self, tier: int, n: int, k: int, batch: int, iters: int = 50) -> float:
        """Mean ms per launch of one GEMM shape, launched back to back."""
        ms = C.c_double()
        _check(self.lib.eeb_debug_bench_gemm(self.h, tier, n, k, batch, iters, C.byref(ms)))
        return ms.value

    # -- caller-supplied weights (eeb_weight_layout / eeb_host_stage_* / eeb_load_layers_from)
    def weight_layout(self, model: int) -> dict:
        lo = _Layout()
        _check(self.lib.eeb_weight_layout(self.h, model, C.byref(lo)))
        n = len(self.models[model].exit_layers)
        return {"layer_bytes": lo.layer_bytes, "base_bytes": lo.base_bytes, "layer_off": list(lo.layer_off),
                "base_off": list(lo.base_off)[:1 + 2 * n]}

    def pack_layer(self, model: int, attn_norm, mlp_norm, wqkv, wo, wup, wdown) -> np.ndarray:
        """One layer's tensors (f32 arrays of the documented shapes) packed into
        the eeb.h host layout (norm gains f32, matrices in the model dtype)."""
        desc, lo = self.models[model], self.weight_layout(model)
        buf = np.zeros(lo["layer_bytes"], np.uint8)
        for off, t, norm in zip(lo["layer_off"], (attn_norm, mlp_norm, wqkv, wo, wup, wdown),
                                (True, True, False, False, False, False)):
            b = _as_dtype_bytes(t, 0 if norm else desc.dtype)
            buf[off:off + b.size] = b
        return buf

    def pack_base(self, model: int, embedding, heads, head_norms) -> np.ndarray:
        desc, lo = self.models[model], self.weight_layout(model)
        buf = np.zeros(lo["base_bytes"], np.uint8)
        parts = [(embedding, desc.dtype)] + [(h, desc.dtype) for h in heads] + [(g, 0) for g in head_norms]
        for off, (t, dt) in zip(lo["base_off"], parts):
            b = _as_dtype_bytes(t, dt)
            buf[off:off + b.size] = b
        return buf

    def host_stage_layer(self, model: int, layer: int, packed: np.ndarray) -> None:
        packed = np.ascontiguousarray(packed, np.uint8)
        _check(self.lib.eeb_host_stage_layer(self.h, model, layer, packed.ctypes.data, packed.size))

    def host_stage_base(self, model: int, packed: np.ndarray) -> None:
        packed = np.ascontiguousarray(packed, np.uint8)
        _check(self.lib.eeb_host_stage_base(self.h, model, packed.ctypes.data, packed.size))

    def load_layers_from(self, model: int, first: int, last: int, packed: np.ndarray) -> None:
        packed = np.ascontiguousarray(packed, np.uint8)
        _check(self.lib.eeb_load_layers_from(self.h, model, first, last, packed.ctypes.data, packed.size))

    def stamps(self, max_launches: int) -> None:
        """In-graph launch timeline of every later decode step (0 = off)."""
        _check(self.lib.eeb_debug_stamps(self.h, int(max_launches)))

    def stamps_read(self) -> list[dict]:
        """[{kernel, start_ns, end_ns, ctas}] of the last decode step, launch order."""
        import json

        n = 1 << 20
        buf = C.create_string_buffer(n)
        _check(self.lib.eeb_debug_stamps_read(self.h, buf, n))
        return json.loads(buf.value.decode())["launches"]

    def stamps_cta(self, launch: int, n: int) -> np.ndarray:
        """[n, 4] per-CTA (start, end, wait, mark) ns of one launch of the last stamped step."""
        a = np.zeros((4, n), np.int64)
        _check(self.lib.eeb_debug_stamps_cta(self.h, launch, a[0].ctypes.data, a[1].ctypes.data, a[2].ctypes.data,
                                             a[3].ctypes.data, n))
        return a.T

    def profile_enable(self, on: bool) -> None:
        _check(self.lib.eeb_profile_enable(self.h, 1 if on else 0))

    def profile_read(self) -> dict:
        import json

        buf = C.create_string_buffer(4096)
        _check(self.lib.eeb_profile_read(self.h, buf, 4096))
        return json.loads(buf.value.decode())

    # -- NCCL (replica profiling all-reduce) ----------------------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        import torch  # noqa: F401  (load torch's NCCL first; libeeb dlopens the loaded one)

        lib = load_library()
        b = (C.c_uint8 * 128)()
        _check(lib.eeb_nccl_unique_id(b))
        return bytes(b)

    def nccl_init(self, uid: bytes, nranks: int, rank: int) -> None:
        import torch  # noqa: F401

        b = (C.c_uint8 * 128)(*uid)
        _check(self.lib.eeb_nccl_init(self.h, b, nranks, rank))

    # -- peer-memory tensor parallelism ---------------------------------------------
    def tp_px_alloc(self, model: int) -> tuple[int, bytes]:
        """This rank's TP exchange buffer: (device pointer, CUDA IPC handle)."""
        ptr = C.c_void_p()
        h = (C.c_uint8 * 64)()
        _check(self.lib.eeb_tp_px_alloc(self.h, model, C.byref(ptr), h))
        return int(ptr.value), bytes(h)

    def tp_px_attach(self, model: int, nranks: int, ptrs=None, handles=None) -> None:
        """Attach every rank's exchange buffer (rank order): device pointers of
        this process (`ptrs`) or CUDA IPC handles from other processes."""
        p = (C.c_void_p * nranks)(*([int(x) if x else None for x in ptrs] if ptrs else [None] * nranks))
        hb = None
        if handles is not None:
            hb = (C.c_uint8 * (64 * nranks))(*b"".join(handles))
        _check(self.lib.eeb_tp_px_attach(self.h, model, nranks, p if ptrs else None, hb))

    def profile_allreduce(self, counters: np.ndarray, sum_neg_logprob: float) -> tuple[np.ndarray, float]:
        c = np.ascontiguousarray(counters, dtype=np.int64).copy()
        s = np.array([sum_neg_logprob], np.float64)
        _check(self.lib.eeb_profile_allreduce(self.h, c.ctypes.data, len(c), s.ctypes.data))
        return c, float(s[0])
