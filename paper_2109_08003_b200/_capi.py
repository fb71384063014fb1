"""ctypes binding of ``libfnmt_b200.so`` (declared in ``include/fnmt_b200.h``).

There is no fallback: if the library is missing or fails to load, importing
anything that needs it raises ``ImportError`` with the build command.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libfnmt_b200.so"

FNMT_OK, FNMT_E_INVALID, FNMT_E_CUDA, FNMT_E_LENGTH, FNMT_E_STATE = 0, -1, -2, -3, -4
F32, F16, BF16, INT8 = 0, 1, 2, 3
DTYPES = {"f32": F32, "fp32": F32, "f16": F16, "fp16": F16, "bf16": BF16, "int8": INT8}


class fnmt_arch(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "n_enc_layers", "n_dec_layers", "d_model", "n_heads_enc", "n_heads_dec",
        "ffn_dim_enc", "ffn_dim_dec", "vocab_size", "max_positions", "norm_l1",
        "shared_embeddings")]


class fnmt_run(C.Structure):
    _fields_ = [("sbatch", C.c_int32), ("wbatch", C.c_int32), ("max_len_ratio", C.c_double),
                ("max_len_offset", C.c_int32), ("beam_size", C.c_int32), ("bos_id", C.c_int32),
                ("eos_id", C.c_int32), ("pad_id", C.c_int32)]


class fnmt_stats(C.Structure):
    _fields_ = [("sentences", C.c_int64), ("source_tokens", C.c_int64),
                ("target_tokens", C.c_int64), ("batches", C.c_int64),
                ("decode_steps", C.c_int64), ("gpu_launches", C.c_int64),
                ("encode_ms", C.c_double), ("decode_ms", C.c_double), ("total_ms", C.c_double),
                ("device_bytes", C.c_int64)]


class FnmtError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[fnmt {code}] {msg}")
        self.code = code


class FnmtLengthError(FnmtError, ValueError):
    """Mirrors the reference's LengthError (model.py:41)."""


_VP, _I, _I64, _F = C.c_void_p, C.c_int, C.c_int64, C.c_float
_SIGNATURES = {
    "fnmt_last_error": (C.c_char_p, []),
    "fnmt_version": (C.c_char_p, []),
    "fnmt_linear": (_I, [_VP, _I, _I, _VP, _I, _VP, _VP, _I, _I, _I, _I, _I, _I, _VP, _I, _VP]),
    "fnmt_linear_argmax": (_I, [_VP, _I, _I, _VP, _I, _VP, _I, _I, _I, _VP, _VP, _VP]),
    "fnmt_linear_add_norm": (_I, [_VP, _I, _I, _VP, _I, _VP, _VP, _VP, _VP, _VP, _I, _I, _I, _I,
                                  _VP]),
    "fnmt_qgemm_workspace": (_I64, [_I64, _I]),
    "fnmt_qgemm": (_I, [_VP, _I, _VP, _VP, _VP, _VP, _VP, _VP, _I, _I, _I, _I, _I, _VP, _I64,
                        _VP]),
    "fnmt_embed": (_I, [_VP, _VP, _VP, _VP, _F, _VP, _VP, _I, _I, _I, _VP]),
    "fnmt_add_norm": (_I, [_VP, _VP, _VP, _VP, _I, _VP, _VP, _I, _I, _I, _VP]),
    "fnmt_attention": (_I, [_VP, _I, _VP, _VP, _I, _VP, _I, _I, _I, _I, _VP, _VP, _VP, _VP,
                            _I, _I, _I, _I, _VP]),
    "fnmt_argmax_rows": (_I, [_VP, _I, _I, _I, _VP, _VP]),
    "fnmt_gather_rows": (_I, [_VP, _VP, _VP, _I, _I64, _I64, _I64, _VP]),
    "fnmt_engine_create": (_I, [C.POINTER(fnmt_arch), _I, _I, C.POINTER(_VP)]),
    "fnmt_engine_destroy": (None, [_VP]),
    "fnmt_engine_set_tensor": (_I, [_VP, C.c_char_p, _VP, _I64]),
    "fnmt_engine_set_qtensor": (_I, [_VP, C.c_char_p, _VP, _VP, _VP, _I64, _I64]),
    "fnmt_engine_finalize": (_I, [_VP]),
    "fnmt_engine_reserve": (_I, [_VP, C.POINTER(fnmt_run)]),
    "fnmt_budgets": (_I64, [_VP, _I, C.c_double, _I, _I, _VP]),
    "fnmt_plan_batches": (_I, [_VP, _I, _I, _I, _VP, _VP, _VP, _VP]),
    "fnmt_engine_translate": (_I, [_VP, _VP, _VP, _I, C.POINTER(fnmt_run), _VP, _VP, _VP,
                                   C.POINTER(fnmt_stats)]),
    "fnmt_engine_translate_device": (_I, [_VP, _VP, _VP, _VP, _I, C.POINTER(fnmt_run), _VP, _VP,
                                          _VP, _VP, C.POINTER(fnmt_stats)]),
    "fnmt_engine_encode_padded": (_I, [_VP, _VP, _VP, _I, _I, _VP, _VP]),
    "fnmt_engine_cross_kv": (_I, [_VP, _VP, _I, _I, _VP]),
    "fnmt_engine_decode_step": (_I, [_VP, _VP, _I, _I, _I, _VP, _VP, _VP, _VP, _VP, _I, _I,
                                     _VP]),
    "fnmt_engine_device_bytes": (_I64, [_VP]),
    "fnmt_engine_set_lanes": (_I, [_VP, _I]),
    "fnmt_engine_stream": (_VP, [_VP]),
    "fnmt_engine_profile": (_I, [_VP, _I]),
    "fnmt_engine_profile_log": (_I64, [_VP, _VP, _VP, _VP, _VP, _I64]),
    "fnmt_engine_profile_read": (_I, [_VP, _VP, _VP, _VP, _VP]),
}

KERNEL_CLASSES = ("embed", "gemm_enc", "attn_enc", "norm", "gemm_dec", "attn_dec", "vocab_argmax",
                  "search", "other")

EXPORTED = tuple(_SIGNATURES)


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (or `make -C paper_2109_08003_b200/csrc`). There is no CPU fallback.")
    lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | C.RTLD_GLOBAL)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int, what: str = "") -> int:
    if status >= 0:
        return status
    msg = lib.fnmt_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if status == FNMT_E_LENGTH:
        raise FnmtLengthError(status, msg)
    if status == FNMT_E_INVALID:
        err = FnmtError(status, msg)
        raise ValueError(str(err))
    raise FnmtError(status, msg)


def ptr(t) -> int | None:
    """Device / host address of a torch tensor or numpy array (None for None)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data
