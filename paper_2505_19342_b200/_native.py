"""ctypes binding of the C-ABI library (include/astra_b200.h).

There is deliberately no fallback: if the shared object is missing or was
built for another ABI, every hot-path call raises.  Status codes map to the
reference's exception taxonomy (seqvq/errors.py:4-33).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import IndexCorruptionError, MaskError, ShapeError

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libastra_b200.so"
ABI_VERSION = 2

_c_int = ctypes.c_int
_c_ll = ctypes.c_longlong
_vp = ctypes.c_void_p
_fp = ctypes.c_void_p  # float*, passed as raw device addresses

# name -> argtypes; every symbol declared in include/astra_b200.h
SIGNATURES: dict[str, list] = {
    "astra_last_error": [],
    "astra_abi_version": [],
    "astra_gemm": [_vp, _vp, _c_int, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _fp, _fp,
                   _c_int, _fp, _c_int, _vp, _vp, _c_int, _c_int, _vp],
    "astra_vq_prepare": [_vp, _vp],
    "astra_vq_encode_workspace": [_c_int, _c_int, _c_int, _c_int],
    "astra_vq_encode": [_vp, _vp, _c_int, _c_int, _vp, _vp, _vp, _vp, _c_ll, _vp],
    "astra_vq_decode": [_vp, _vp, _c_int, _vp, _c_int, _vp, _vp],
    "astra_vq_decode_layernorm": [_vp, _vp, _c_int, _vp, _vp, ctypes.c_float, _vp, _vp, _c_int,
                                  _vp, _vp],
    "astra_vq_encode_split_workspace": [_c_int, _c_int],
    "astra_vq_encode_split": [_vp, _vp, _c_int, _vp, _vp, _c_int, _vp, _c_int, _vp, _c_int, _vp,
                              _vp, _vp, _c_ll, _vp],
    "astra_vq_encode_split_ex": [_vp, _vp, _c_int, _vp, _vp, _c_int, _vp, _c_int, _vp, _c_int, _vp,
                                 _vp, _vp, _vp, _c_ll, _vp],
    "astra_layernorm_ex": [_vp, _c_int, _c_int, _c_int, _vp, _vp, ctypes.c_float, _vp, _c_int,
                           _vp, _vp, _c_int, _vp, _vp, _c_int, _vp, _vp],
    "astra_pack_indices": [_vp, _c_int, _c_int, _vp, _vp],
    "astra_unpack_indices": [_vp, _c_int, _c_int, _c_int, _vp, _vp, _vp],
    "astra_layernorm": [_vp, _c_int, _c_int, _c_int, _vp, _vp, ctypes.c_float, _vp, _c_int, _vp,
                        _vp, _c_int, _vp],
    "astra_embed_stack": [_vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _vp, _vp],
    "astra_replica_mean": [_vp, _c_int, _c_int, _c_int, _vp, _vp],
    "astra_embed_tokens": [_vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _vp, _vp],
    "astra_gather_rows": [_vp, _c_int, _vp, _c_int, _c_int, _vp, _c_int, _vp],
    "astra_key_map": [_vp, _c_int, _vp, _vp, _vp],
    "astra_key_map_packed": [_vp, _c_int, _vp, _c_int, _c_int, _c_int, _vp, _c_int, _vp, _vp, _vp],
    "astra_attention": [_vp, _c_int, _vp, _vp, _c_int, _vp, _vp, _c_int, _vp, _vp, _vp, _c_int,
                        _c_int, _c_int, _c_int, _c_int, _c_int, ctypes.c_float, _vp, _vp, _vp,
                        _c_int, _c_int, _c_int, _c_int, _vp],
    "astra_attention_force_simt": [_c_int],
    "astra_attention_variant": [_c_int],
    "astra_pdl_override": [_c_int],
    "astra_attention_trace": [_vp],
    "astra_gather_kv": [_vp, _c_int, _c_int, _c_int, _vp, _vp, _c_int, _vp, _vp, _c_int, _c_int,
                        _vp, _c_int, _vp],
    "astra_append_kv": [_vp, _vp, _c_int, _c_int, _vp, _c_int, _c_int, _vp, _c_int, _vp],
    "astra_argmax_rows": [_vp, _c_int, _c_int, _c_int, _vp, _c_int, _vp, _c_int, _vp, _vp],
    "astra_decode_advance": [_vp, _vp, _c_int, _vp],
    "astra_segment_mean_f64": [_vp, _c_int, _vp, _vp, _c_int, _c_int, _vp, _vp, _vp],
    "astra_attention_masked": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp,
                               _vp],
}
_RESTYPES = {"astra_last_error": ctypes.c_char_p, "astra_vq_encode_workspace": ctypes.c_longlong,
             "astra_vq_encode_split_workspace": ctypes.c_longlong}

_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def lib_path() -> Path:
    return Path(os.environ.get("ASTRA_B200_LIB", _LIB_PATH))


def load():
    """Load (once) and type the native library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not path.exists():
        raise NativeLibraryMissing(
            f"native library {path} not built; run `python -m paper_2505_19342_b200.build`")
    lib = ctypes.CDLL(str(path))
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    if lib.astra_abi_version() != ABI_VERSION:
        raise NativeLibraryMissing("native library ABI mismatch; rebuild it")
    if os.environ.get("ASTRA_ATTN_VARIANT"):   # A/B hook: attention kernel variant
        lib.astra_attention_variant(int(os.environ["ASTRA_ATTN_VARIANT"]))
    _lib = lib
    return lib


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    msg = (_lib.astra_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == 1:
        raise ShapeError(text)
    if status == 2:
        raise IndexCorruptionError(text)
    if status == 5:
        raise MaskError(text)
    raise RuntimeError(text)


# kernels each C-ABI call enqueues (for launch accounting in bench.py)
LAUNCHES = {"astra_vq_encode": 3, "astra_vq_prepare": 2, "astra_vq_encode_split": 3,
            "astra_vq_encode_split_ex": 3}
_counter: dict | None = None


def count_launches(enable: bool) -> dict | None:
    """Start (enable=True) or stop counting native kernel launches; returns the tally."""
    global _counter
    out = _counter
    _counter = {} if enable else None
    return out


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args), name)
    if _counter is not None:
        _counter[name] = _counter.get(name, 0) + LAUNCHES.get(name, 1)
