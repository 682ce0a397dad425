"""ctypes binding of the C-ABI in ``include/acco.h`` (``_acco_b200.so``).

There is no CPU fallback: if the library is missing this raises, and every
wrapper raises :class:`AccoError` when a call returns a non-zero status.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_acco_b200.so")

OK, VERIFY_FAIL, INVALID, DIVERGED, CUDA_ERROR, LOGIC_ERROR = 0, 1, 2, 3, 4, 5
DTYPE_F32, DTYPE_BF16 = 0, 1


class AccoError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[acco status {code}] {msg}")
        self.code = code


class InvalidArgument(AccoError, ValueError):
    """Status 2: the reference's std::invalid_argument."""


class LogicError(AccoError):
    """Status 5: the reference's std::logic_error."""


_lib = None


class OptCfg(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("learning_rate", C.c_double), ("adam_beta1", C.c_double),
        ("adam_beta2", C.c_double), ("adam_eps", C.c_double), ("weight_decay", C.c_double),
        ("scheduler", C.c_int), ("n_warmup_steps", C.c_int), ("total_steps", C.c_longlong),
        ("cosine_min_factor", C.c_double),
    ]


class ShardState(C.Structure):
    _fields_ = [
        ("step", C.c_longlong), ("theta", C.c_void_p), ("m", C.c_void_p), ("v", C.c_void_p),
        ("lo", C.c_uint64), ("hi", C.c_uint64),
    ]


_P = C.c_void_p
_PROTOS = {
    "acco_last_error": (C.c_char_p, []),
    "acco_launch_count": (C.c_longlong, []),
    "acco_prof_enable": (None, [C.c_int]),
    "acco_prof_reset": (C.c_int, []),
    "acco_prof_read": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "acco_version": (C.c_int, []),
    "acco_shard_partition": (C.c_int, [C.c_uint64, C.c_int, _P, _P]),
    "acco_rng_derive": (C.c_uint64, [C.c_uint64] * 5),
    "acco_sample_indices": (C.c_int, [C.c_uint64, C.c_int, C.c_int, _P]),
    "acco_scheduled_lr": (C.c_double, [C.POINTER(OptCfg), C.c_longlong]),
    "acco_opt_estimate": (C.c_int, [C.POINTER(OptCfg), C.POINTER(ShardState), _P, _P, _P, C.c_int, _P, _P]),
    "acco_opt_commit": (C.c_int, [C.POINTER(OptCfg), C.POINTER(ShardState), _P, _P, _P, _P, _P,
                                  C.c_int, _P, _P]),
    "acco_comm_unique_id": (C.c_int, [_P]),
    "acco_comm_init_rank": (C.c_int, [C.c_int, C.c_int, _P, C.c_int, C.POINTER(C.c_void_p)]),
    "acco_comm_destroy": (C.c_int, [_P]),
    "acco_comm_size": (C.c_int, [_P]),
    "acco_comm_rank": (C.c_int, [_P]),
    "acco_all_reduce_f32": (C.c_int, [_P, _P, _P, C.c_uint64, _P]),
    "acco_all_reduce_i64": (C.c_int, [_P, _P, _P, C.c_uint64, _P]),
    "acco_reduce_scatter_f32": (C.c_int, [_P, _P, _P, C.c_uint64, _P]),
    "acco_all_gather": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_int, _P]),
    "acco_pack_padded": (C.c_int, [_P, _P, C.c_uint64, C.c_int, _P]),
    "acco_unpack_padded": (C.c_int, [_P, _P, C.c_uint64, C.c_int, C.c_int, _P]),
    "acco_gemm": (C.c_int, [_P, C.c_int64, C.c_int, _P, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                            C.c_int, C.c_int, _P, C.c_int64, _P, _P, C.c_int64, _P, C.c_int64,
                            C.c_int, _P]),
    "acco_gemm_bias_grad": (C.c_int, [_P, C.c_int64, C.c_int, _P, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                      _P, C.c_int64, _P, C.c_int, _P]),
}


def lib() -> C.CDLL:
    """Load the library (built in-tree by ``build.py``); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: run `python -m paper_2406_02613_b200.build` "
            "(there is no CPU fallback for the ACCO hot path)")
    try:  # make torch's NCCL / CUDA runtime the ones the soname resolves to
        import torch  # noqa: F401
    except Exception:
        pass
    l = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    for name, (res, args) in _PROTOS.items():
        f = getattr(l, name, None)
        if f is None:
            continue  # symbol presence is checked by tests/test_capi.py against acco.h
        f.restype = res
        f.argtypes = args
    _lib = l
    return l


def register(protos: dict) -> None:
    """Add prototypes (applied now if the library is already loaded)."""
    _PROTOS.update(protos)
    if _lib is not None:
        for name, (res, args) in protos.items():
            f = getattr(_lib, name, None)
            if f is not None:
                f.restype = res
                f.argtypes = args


def check(status: int) -> None:
    if status == OK:
        return
    msg = lib().acco_last_error().decode(errors="replace")
    if status == INVALID:
        raise InvalidArgument(status, msg)
    if status == LOGIC_ERROR:
        raise LogicError(status, msg)
    raise AccoError(status, msg)


def call(name: str, *args):
    check(getattr(lib(), name)(*args))
