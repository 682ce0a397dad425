"""Thin torch-tensor conveniences over the raw C-ABI ops (tests, bench, tools).

torch is only the device-memory / stream plumbing here: every op dispatches to
``_acco_b200.so`` and raises if it is unavailable.
"""
from __future__ import annotations

import ctypes as C

from . import _lib

_EPI = {"store": 0, "gelu": 1, "dgelu": 2, "acc_f32": 3}


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _dtype_code(t):
    import torch

    if t.dtype == torch.bfloat16:
        return _lib.DTYPE_BF16
    if t.dtype == torch.float32:
        return _lib.DTYPE_F32
    raise TypeError(f"unsupported dtype {t.dtype}")


def gemm(a, a_mn: bool, b, b_mn: bool, m: int, n: int, k: int, c, *, mode=0, bias=None,
         residual=None, aux=None, beta=0, stream=None):
    """C[m,n] (op)= sum_k A(m,k) B(n,k); see include/acco.h acco_gemm."""
    _lib.call("acco_gemm", _ptr(a), a.stride(0), int(a_mn), _ptr(b), b.stride(0), int(b_mn),
              m, n, k, _dtype_code(a), int(_EPI.get(mode, mode)), _ptr(c), c.stride(0),
              _ptr(bias), _ptr(residual), residual.stride(0) if residual is not None else 0,
              _ptr(aux), aux.stride(0) if aux is not None else 0, int(beta), _stream(stream))


def gemm_bias_grad(a, a_mn: bool, b, b_mn: bool, m: int, n: int, k: int, c, bias_grad, *, beta=0, stream=None):
    """C[m,n] (+)= A B^T and bias_grad[m] (+)= row sums of A, bf16 operands;
    see include/acco.h acco_gemm_bias_grad."""
    _lib.call("acco_gemm_bias_grad", _ptr(a), a.stride(0), int(a_mn), _ptr(b), b.stride(0), int(b_mn),
              m, n, k, _ptr(c), c.stride(0), _ptr(bias_grad), int(beta), _stream(stream))
