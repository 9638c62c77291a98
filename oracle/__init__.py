"""CPU oracle for the Cubical Ripser hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product package
``paper_2005_12692_b200`` never imports it, and this package never imports the product.

The arithmetic lives in ``cr_oracle.cpp`` (plain C++, explicit boundary-matrix reduction);
this file only compiles it with g++ and marshals numpy arrays through ctypes.
See cr_oracle.cpp's header for the step-by-step citations to PAPER.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cr_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

PARTNER_ESSENTIAL = 0xFFFFFFFF
PARTNER_ABSENT = 0xFFFFFFFE


def build(force: bool = False) -> str:
    """Compile cr_oracle.cpp -> liboracle.so with g++ (no GPU needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i64p = ctypes.POINTER(ctypes.c_int64)
        vp = ctypes.c_void_p
        lib.oracle_ph.restype = ctypes.c_int64
        lib.oracle_ph.argtypes = [vp, i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  vp, vp, vp, vp, ctypes.c_int64, vp, vp]
        lib.oracle_births.restype = ctypes.c_int
        lib.oracle_births.argtypes = [vp, i64p, ctypes.c_int, vp]
        lib.oracle_ph_f64.restype = ctypes.c_int64
        lib.oracle_ph_f64.argtypes = lib.oracle_ph.argtypes
        lib.oracle_births_f64.restype = ctypes.c_int
        lib.oracle_births_f64.argtypes = lib.oracle_births.argtypes
        _lib = lib
    return _lib


def _shape_arg(shape):
    arr = (ctypes.c_int64 * len(shape))(*[int(s) for s in shape])
    return arr


def khalimsky_shape(shape):
    """(KZ, KY, KX) of the Khalimsky grid, leading sizes of 1 for 1D/2D images."""
    s = [1] * (3 - len(shape)) + [int(v) for v in shape]
    return tuple(2 * v - 1 for v in s)


def max_pairs(shape, maxdim: int) -> int:
    """Number of cells of dims 0..maxdim: an upper bound on the output size."""
    KZ, KY, KX = khalimsky_shape(shape)
    n = 0
    for Z in (0, 1):
        for Y in (0, 1):
            for X in (0, 1):
                if X + Y + Z <= maxdim:
                    n += ((KZ - Z + 1) // 2) * ((KY - Y + 1) // 2) * ((KX - X + 1) // 2)
    return n


@dataclass
class OracleResult:
    dim: np.ndarray        # int32 (M,)
    birth: np.ndarray      # float32 (M,) (float64 for ph(..., dtype=np.float64))
    death: np.ndarray      # same dtype as birth, +inf for essential classes
    cell: np.ndarray       # uint32 (M,), kidx of the birth cell
    partner: np.ndarray | None  # uint32 Khalimsky-size or None
    stats: np.ndarray      # int64 (4, 3): per dim [positive, zero-length, essential]

    def triples(self) -> np.ndarray:
        """(M,3) float64 rows (dim, birth, death) in output order (dim, birth cell)."""
        return np.stack([self.dim.astype(np.float64), self.birth.astype(np.float64),
                         self.death.astype(np.float64)], axis=1)


def ph(image: np.ndarray, maxdim: int, twist: bool = True, partner: bool = False,
       dtype=np.float32) -> OracleResult:
    """Persistence of K(image) over Z/2; see cr_oracle.cpp for the algorithm and citations.

    dtype=np.float32 (default) computes in float32 (the image is cast); np.float64 runs the same
    algorithm in double precision (oracle_ph_f64, the paper's precision PAPER.md:188)."""
    lib = _load()
    dtype = np.dtype(dtype)
    if dtype not in (np.float32, np.float64):
        raise ValueError("dtype must be float32 or float64")
    img = np.ascontiguousarray(image, dtype=dtype)
    shape = img.shape
    if img.ndim < 1 or img.ndim > 3:
        raise ValueError("ndim must be 1, 2 or 3")
    cap = max_pairs(shape, max(0, min(maxdim, 3)))
    dim = np.empty(cap, np.int32)
    birth = np.empty(cap, dtype)
    death = np.empty(cap, dtype)
    cell = np.empty(cap, np.uint32)
    part = np.empty(int(np.prod(khalimsky_shape(shape))), np.uint32) if partner else None
    stats = np.zeros(12, np.int64)
    fn = lib.oracle_ph if dtype == np.float32 else lib.oracle_ph_f64
    n = fn(img.ctypes.data, _shape_arg(shape), img.ndim, int(maxdim), int(bool(twist)),
                      dim.ctypes.data, birth.ctypes.data, death.ctypes.data, cell.ctypes.data,
                      cap, part.ctypes.data if part is not None else None, stats.ctypes.data)
    if n < 0:
        raise ValueError("oracle: invalid input (NaN, bad shape or maxdim < 0)")
    assert n <= cap
    return OracleResult(dim[:n], birth[:n], death[:n], cell[:n], part, stats.reshape(4, 3))


def births(image: np.ndarray, dtype=np.float32) -> np.ndarray:
    """Khalimsky-grid cell births (+inf = absent), shape khalimsky_shape(image.shape)."""
    lib = _load()
    dtype = np.dtype(dtype)
    img = np.ascontiguousarray(image, dtype=dtype)
    out = np.empty(khalimsky_shape(img.shape), dtype)
    fn = lib.oracle_births if dtype == np.float32 else lib.oracle_births_f64
    if fn(img.ctypes.data, _shape_arg(img.shape), img.ndim, out.ctypes.data) != 0:
        raise ValueError("oracle: invalid input")
    return out
