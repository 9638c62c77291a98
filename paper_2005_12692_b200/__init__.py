"""paper_2005_12692_b200 -- B200-native Cubical Ripser hot path (arXiv 2005.12692).

Thin Python binding over the C ABI of ``libcr.so`` (include/cr.h).  This module only marshals
arguments: every step of the computation runs in the sm_100a CUDA kernels behind the ABI.
PyTorch provides device memory and the current stream.  There is no CPU fallback: if the
library is missing or fails to load, importing this package raises.

Public names mirror the ABI: ``barcodes``, ``barcodes_host``, ``barcodes_batched``, ``pairing``,
``max_pairs``, ``num_cells``, ``last_stats``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcr.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libcr.so not built ({LIB_PATH}); run `python -m paper_2005_12692_b200.build` "
                      "or __graft_entry__.build()")
_lib = ctypes.CDLL(LIB_PATH)

CR_OK, CR_EINVAL, CR_ERANGE, CR_ENOMEM, CR_ECUDA, CR_EINTERNAL = 0, -1, -2, -3, -4, -5
PARTNER_ESSENTIAL = 0xFFFFFFFF
PARTNER_ABSENT = 0xFFFFFFFE

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i64p = ctypes.POINTER(ctypes.c_int64)


class CrStats(ctypes.Structure):
    _fields_ = [("cells", _i64 * 4), ("apparent", _i64 * 4), ("columns", _i64 * 4),
                ("rounds", _i64 * 4), ("pairs", _i64 * 4), ("essential", _i64 * 4),
                ("path", _i64), ("nstages", ctypes.c_int32), ("stage_ms", ctypes.c_float * 16),
                ("stage_name", (ctypes.c_char * 24) * 16), ("launches", _i64),
                ("additions", _i64 * 4), ("addlen", _i64 * 4), ("maxlen", _i64 * 4),
                ("kf_tma", _i64)]

    def as_dict(self):
        d = {f: list(getattr(self, f)) for f in ("cells", "apparent", "columns", "rounds", "pairs",
                                                  "essential", "additions", "addlen", "maxlen")}
        d["path"] = int(self.path)
        d["launches"] = int(self.launches)
        d["kf_tma"] = int(self.kf_tma)
        d["stages"] = {self.stage_name[i].value.decode(): float(self.stage_ms[i])
                       for i in range(int(self.nstages))}
        return d


_lib.cr_barcodes.restype = ctypes.c_int
_lib.cr_barcodes.argtypes = [_vp, _i64p, ctypes.c_int, ctypes.c_int, _vp, _vp, _i64, _i64p, _vp]
_lib.cr_barcodes_host.restype = ctypes.c_int
_lib.cr_barcodes_host.argtypes = [_vp, _i64p, ctypes.c_int, ctypes.c_int, _vp, _vp, _i64, _i64p, _vp]
_lib.cr_barcodes_batched.restype = ctypes.c_int
_lib.cr_barcodes_batched.argtypes = [_vp, _i64, _i64p, ctypes.c_int, ctypes.c_int, _vp, _vp, _i64,
                                     _vp, _i64p, _vp]
_lib.cr_barcodes_batched_host.restype = ctypes.c_int
_lib.cr_barcodes_batched_host.argtypes = [_vp, _i64, _i64p, ctypes.c_int, ctypes.c_int, _vp, _vp,
                                          _i64, _vp, _i64p, _vp]
_lib.cr_barcodes_topdim.restype = ctypes.c_int
_lib.cr_barcodes_topdim.argtypes = [_vp, _i64p, ctypes.c_int, _vp, _vp, _i64, _i64p, _vp]
_lib.cr_death_cells.restype = ctypes.c_int
_lib.cr_barcodes_f64.argtypes = [_vp, _i64p, ctypes.c_int, ctypes.c_int, _vp, _vp, _i64, _i64p, _vp]
_lib.cr_barcodes_f64.restype = ctypes.c_int
_lib.cr_death_cells.argtypes = [_vp, _i64p, ctypes.c_int, _vp, _i64, _vp, _vp]
_lib.cr_lifetime_image.restype = ctypes.c_int
_lib.cr_lifetime_image.argtypes = [_vp, _i64, _i64p, ctypes.c_int, ctypes.c_int, ctypes.c_float,
                                   _vp, _vp]
_lib.cr_pairing.restype = ctypes.c_int
_lib.cr_pairing.argtypes = [_vp, _i64p, ctypes.c_int, _vp, _vp]
_lib.cr_max_pairs.restype = _i64
_lib.cr_max_pairs.argtypes = [_i64p, ctypes.c_int, ctypes.c_int]
_lib.cr_num_cells.restype = _i64
_lib.cr_num_cells.argtypes = [_i64p, ctypes.c_int]
_lib.cr_status_string.restype = ctypes.c_char_p
_lib.cr_status_string.argtypes = [ctypes.c_int]
_lib.cr_last_stats.restype = None
_lib.cr_last_stats.argtypes = [ctypes.POINTER(CrStats)]
_lib.cr_set_profiling.restype = None
_lib.cr_set_profiling.argtypes = [ctypes.c_int]
_lib.cr_release_workspace.restype = None
_lib.cr_release_workspace.argtypes = []
_lib.cr_workspace_bytes.restype = _i64
_lib.cr_workspace_bytes.argtypes = []
_lib.cr_set_option.restype = ctypes.c_int
_lib.cr_set_option.argtypes = [ctypes.c_int, _i64]

EXPORTED = ["cr_barcodes", "cr_barcodes_host", "cr_barcodes_batched", "cr_pairing", "cr_max_pairs",
            "cr_num_cells", "cr_status_string", "cr_last_stats", "cr_set_profiling",
            "cr_death_cells", "cr_lifetime_image", "cr_barcodes_topdim", "cr_barcodes_f64",
            "cr_set_option", "cr_barcodes_batched_host", "cr_release_workspace",
            "cr_workspace_bytes"]

# cr_option (include/cr.h): validation / measurement switches, 0 = the product path
OPTIONS = {"force_general": 1, "1d_tree": 2, "top_reduce": 3, "k5_blocks_per_sm": 4,
           "k5_jitter_ns": 5, "debug": 6, "kf_tma": 7, "kf_rcap": 8}


class CrError(RuntimeError):
    def __init__(self, status: int):
        self.status = status
        super().__init__(f"cr status {status}: {_lib.cr_status_string(status).decode()}")


_SHAPE_T = [ctypes.c_int64 * k for k in range(4)]


def _shape(shape):
    return _SHAPE_T[len(shape)](*shape) if len(shape) < 4 else (ctypes.c_int64 * len(shape))(*shape)


def _check(st):
    if st != CR_OK:
        raise CrError(st)


def max_pairs(shape, maxdim: int) -> int:
    n = _lib.cr_max_pairs(_shape(shape), len(shape), int(maxdim))
    if n < 0:
        raise CrError(CR_EINVAL)
    return int(n)


def num_cells(shape) -> int:
    n = _lib.cr_num_cells(_shape(shape), len(shape))
    if n < 0:
        raise CrError(CR_EINVAL)
    return int(n)


def set_profiling(enable: bool) -> None:
    """Per-stage CUDA-event timing of subsequent calls on this thread (see cr_set_profiling)."""
    _lib.cr_set_profiling(1 if enable else 0)


def release_workspace() -> None:
    """Return this thread's cached device workspace to the driver (cr_release_workspace)."""
    _lib.cr_release_workspace()


def workspace_bytes() -> int:
    """Device bytes held by this thread's workspace cache (cr_workspace_bytes)."""
    return int(_lib.cr_workspace_bytes())


def set_option(name: str, value: int) -> None:
    """cr_set_option for this host thread (see OPTIONS)."""
    _check(_lib.cr_set_option(OPTIONS[name], int(value)))


class options:
    """``with cr.options(top_reduce=1): ...`` sets options for the block, then restores 0."""

    def __init__(self, **kw):
        self.kw = kw

    def __enter__(self):
        for k, v in self.kw.items():
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k in self.kw:
            set_option(k, 0)
        return False


def last_stats() -> dict:
    s = CrStats()
    _lib.cr_last_stats(ctypes.byref(s))
    return s.as_dict()


@dataclass
class Barcode:
    """Bars ordered by (dim, birth cell kidx).  ``pairs`` is the raw (M,3) int32 buffer of
    cr_pair {int32 dim; float birth; float death}."""
    pairs: "object"           # torch int32 (M,3) or numpy
    cells: "object | None"    # uint32 (as int32 storage) kidx of birth cells, or None

    @property
    def dim(self):
        return self.pairs[:, 0]

    @property
    def birth(self):
        return self.pairs[:, 1].view(_float_dtype(self.pairs))

    @property
    def death(self):
        return self.pairs[:, 2].view(_float_dtype(self.pairs))

    def numpy(self):
        p = self.pairs.cpu().numpy() if hasattr(self.pairs, "cpu") else np.asarray(self.pairs)
        c = None
        if self.cells is not None:
            c = (self.cells.cpu().numpy() if hasattr(self.cells, "cpu") else np.asarray(self.cells))
            c = c.view(np.uint32)
        return p[:, 0].copy(), p[:, 1].view(np.float32).copy(), p[:, 2].view(np.float32).copy(), c


def _float_dtype(arr):
    if isinstance(arr, np.ndarray):
        return np.float32
    import torch
    return torch.float32


def _stream_ptr(torch, device):
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)  # ~10x cheaper than current_stream
    if raw is not None:
        return ctypes.c_void_p(raw(device.index if device.index is not None else
                                   torch.cuda.current_device()))
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def barcodes(image, maxdim: int = 1, cells: bool = False, capacity: int | None = None,
             out=None) -> Barcode:
    """Barcode of one image (torch CUDA float32 tensor, 1-3 dims, x = last axis).

    ``out``: optional preallocated (pairs int32 (cap,3), cells int32 (cap,) or None) buffers.
    """
    import torch
    if not (isinstance(image, torch.Tensor) and image.is_cuda and image.dtype == torch.float32):
        raise TypeError("image must be a CUDA float32 tensor")
    image = image.contiguous()
    shape = tuple(image.shape)
    if out is None:
        cap = max_pairs(shape, maxdim) if capacity is None else int(capacity)
        pairs = torch.empty((max(cap, 1), 3), dtype=torch.int32, device=image.device)
        cbuf = torch.empty((max(cap, 1),), dtype=torch.int32, device=image.device) if cells else None
    else:
        pairs, cbuf = out
        cap = pairs.shape[0]
    n = ctypes.c_int64(0)
    with torch.cuda.device(image.device):  # the library runs on the current device
        st = _lib.cr_barcodes(image.data_ptr(), _shape(shape), len(shape), int(maxdim), pairs.data_ptr(),
                              cbuf.data_ptr() if cbuf is not None else None, cap, ctypes.byref(n),
                              _stream_ptr(torch, image.device))
    _check(st)
    m = int(n.value)
    return Barcode(pairs[:m], cbuf[:m] if cbuf is not None else None)


def barcodes_host(image: np.ndarray, maxdim: int = 1, cells: bool = False, out=None,
                  stream=None) -> Barcode:
    """End-to-end entry: host (numpy, ideally pinned) image in, host bars out."""
    import torch
    img = np.ascontiguousarray(image, dtype=np.float32) if isinstance(image, np.ndarray) else image
    shape = tuple(img.shape)
    if out is None:
        cap = max_pairs(shape, maxdim)
        pairs = np.empty((max(cap, 1), 3), np.int32)
        cbuf = np.empty((max(cap, 1),), np.uint32) if cells else None
    else:
        pairs, cbuf = out
        cap = pairs.shape[0]
    ptr_img = img.ctypes.data if isinstance(img, np.ndarray) else img.data_ptr()
    ptr_out = pairs.ctypes.data if isinstance(pairs, np.ndarray) else pairs.data_ptr()
    ptr_c = None
    if cbuf is not None:
        ptr_c = cbuf.ctypes.data if isinstance(cbuf, np.ndarray) else cbuf.data_ptr()
    n = ctypes.c_int64(0)
    s = stream if stream is not None else torch.cuda.current_stream()
    st = _lib.cr_barcodes_host(ptr_img, _shape(shape), len(shape), int(maxdim), ptr_out, ptr_c, cap,
                               ctypes.byref(n), ctypes.c_void_p(s.cuda_stream))
    _check(st)
    m = int(n.value)
    return Barcode(pairs[:m], cbuf[:m] if cbuf is not None else None)


def barcodes_batched(images, maxdim: int = 1, cells: bool = False, capacity: int | None = None):
    """Barcodes of a batch (torch CUDA float32 tensor (B, *shape)).  Returns (Barcode, offsets)
    with offsets an int64 CUDA tensor of B+1 CSR offsets."""
    import torch
    if not (isinstance(images, torch.Tensor) and images.is_cuda and images.dtype == torch.float32):
        raise TypeError("images must be a CUDA float32 tensor")
    images = images.contiguous()
    B = int(images.shape[0])
    shape = tuple(images.shape[1:])
    cap = (max_pairs(shape, maxdim) * B) if capacity is None else int(capacity)
    pairs = torch.empty((max(cap, 1), 3), dtype=torch.int32, device=images.device)
    cbuf = torch.empty((max(cap, 1),), dtype=torch.int32, device=images.device) if cells else None
    offsets = torch.empty((B + 1,), dtype=torch.int64, device=images.device)
    n = ctypes.c_int64(0)
    with torch.cuda.device(images.device):  # the library runs on the current device
        st = _lib.cr_barcodes_batched(images.data_ptr(), B, _shape(shape), len(shape), int(maxdim),
                                      pairs.data_ptr(), cbuf.data_ptr() if cbuf is not None else None,
                                      cap, offsets.data_ptr(), ctypes.byref(n),
                                      _stream_ptr(torch, images.device))
    _check(st)
    m = int(n.value)
    return Barcode(pairs[:m], cbuf[:m] if cbuf is not None else None), offsets


def barcodes_batched_host(images, maxdim: int = 1, cells: bool = False, out=None, stream=None):
    """End-to-end batch entry: host images (numpy or pinned CPU tensor, shape (B, *shape)) in,
    host bars + CSR offsets out (cr_barcodes_batched_host).  ``out``: optional preallocated host
    (pairs int32 (cap,3), offsets int64 (B+1,), cells uint32 (cap,) or None).  Returns
    (Barcode, offsets) as host arrays/tensors."""
    import torch
    img = np.ascontiguousarray(images, dtype=np.float32) if isinstance(images, np.ndarray) else images
    B = int(img.shape[0])
    shape = tuple(img.shape[1:])
    if out is None:
        cap = max(max_pairs(shape, maxdim) * B, 1)
        pairs = np.empty((cap, 3), np.int32)
        offs = np.empty((B + 1,), np.int64)
        cbuf = np.empty((cap,), np.uint32) if cells else None
    else:
        pairs, offs, cbuf = out
    cap = int(pairs.shape[0])

    def ptr(a):
        return None if a is None else (a.ctypes.data if isinstance(a, np.ndarray) else a.data_ptr())
    n = ctypes.c_int64(0)
    s = stream if stream is not None else torch.cuda.current_stream()
    st = _lib.cr_barcodes_batched_host(ptr(img), B, _shape(shape), len(shape), int(maxdim),
                                       ptr(pairs), ptr(cbuf), cap, ptr(offs), ctypes.byref(n),
                                       ctypes.c_void_p(s.cuda_stream))
    _check(st)
    m = int(n.value)
    return Barcode(pairs[:m], cbuf[:m] if cbuf is not None else None), offs


def pairing(image):
    """Full cell pairing (uint32 stored in an int32 CUDA tensor of Khalimsky size)."""
    import torch
    image = image.contiguous()
    shape = tuple(image.shape)
    part = torch.empty((num_cells(shape),), dtype=torch.int32, device=image.device)
    with torch.cuda.device(image.device):  # the library runs on the current device
        st = _lib.cr_pairing(image.data_ptr(), _shape(shape), len(shape), part.data_ptr(),
                             _stream_ptr(torch, image.device))
    _check(st)
    return part


def death_cells(image, birth_cells):
    """kidx of the cell that kills each bar (PAPER.md:326-331 location="death"), given the bars'
    birth cells from ``barcodes(..., cells=True)``; 0xFFFFFFFF (as int32 -1) for essential bars."""
    import torch
    image = image.contiguous()
    shape = tuple(image.shape)
    birth_cells = birth_cells.contiguous()
    n = int(birth_cells.numel())
    out = torch.empty((max(n, 1),), dtype=torch.int32, device=image.device)
    with torch.cuda.device(image.device):  # the library runs on the current device
        st = _lib.cr_death_cells(image.data_ptr(), _shape(shape), len(shape), birth_cells.data_ptr(), n,
                                 out.data_ptr(), _stream_ptr(torch, image.device))
    _check(st)
    return out[:n]


def cell_coords(cells, shape):
    """Khalimsky (X, Y, Z) of cells and their base voxel (x, y, z) = (X//2, Y//2, Z//2) -- the
    paper's cell location (x, y, z, m).  cells: int64/uint32 array."""
    s = [1] * (3 - len(shape)) + [int(v) for v in shape]
    KX, KY = 2 * s[2] - 1, 2 * s[1] - 1
    k = np.asarray(cells).astype(np.int64) & 0xFFFFFFFF
    X, Y, Z = k % KX, (k // KX) % KY, k // (KX * KY)
    return np.stack([X, Y, Z], -1), np.stack([X // 2, Y // 2, Z // 2], -1)


def lifetime_image(images, maxdim: int = 2, inf_value: float | None = None, batched: bool = False):
    """Lifetime-enhanced image(s): channel 0 the image, channel 1+d the largest
    dim-d lifetime born at each voxel (0 elsewhere).  Essential bars die at ``inf_value``
    (default: the largest finite value of the input).  Returns (C, *shape), or (B, C, *shape)
    with ``batched=True`` (images of shape (B, *shape))."""
    import torch
    images = images.contiguous()
    shape = tuple(images.shape[1:] if batched else images.shape)
    B = int(images.shape[0]) if batched else 1
    if inf_value is None:
        fin = images[torch.isfinite(images)]
        inf_value = float(fin.max().item()) if fin.numel() else 0.0
    D = sum(1 for v in shape if v > 1)
    C = 2 + min(int(maxdim), max(D - 1, 0))
    out = torch.empty((B, C) + shape, dtype=torch.float32, device=images.device)
    with torch.cuda.device(images.device):  # the library runs on the current device
        st = _lib.cr_lifetime_image(images.data_ptr(), B, _shape(shape), len(shape), int(maxdim),
                                    float(inf_value), out.data_ptr(), _stream_ptr(torch, images.device))
    _check(st)
    return out if batched else out[0]


def barcodes_topdim(image, cells: bool = False) -> "Barcode":
    """Top-dimension bars only (dim D-1; the paper's --top_dim) by Alexander
    duality.  image: CUDA float32 tensor with >= 2 axes of extent > 1."""
    import torch
    image = image.contiguous()
    shape = tuple(image.shape)
    D = sum(1 for v in shape if v > 1)
    cap = max(max_pairs(shape, D - 1) - max_pairs(shape, D - 2), 1)
    pairs = torch.empty((cap, 3), dtype=torch.int32, device=image.device)
    cbuf = torch.empty((cap,), dtype=torch.int32, device=image.device) if cells else None
    n = ctypes.c_int64(0)
    with torch.cuda.device(image.device):  # the library runs on the current device
        st = _lib.cr_barcodes_topdim(image.data_ptr(), _shape(shape), len(shape), pairs.data_ptr(),
                                     cbuf.data_ptr() if cbuf is not None else None, cap,
                                     ctypes.byref(n), _stream_ptr(torch, image.device))
    _check(st)
    m = int(n.value)
    return Barcode(pairs[:m], cbuf[:m] if cbuf is not None else None)


@dataclass
class Barcode64:
    """Bars of a float64 image (cr_barcodes_f64), ordered by (dim, birth cell kidx)."""
    dim: "object"             # torch int32 (M,)
    birth: "object"           # torch float64 (M,)
    death: "object"           # torch float64 (M,), +inf for essential classes
    cells: "object | None"    # uint32 (as int32 storage) kidx of birth cells, or None

    def numpy(self):
        c = self.cells.cpu().numpy().view(np.uint32) if self.cells is not None else None
        return (self.dim.cpu().numpy(), self.birth.cpu().numpy(), self.death.cpu().numpy(), c)


def barcodes_f64(image, maxdim: int = 1, cells: bool = False,
                 capacity: int | None = None) -> Barcode64:
    """Barcode of a CUDA float64 tensor in float64 (the paper's precision)."""
    import torch
    if not (isinstance(image, torch.Tensor) and image.is_cuda and image.dtype == torch.float64):
        raise TypeError("image must be a CUDA float64 tensor")
    image = image.contiguous()
    shape = tuple(image.shape)
    cap = max_pairs(shape, maxdim) if capacity is None else int(capacity)
    raw = torch.empty((max(cap, 1), 3), dtype=torch.float64, device=image.device)  # cr_pair64
    cbuf = torch.empty((max(cap, 1),), dtype=torch.int32, device=image.device) if cells else None
    n = ctypes.c_int64(0)
    with torch.cuda.device(image.device):  # the library runs on the current device
        st = _lib.cr_barcodes_f64(image.data_ptr(), _shape(shape), len(shape), int(maxdim),
                                  raw.data_ptr(), cbuf.data_ptr() if cbuf is not None else None, cap,
                                  ctypes.byref(n), _stream_ptr(torch, image.device))
    _check(st)
    m = int(n.value)
    raw = raw[:m]
    dim = raw.view(torch.int32).view(-1, 6)[:, 0]  # int32 dim at byte 0 of each 24-byte pair
    return Barcode64(dim, raw[:, 1], raw[:, 2], cbuf[:m] if cbuf is not None else None)
