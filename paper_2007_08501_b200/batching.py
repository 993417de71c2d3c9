"""Packed <-> padded bookkeeping of heterogeneous batches on the GPU (C-ABI dr_packed_to_padded & co.).

Mirrors the reference's PackedView helpers (/root/reference/proj/include/dr/batching.hpp): packed_to_padded
(:48-59), padded_to_packed (:61-75), PackedView::item_to_element (:20-27). Ranges are given as
(first, num) per batch element like the rasterizer's mesh_to_face_first_idx / num_faces_per_mesh.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .raster import _check, _ptr, _stream, UsageError


def _ranges(first, num, dev):
    first = torch.as_tensor(first, dtype=torch.int64, device=dev).contiguous()
    num = torch.as_tensor(num, dtype=torch.int64, device=dev).contiguous()
    return first, num


def packed_to_padded(packed: torch.Tensor, first, num, max_count: int | None = None, pad_value=0):
    """packed [P, *row] -> padded [N, max_count, *row]; rows beyond num[b] hold pad_value."""
    if not packed.is_cuda:
        raise UsageError("packed must be a CUDA tensor")
    L = _lib.load()
    packed = packed.contiguous()
    first, num = _ranges(first, num, packed.device)
    N = int(first.numel())
    if max_count is None:
        max_count = int(num.max().item()) if N else 0
    row = tuple(packed.shape[1:])
    out = torch.empty((N, max_count) + row, dtype=packed.dtype, device=packed.device)
    row_bytes = packed.element_size() * max(1, int(torch.tensor(row).prod().item()) if row else 1)
    pad = torch.full(row if row else (), pad_value, dtype=packed.dtype).contiguous()
    pad_bytes = bytes(pad.numpy().tobytes()) if pad.numel() else b"\0" * row_bytes
    buf = C.create_string_buffer(pad_bytes, len(pad_bytes))
    with torch.cuda.device(packed.device):
        rc = L.dr_packed_to_padded(_ptr(packed), _ptr(first), _ptr(num), N, max_count, row_bytes,
                                   C.cast(buf, C.c_void_p), _ptr(out), _stream(packed.device))
    _check(rc, "packed_to_padded")
    return out


def padded_to_packed(padded: torch.Tensor, first, num, total: int | None = None):
    """padded [N, M, *row] -> packed [total, *row] (rows first[b] .. first[b]+num[b]-1 written)."""
    L = _lib.load()
    padded = padded.contiguous()
    first, num = _ranges(first, num, padded.device)
    N, M = int(padded.shape[0]), int(padded.shape[1])
    if total is None:
        total = int((first + num).max().item()) if N else 0
    row = tuple(padded.shape[2:])
    out = torch.zeros((total,) + row, dtype=padded.dtype, device=padded.device)
    row_bytes = padded.element_size() * (int(torch.tensor(row).prod().item()) if row else 1)
    with torch.cuda.device(padded.device):
        rc = L.dr_padded_to_packed(_ptr(padded), _ptr(first), _ptr(num), N, M, row_bytes, _ptr(out),
                                   _stream(padded.device))
    _check(rc, "padded_to_packed")
    return out


def item_to_element(first, num, total: int, device) -> torch.Tensor:
    """int32 [total]: owning batch element of each packed row (-1 where no range covers it)."""
    L = _lib.load()
    first, num = _ranges(first, num, device)
    out = torch.empty(total, dtype=torch.int32, device=device)
    with torch.cuda.device(device):
        rc = L.dr_packed_item_to_element(_ptr(first), _ptr(num), int(first.numel()), total, _ptr(out),
                                         _stream(torch.device(device)))
    _check(rc, "item_to_element")
    return out
