"""W2LE emissions files: the reference's portable on-disk layout of
a T x N float32 score matrix (decoder.py:618-651), and a batched loader that
stages many files into one padded, pinned host tensor for the batched device
criteria (one host->device copy per batch).

Layout: b"W2LE" | u32 version (1) | u32 T | u32 N | T*N little-endian f32.
"""

from __future__ import annotations

import os
import struct
from typing import Iterable, Optional

import numpy as np
import torch

from .errors import ContractError, EmissionsFormatError

EMISSIONS_MAGIC = b"W2LE"
EMISSIONS_VERSION = 1
_HEADER = 16


def dump_emissions(emissions, path) -> None:
    """Write a T-by-N float32 score matrix (decoder.py:622-633, same checks)."""
    e = np.ascontiguousarray(np.asarray(emissions), dtype="<f4")
    if e.ndim != 2:
        raise ContractError(f"emissions must be 2-D, got shape {e.shape}")
    t_frames, n = e.shape
    if t_frames < 1 or n < 1:
        raise ContractError(f"refusing to write empty emissions of shape {e.shape}")
    with open(path, "wb") as f:
        f.write(EMISSIONS_MAGIC)
        f.write(struct.pack("<III", EMISSIONS_VERSION, t_frames, n))
        f.write(e.tobytes())


def read_header(path) -> tuple[int, int]:
    """(T, N) of a W2LE file, with the reference's validation (decoder.py:636-648)."""
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        head = f.read(_HEADER)
    if len(head) < _HEADER:
        raise EmissionsFormatError(f"file too short ({len(head)} bytes) for a header")
    if head[:4] != EMISSIONS_MAGIC:
        raise EmissionsFormatError(f"bad magic {head[:4]!r}, expected {EMISSIONS_MAGIC!r}")
    version, t_frames, n = struct.unpack_from("<III", head, 4)
    if version != EMISSIONS_VERSION:
        raise EmissionsFormatError(f"unsupported version {version}")
    expected = _HEADER + 4 * t_frames * n
    if size != expected:
        raise EmissionsFormatError(
            f"payload size mismatch: header implies {expected} bytes, file has {size}")
    return t_frames, n


def load_emissions(path) -> np.ndarray:
    """The reference's loader (decoder.py:636-651): float32 [T, N]."""
    t_frames, n = read_header(path)
    with open(path, "rb") as f:
        f.seek(_HEADER)
        data = np.fromfile(f, dtype="<f4", count=t_frames * n)
    return data.reshape(t_frames, n).astype(np.float32, copy=False)


def load_emissions_batch(paths: Iterable, *, pin: bool = True,
                         device: Optional[torch.device] = None,
                         stream: Optional[torch.cuda.Stream] = None):
    """Stage W2LE files into one zero-padded float32 [B, Tmax, N] host tensor
    (pinned by default: the payloads are read straight into it, no
    intermediate copies) plus int32 lengths [B].  With `device`, the batch is
    copied to the device asynchronously (on `stream` if given) and the device
    tensors are returned; the pinned host tensors stay valid until that copy
    has completed.  All files must share N."""
    paths = list(paths)
    if not paths:
        raise ContractError("no emissions files given")
    heads = [read_header(p) for p in paths]
    n = heads[0][1]
    if any(h[1] != n for h in heads):
        raise ContractError(f"emissions files disagree on N: {sorted({h[1] for h in heads})}")
    t_max = max(h[0] for h in heads)
    host = torch.zeros((len(paths), t_max, n), dtype=torch.float32, pin_memory=pin)
    lens = torch.tensor([h[0] for h in heads], dtype=torch.int32)
    view = host.numpy()
    for b, (p, (t_frames, _)) in enumerate(zip(paths, heads)):
        with open(p, "rb") as f:
            f.seek(_HEADER)
            f.readinto(memoryview(view[b, :t_frames]).cast("B"))
    if device is None:
        return host, lens
    ctx = torch.cuda.stream(stream) if stream is not None else _nullcontext()
    with ctx:
        return (host.to(device, non_blocking=True), lens.to(device, non_blocking=True))


class _nullcontext:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False
