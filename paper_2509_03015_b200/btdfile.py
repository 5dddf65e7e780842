"""BTD1 binary container (drop-in for `blocktri.btdfile`, /root/reference/pkg/src/blocktri/btdfile.py).

Same on-disk layout (40-byte little-endian header: magic "BTD1", u32 version 1, u64 N, u32 n,
u32 d, u32 flags (bit 0: rhs follows), 12 reserved zero bytes; then the N diagonal blocks, the
N-1 sub-diagonal blocks and the optional rhs panels as float64, block-major, row-major), same
errors and bit-exact round trips (the reader wraps the raw blocks, no re-symmetrisation).

B200 path: ``read_btd(path, pinned=True)`` reads the payload straight into page-locked torch
tensors (one ``readinto`` per array, no intermediate copy), which ``recursive_factorize`` then
streams to the GPU in chunks overlapped with the level-0 elimination (btd_factorize_from_host).
"""

from __future__ import annotations

import os
import struct

import numpy as np

from .core import BlockRhs, BlockTridiagonalMatrix
from .errors import BadMagic, BtdFormatError, IoError, TruncatedPayload, VersionUnsupported

MAGIC = b"BTD1"
VERSION = 1
HEADER_SIZE = 40
_HEADER = struct.Struct("<4sIQIII")
_FLAG_RHS = 1


def _payload_bytes(N: int, n: int, d: int, has_rhs: bool) -> int:
    return 8 * (N * n * n + (N - 1) * n * n + (N * n * d if has_rhs else 0))


def write_btd(path, matrix: BlockTridiagonalMatrix, rhs: BlockRhs | None = None) -> None:
    """Write a system (and optional rhs) to ``path`` (btdfile.py:56-74)."""
    N, n = matrix.num_blocks, matrix.block_size
    if rhs is not None and (rhs.num_blocks != N or rhs.block_size != n):
        raise BtdFormatError("rhs is not conformal with the matrix")
    d = rhs.num_columns if rhs is not None else 0
    head = _HEADER.pack(MAGIC, VERSION, N, n, d, _FLAG_RHS if rhs is not None else 0)
    head = head.ljust(HEADER_SIZE, b"\x00")
    arrays = [matrix.diag, matrix.sub] + ([rhs.blocks] if rhs is not None else [])
    try:
        with open(path, "wb") as fh:
            fh.write(head)
            for a in arrays:
                a = a.cpu().numpy() if hasattr(a, "cpu") else a
                fh.write(memoryview(np.ascontiguousarray(a, dtype="<f8")).cast("B"))
    except OSError as err:
        raise IoError(f"cannot write {path}: {err}") from err


def _read_into(fh, buf: memoryview, nbytes: int) -> None:
    got = 0
    while got < nbytes:
        k = fh.readinto(buf[got:nbytes])
        if not k:
            raise TruncatedPayload(nbytes, got)
        got += k


def read_btd(path, *, pinned: bool = False):
    """Read a system written by :func:`write_btd`, bit-exactly (btdfile.py:77-107).

    Returns (BlockTridiagonalMatrix, BlockRhs | None) with numpy arenas, or page-locked CPU torch
    tensors with ``pinned=True`` (the GPU path's input format)."""
    try:
        with open(path, "rb") as fh:
            head = fh.read(HEADER_SIZE)
            if len(head) < HEADER_SIZE:
                raise TruncatedPayload(HEADER_SIZE, len(head))
            magic, version, N, n, d, flags = _HEADER.unpack(head[:_HEADER.size])
            if magic != MAGIC:
                raise BadMagic(f"bad magic {magic!r}, expected {MAGIC!r}")
            if version != VERSION:
                raise VersionUnsupported(f"container version {version} unsupported")
            if N < 1 or n < 1:
                raise BtdFormatError(f"invalid header dimensions N={N}, n={n}")
            has_rhs = bool(flags & _FLAG_RHS)
            expected = HEADER_SIZE + _payload_bytes(N, n, d, has_rhs)
            actual = os.fstat(fh.fileno()).st_size
            if actual != expected:
                raise TruncatedPayload(expected, actual)
            shapes = [(N, n, n), (N - 1, n, n)] + ([(N, n, d)] if has_rhs else [])
            out = []
            for shp in shapes:
                if pinned:
                    import torch
                    t = torch.empty(shp, dtype=torch.float64).pin_memory()
                    arr = t.numpy()
                else:
                    t = arr = np.empty(shp, dtype=np.float64)
                if arr.size:
                    _read_into(fh, memoryview(arr.reshape(-1)).cast("B"), arr.nbytes)
                if np.little_endian is False:  # pragma: no cover - the container is little-endian
                    arr.byteswap(inplace=True)
                out.append(t)
            matrix = BlockTridiagonalMatrix(out[0], out[1])
            return matrix, (BlockRhs(out[2]) if has_rhs else None)
    except OSError as err:
        raise IoError(f"cannot read {path}: {err}") from err
