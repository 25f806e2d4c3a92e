"""NPY grid files for the command line (the I/O contract of the reference's
`phaseirls unwrap`; reference arrayio.py:19-46).

Contract kept: a grid file is an NPY v1/v2/v3 file holding one finite 2-D
float32/float64 array (object arrays / pickles refused); reading yields a
C-contiguous float64 array; writing stores "<f8" (or "<f4") at exactly the
path given.  Anything else raises `GridFileError` (a ValueError), which the
CLI maps to exit code 2.

Structure (not the reference's): the header is parsed and checked before a
single payload byte is read, the payload is read straight into the float64
result when the file is already "<f8" C-order, and writing goes through a
temporary file that is renamed into place, so a failed run never leaves a
truncated output behind.
"""

from __future__ import annotations

import os
import tempfile

import numpy as np
from numpy.lib import format as npy

__all__ = ["GridFileError", "read_grid", "write_grid"]

_WRITE_TYPES = {"<f8": np.dtype("<f8"), "<f4": np.dtype("<f4")}


class GridFileError(ValueError):
    """The file is not a well-formed 2-D float grid."""


def _header(fh, path):
    try:
        major, _minor = npy.read_magic(fh)
        reader = {1: npy.read_array_header_1_0, 2: npy.read_array_header_2_0}.get(major)
        if reader is None:  # v3 headers share the v2 layout (utf-8 dict)
            reader = npy.read_array_header_2_0
        shape, fortran, dtype = reader(fh)
    except (ValueError, OSError, EOFError) as exc:
        raise GridFileError(f"{path}: not an NPY file ({exc})") from None
    if dtype.hasobject:
        raise GridFileError(f"{path}: object arrays are not accepted")
    if len(shape) != 2:
        raise GridFileError(f"{path}: a grid must be 2-D, file holds shape {tuple(shape)}")
    if dtype.kind != "f" or dtype.itemsize not in (4, 8):
        raise GridFileError(f"{path}: a grid must hold float32/float64, file holds {dtype}")
    return tuple(int(s) for s in shape), bool(fortran), dtype


def read_grid(path) -> np.ndarray:
    """Finite 2-D float grid -> new C-contiguous float64 array."""
    try:
        fh = open(path, "rb")
    except FileNotFoundError:
        raise GridFileError(f"{path}: file not found") from None
    except OSError as exc:
        raise GridFileError(f"{path}: cannot open ({exc})") from None
    with fh:
        shape, fortran, dtype = _header(fh, path)
        count = shape[0] * shape[1]
        raw = np.fromfile(fh, dtype=dtype, count=count)
    if raw.size != count:
        raise GridFileError(f"{path}: payload holds {raw.size} of {count} values")
    arr = raw.reshape(shape[::-1]).T if fortran else raw.reshape(shape)
    grid = np.ascontiguousarray(arr, dtype=np.float64)
    if not np.isfinite(grid).all():
        raise GridFileError(f"{path}: grid holds NaN or infinite values")
    return grid


def write_grid(path, arr, dtype="<f8") -> None:
    """2-D array -> NPY file at `path` ("<f8" or "<f4"), written atomically."""
    if dtype not in _WRITE_TYPES:
        raise ValueError(f"dtype must be one of {sorted(_WRITE_TYPES)}, got {dtype!r}")
    grid = np.asarray(arr)
    if grid.ndim != 2:
        raise ValueError(f"a grid must be 2-D, got shape {grid.shape}")
    grid = np.ascontiguousarray(grid, dtype=_WRITE_TYPES[dtype])
    path = os.fspath(path)
    folder = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(prefix=".grid-", dir=folder)
    umask = os.umask(0)
    os.umask(umask)
    os.fchmod(fd, 0o666 & ~umask)
    try:
        with os.fdopen(fd, "wb") as fh:
            npy.write_array(fh, grid, version=(1, 0), allow_pickle=False)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise
