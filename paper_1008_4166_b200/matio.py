"""HJAC matrix files: the reference's on-disk input format (pkg/src/hjacobi/
matio.py:1-62) read straight into the layout the GPU path wants.

Binary layout (little-endian): ``HJAC`` | u32 version (1) | u32 scalar kind
(0 float64, 1 complex128) | u64 m | u64 n | m*n elements, column-major --
which is exactly G's device layout, so ``read_matrix``
memory-maps the payload and returns a Fortran-ordered array without a
transposing copy, and ``read_matrix_pinned`` fills a page-locked buffer for a
full-speed H2D.  The whitespace text form (``m n`` then the rows, complex
entries as Python literals) is accepted too; files are told apart by the
magic.  Errors are ``MatrixFormatError`` as in the reference.
"""

from __future__ import annotations

import numpy as np

from .errors import HJacobiError

MAGIC = b"HJAC"
VERSION = 1
HEADER_BYTES = 4 + 4 + 4 + 8 + 8
_HEADER_DT = np.dtype([("magic", "S4"), ("version", "<u4"), ("kind", "<u4"), ("m", "<u8"), ("n", "<u8")])
_KINDS = (np.dtype("<f8"), np.dtype("<c16"))


class MatrixFormatError(HJacobiError):
    """Malformed or unsupported matrix file (matio.py:22-23)."""


def _as_payload(M):
    A = np.asarray(M)
    if A.ndim != 2:
        raise ValueError("expected a 2-d array")
    dt = _KINDS[1] if np.iscomplexobj(A) else _KINDS[0]
    return np.asfortranarray(A, dtype=dt)


def write_matrix(path, M, text=False):
    A = _as_payload(M)
    m, n = A.shape
    if text:
        with open(path, "w") as fh:
            fh.write(f"{m} {n}\n")
            cx = A.dtype.kind == "c"
            for row in A:
                fh.write(" ".join(repr(complex(v)) if cx else repr(float(v)) for v in row) + "\n")
        return
    head = np.zeros((), _HEADER_DT)
    head["magic"], head["version"], head["kind"], head["m"], head["n"] = MAGIC, VERSION, int(A.dtype.kind == "c"), m, n
    with open(path, "wb") as fh:
        fh.write(head.tobytes())
        fh.write(A.tobytes(order="F"))


def _header(path):
    with open(path, "rb") as fh:
        raw = fh.read(HEADER_BYTES)
        fh.seek(0, 2)
        size = fh.tell()
    if raw[:4] != MAGIC:
        return None
    if len(raw) < HEADER_BYTES:
        raise MatrixFormatError(f"{path}: truncated header")
    h = np.frombuffer(raw, _HEADER_DT)[0]
    if int(h["version"]) != VERSION:
        raise MatrixFormatError(f"{path}: unknown version {int(h['version'])}")
    if int(h["kind"]) >= len(_KINDS):
        raise MatrixFormatError(f"{path}: unknown scalar kind {int(h['kind'])}")
    dt = _KINDS[int(h["kind"])]
    m, n = int(h["m"]), int(h["n"])
    need = m * n * dt.itemsize
    have = size - HEADER_BYTES
    if have < need:
        raise MatrixFormatError(f"{path}: truncated payload ({have} of {need} bytes)")
    if have > need:
        raise MatrixFormatError(f"{path}: trailing bytes after payload")
    return dt, m, n


def _read_text(path):
    with open(path) as fh:
        tok = fh.read().split()
    if len(tok) < 2:
        raise MatrixFormatError(f"{path}: missing text header")
    try:
        m, n = int(tok[0]), int(tok[1])
        if len(tok) - 2 != m * n:
            raise ValueError
        vals = np.array([complex(t) for t in tok[2:]], np.complex128).reshape(m, n)
    except ValueError as exc:
        raise MatrixFormatError(f"{path}: malformed text matrix") from exc
    if vals.size == 0 or not vals.imag.any():
        return np.asfortranarray(vals.real)
    return np.asfortranarray(vals)


def read_matrix(path):
    """The matrix as a Fortran-ordered float64 / complex128 array."""
    h = _header(path)
    if h is None:
        return _read_text(path)
    dt, m, n = h
    if m * n == 0:
        return np.zeros((m, n), dt.newbyteorder("="), order="F")
    flat = np.fromfile(path, dtype=dt, count=m * n, offset=HEADER_BYTES)
    return flat.reshape((m, n), order="F")  # the payload already is column-major


def read_matrix_pinned(path):
    """Binary HJAC file -> page-locked column-major host tensor (torch), the
    buffer ``parallel_jacobi`` / ``hjb_solve`` copy from at full PCIe speed."""
    from . import _device

    h = _header(path)
    if h is None:
        raise MatrixFormatError(f"{path}: not a binary HJAC file")
    dt, m, n = h
    out = _device.pinned_host_colmajor(m, n, np.dtype(dt.str.replace("<", "=")))
    with open(path, "rb") as fh:
        fh.seek(HEADER_BYTES)
        if out.size:
            fh.readinto(out.T.reshape(-1).view(np.uint8))  # out.T is the C-contiguous (n, m) buffer
    return out


def write_signs(path, signs):
    s = np.asarray(signs, dtype=np.int8)
    with open(path, "w") as fh:
        fh.write(" ".join(str(int(v)) for v in s) + "\n")


def read_signs(path):
    with open(path) as fh:
        tok = fh.read().split()
    try:
        return np.array([int(t) for t in tok], dtype=np.int8)
    except ValueError as exc:
        raise MatrixFormatError(f"{path}: malformed sign vector") from exc
