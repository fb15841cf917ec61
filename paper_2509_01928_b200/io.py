"""The binary CSR container of dc/io.py:246-305 with the ingest check on the device.

Format (little-endian): magic ``ICSR1``, u64 n, u64 nnz, row offsets ((n+1) x u64),
column indices (nnz x u64), values (nnz x f64). ``csr_save`` writes the reference's
bytes; ``csr_load`` parses them with the reference's FormatError cases and runs
CsrCoupling's invariants (dc/coupling.py:153-176, including symmetry) as one device
pass (``dcx_validate_csr``) instead of the reference's per-row Python loop and
scipy transpose comparison. The arrays are views of the file's bytes (no copies).
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from .coupling import CouplingError, CsrCoupling, is_csr, is_dense

MAGIC = b"ICSR1"


class FormatError(ValueError):
    """Malformed file content (dc/io.py:35-36)."""


def _open(target, mode):
    if isinstance(target, (str, Path)):
        return True, open(target, mode)
    return False, target


def coupling_to_csr(J) -> CsrCoupling:
    """dc/io.py:246-253: CSR couplings pass through; dense ones keep their nonzeros."""
    if is_csr(J):
        return J
    if is_dense(J):
        a = np.asarray(J.array)
        rows, cols = np.nonzero(a)
        ro = np.zeros(a.shape[0] + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows, minlength=a.shape[0]), out=ro[1:])
        return CsrCoupling(a.shape[0], a[rows, cols], cols, ro, value_kind=J.value_kind, validate=False)
    raise ValueError("only dense or CSR matrices can be converted to the CSR container")


def csr_save(J, sink) -> None:
    """Write a coupling matrix to the binary CSR container (dc/io.py:256-269)."""
    m = coupling_to_csr(J)
    own, fh = _open(sink, "wb")
    try:
        fh.write(MAGIC)
        fh.write(np.uint64(m.n).tobytes())
        fh.write(np.uint64(m.nnz).tobytes())
        fh.write(np.asarray(m.row_offsets).astype("<u8").tobytes())
        fh.write(np.asarray(m.col_indices).astype("<u8").tobytes())
        fh.write(np.asarray(m.values).astype("<f8").tobytes())
    finally:
        if own:
            fh.close()


_CHECKS = {
    2: "row_offsets must be nondecreasing and start at 0",
    3: "values/col_indices length must match row_offsets[-1]",
    4: "column index out of range",
    5: "column indices not strictly increasing in row {row}",
    6: "stored diagonal entry in row {row}",
    7: "couplings must be finite",
    8: "coupling matrix must be symmetric",
}


def parse_csr(blob: bytes):
    """(n, row_offsets, col_indices, values) of a container, FormatError on malformed bytes
    (dc/io.py:280-296). Host-only: no device work."""
    if blob[: len(MAGIC)] != MAGIC:
        raise FormatError("bad magic: not a CSR container")
    off = len(MAGIC)

    def take(count: int, dtype: str) -> np.ndarray:
        nonlocal off
        nbytes = count * np.dtype(dtype).itemsize
        if off + nbytes > len(blob):
            raise FormatError("truncated CSR container")
        out = np.frombuffer(blob, dtype=dtype, count=count, offset=off)
        off += nbytes
        return out

    n = int(take(1, "<u8")[0])
    nnz = int(take(1, "<u8")[0])
    row_offsets = take(n + 1, "<u8").view(np.int64)
    col_indices = take(nnz, "<u8").view(np.int64)
    values = take(nnz, "<f8")
    if off != len(blob):
        raise FormatError("trailing bytes after CSR payload")
    return n, row_offsets, col_indices, values


def csr_load(source) -> CsrCoupling:
    """Read the binary CSR container, validating magic, sizes and the CSR invariants
    (on the device); truncated files error out with no partial matrix (dc/io.py:272-305)."""
    own, fh = _open(source, "rb")
    try:
        blob = fh.read()
    finally:
        if own:
            fh.close()
    n, ro, ci, v = parse_csr(blob)
    if n < 1:
        raise CouplingError("row_offsets must have length n+1")
    from .generate import _context

    chk, row, all_int = _context().validate_csr(n, ro, ci, v)
    # the reference builds its scipy matrix before validating: scipy's own index-pointer
    # checks fire first for these two cases (plain ValueError, scipy's wording)
    if chk == 2 and ro[0] != 0:
        raise ValueError("index pointer should start with 0")
    if chk == 3 and ro[n] > len(v):
        raise ValueError("Last value of index pointer should be less than the size of index and data arrays")
    if chk:
        raise CouplingError(_CHECKS[chk].format(row=row))
    return CsrCoupling(n, v, ci, ro, value_kind="int" if all_int else "real", validate=False)
