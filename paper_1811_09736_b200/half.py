"""binary16 buffer codecs (drop-in for the buffer helpers of
pkg/src/halftile/half.py:129-154).

The ``.f16`` format is packed little-endian 16-bit words; the text format
is one decimal/scientific literal per line, parsed through binary32 and
rounded to binary16 (blank lines and ``#`` comments skipped).  The
reference's ``Half`` scalar class (half.py:31-127) is a simulator helper
and is not part of the B200 path: numpy's
float16 is the scalar type here.
"""

from __future__ import annotations

import numpy as np

from .errors import ParseError

HALF = np.float16


def halves_to_bytes(values) -> bytes:
    """Serialize as packed little-endian 16-bit words (half.py:129-132)."""
    arr = np.ascontiguousarray(values, dtype=HALF)
    return arr.view(np.uint16).astype("<u2").tobytes()


def halves_from_bytes(data: bytes) -> np.ndarray:
    """Inverse of :func:`halves_to_bytes`; odd byte counts are a ParseError
    (half.py:134-137)."""
    if len(data) % 2:
        raise ParseError("binary16 stream has an odd byte count")
    return np.frombuffer(data, dtype="<u2").astype(np.uint16).view(np.float16)


def parse_half_text(text: str) -> np.ndarray:
    """One literal per line -> float16 array via binary32 (half.py:139-150)."""
    values = []
    for lineno, line in enumerate(text.splitlines(), start=1):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        try:
            values.append(np.float32(line))
        except ValueError as exc:
            raise ParseError(f"line {lineno}: not a numeric literal: {line!r}") from exc
    return np.asarray(values, dtype=np.float32).astype(HALF)


def format_half_text(values) -> str:
    """One ``repr(float)`` per line, newline-terminated (half.py:152-154)."""
    arr = np.asarray(values)
    return "\n".join(repr(float(v)) for v in arr.astype(np.float32)) + "\n"
