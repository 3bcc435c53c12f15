"""Error types raised at the library boundary.

Mirrors the reference hierarchy (/root/reference/pkg/src/qapsolve/errors.py:4-36)
so that callers written against `qapsolve` catch the same classes.  Status codes
returned by the C ABI (include/qapb.h) are mapped onto these in `_lib.check`.
"""

from __future__ import annotations


class QapError(Exception):
    """Root of every error this package raises."""


class DomainError(QapError, ValueError):
    """An argument lies outside what the operation is defined for."""


class IntegrityError(QapError):
    """Persisted or replayed data no longer validates (cost mismatch, bad trail)."""


class MalformedInstanceError(QapError):
    """An instance stream holds the wrong number of tokens."""

    def __init__(self, message: str, byte_offset: int):
        self.byte_offset = byte_offset
        super().__init__(f"{message} (byte offset {byte_offset})")


class TokenParseError(QapError):
    """A token that should have been an integer was not."""

    def __init__(self, message: str, byte_offset: int | None = None, line: int | None = None):
        self.byte_offset = byte_offset
        self.line = line
        parts = []
        if byte_offset is not None:
            parts.append(f"byte offset {byte_offset}")
        if line is not None:
            parts.append(f"line {line}")
        super().__init__(f"{message} ({', '.join(parts)})" if parts else message)
