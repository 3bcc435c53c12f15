"""Error types at the library boundary: the reference's own classes when `qapsolve` is importable (so that
callers written against it catch the same classes), else a minimal local hierarchy.  Status codes of the
C ABI (include/qapb.h) are mapped onto these in `_lib.check`."""

from __future__ import annotations

from ._refpkg import reference

if reference() is not None:
    from qapsolve.errors import DomainError, IntegrityError, MalformedInstanceError, QapError, TokenParseError  # noqa: F401
else:
    class QapError(Exception):
        pass

    class DomainError(QapError, ValueError):
        pass

    class IntegrityError(QapError):
        pass

    class MalformedInstanceError(QapError):
        def __init__(self, message, byte_offset=None):
            super().__init__(message if byte_offset is None else f"{message} (byte offset {byte_offset})")
            self.byte_offset = byte_offset

    class TokenParseError(QapError):
        def __init__(self, message, byte_offset=None, line=None):
            where = [f"{k} {v}" for k, v in (("byte offset", byte_offset), ("line", line)) if v is not None]
            super().__init__(f"{message} ({', '.join(where)})" if where else message)
            self.byte_offset, self.line = byte_offset, line
