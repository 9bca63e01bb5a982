"""Exception types of the B200 backend.

The names and meanings mirror the reference's error hierarchy
(reference: pkg/src/boardlang/errors.py:4-76) so that callers written
against the reference keep their ``except`` clauses.  The C-ABI returns
integer status codes (include/ludax_b200.h, ``LX_E*``); ``raise_status``
maps them back onto these classes.
"""

from __future__ import annotations


class BoardLangError(Exception):
    """Base class (reference errors.py:4)."""


class ParseError(BoardLangError):
    """Game text does not match the grammar (reference errors.py:8-21)."""

    def __init__(self, message, line=None, column=None, expected=None):
        self.line = line
        self.column = column
        self.expected = frozenset(expected) if expected else frozenset()
        loc = f" at line {line}, column {column}" if line is not None else ""
        super().__init__(f"{message}{loc}")


class UnknownKeywordError(ParseError):
    """Unknown keyword in a position (reference errors.py:24)."""


class ArityError(ParseError):
    """Wrong number / type of arguments (reference errors.py:28)."""


class ValidationFailure(BoardLangError):
    """Semantic check findings (reference errors.py:32-37); str = the report."""

    def __init__(self, report):
        self.report = report
        super().__init__(str(report))


class InvalidShapeParam(BoardLangError):
    """Board shape parameters out of range (reference errors.py:40)."""


class UnsupportedConstruct(BoardLangError):
    """A node the lowering has no device template for (reference errors.py:48)."""


class MissingForwardAssignment(BoardLangError):
    """Relative direction without set_forward (reference errors.py:55)."""


class IllegalAction(BoardLangError):
    """Stepped action whose legal-mask entry is false (reference errors.py:59)."""


class TerminalState(BoardLangError):
    """Operation needs a live game (reference errors.py:63)."""


class EmptyMask(BoardLangError):
    """No legal action and no pass (reference errors.py:67)."""


class CompileError(BoardLangError):
    """Lowering / NVRTC failure with the failing stage (reference errors.py:71-76)."""

    def __init__(self, stage, message):
        self.stage = stage
        super().__init__(f"{stage}: {message}")


class DeviceError(BoardLangError):
    """CUDA driver / launch failure reported by the native library."""


# status codes of the C-ABI (keep in sync with include/ludax_b200.h)
LX_OK = 0
LX_EILLEGAL_ACTION = 1
LX_ETERMINAL_STATE = 2
LX_EEMPTY_MASK = 3
LX_ECOMPILE = 4
LX_ECUDA = 5
LX_EINVALID = 6


def raise_status(code, message, bad_row=-1):
    """Re-raise a native status code as the reference exception type."""
    if code == LX_OK:
        return
    row = f" (first bad row {bad_row})" if bad_row >= 0 else ""
    if code == LX_EILLEGAL_ACTION:
        raise IllegalAction(f"{message}{row}")
    if code == LX_ETERMINAL_STATE:
        raise TerminalState(f"{message}{row}")
    if code == LX_EEMPTY_MASK:
        raise EmptyMask(f"{message}{row}")
    if code == LX_ECOMPILE:
        raise CompileError("nvrtc", message)
    if code == LX_ECUDA:
        raise DeviceError(message)
    raise BoardLangError(f"native error {code}: {message}")
