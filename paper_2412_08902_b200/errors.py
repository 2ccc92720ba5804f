"""Exception classes with the reference's names and bases (matrices.py:10-21)."""


class FormatError(ValueError):
    """A text input could not be parsed (reference matrices.py:10-17)."""

    def __init__(self, message: str, line: int | None = None):
        if line is not None:
            message = f"line {line}: {message}"
        super().__init__(message)
        self.line = line


class InvariantError(AssertionError):
    """An internal consistency check failed (reference matrices.py:20-21)."""
