"""Oracle-side error classes (test infrastructure).

Same taxonomy as the reference `errors.py:4-41`; kept separate from the
product's classes so the oracle has no dependency on the package under test.
"""


class PagedKvError(Exception):
    pass


class CapacityExhausted(PagedKvError):
    pass


class DuplicateSequence(PagedKvError):
    pass


class UnknownSequence(PagedKvError):
    pass


class InvalidPrefix(PagedKvError):
    pass


class OutOfRange(PagedKvError):
    pass


class ShapeMismatch(PagedKvError):
    pass


class NoAllowedKeys(PagedKvError):
    pass
