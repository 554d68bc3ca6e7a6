"""pagedkv.errors (reference errors.py) — the engine's exception classes."""

from ..errors import *  # noqa: F401,F403
from ..errors import (  # noqa: F401
    CapacityExhausted,
    ConfigError,
    DeviceError,
    DuplicateSequence,
    InvalidPrefix,
    InvalidTrace,
    NoAllowedKeys,
    OutOfRange,
    PagedKvError,
    ShapeMismatch,
    UnknownSequence,
)
