"""B200-native translation hot path (greedy / beam decoding) with the
skiff API surface: translate, SearchSettings, SentenceInput, Model,
load_model_dir.  Compute runs in hand-written sm_100a CUDA kernels behind
the C ABI in include/skiff_b200.h."""

__version__ = "0.1.0"

from .errors import (CapabilityError, ConfigError, DataError, InputError,  # noqa: F401
                     NumericError, ShapeError, SkiffError, StateError)
