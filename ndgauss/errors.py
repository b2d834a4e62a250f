"""Reference module name `ndgauss.errors` (pkg/src/ndgauss/errors.py) -> the same classes."""
from paper_2405_20067_b200.errors import *  # noqa: F401,F403
from paper_2405_20067_b200.errors import (ConfigError, DegenerateSliceError, FileFormatError,  # noqa: F401
                                          InvalidParameterError, NdgError, NonFiniteGradientError, TrainingAborted)
