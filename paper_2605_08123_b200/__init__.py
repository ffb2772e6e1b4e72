"""B200-native banded balanced entropic-OT attention (arxiv 2605.08123), sm_100a.

Product surface: libsinkattn.so (C-ABI, include/sinkattn.h) and its host
mirror `band.run_surrogate` / `band.r2_backward`.  Importing this package
loads the CUDA library and fails loudly if it is missing.
"""
from . import _lib  # noqa: F401  (raises ImportError when libsinkattn.so is absent)
from .band import (BandSpec, CotangentSet, CudaError, InfeasibleSupport, InvalidTemperature,  # noqa: F401
                   MissingBaseTrace, SizeCapExceeded, SurrogateRun, UnsupportedDepth, Workspace,
                   launch_count, r2_backward, run_surrogate, tail_adjoint, validate_support)
from .configs import CONFIGS, Config, make_inputs  # noqa: F401

__all__ = ["BandSpec", "SurrogateRun", "CotangentSet", "run_surrogate", "r2_backward", "tail_adjoint", "validate_support",
           "CONFIGS", "Config", "make_inputs", "launch_count", "InfeasibleSupport", "InvalidTemperature",
           "UnsupportedDepth", "MissingBaseTrace", "SizeCapExceeded", "CudaError", "Workspace"]
