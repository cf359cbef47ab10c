"""paper_2601_20782_b200 — B200-native (sm_100a) hot path of arXiv 2601.20782:
batched reduced-precision Metropolis–Hastings sampling of an RBM neural
quantum state and the local energies that consume the samples.

The public surface mirrors the reference package ``mpvmc`` (sampler / rbm /
vmc / precision / lattice / hamiltonians / rng / errors); every per-sample
computation runs in ``lib/libmpvmc_b200.so`` (C ABI: include/mpvmc_b200.h).
"""
from .errors import EvaluationFailureError, MpvmcError, NativeLibraryError  # noqa: F401
from .hamiltonians import HeisenbergSpec, TfimSpec  # noqa: F401
from .lattice import LatticeSpec  # noqa: F401
from .precision import BF16, F16, F32, F64, FloatFormat, RoundingMode, parse_format  # noqa: F401
from .rng import derive_key  # noqa: F401

__version__ = "0.1.0"
