"""B200-native α-DFT / α-FFT (arXiv 2403.16665), drop-in for the reference's
``alpha_spectra`` transform API.

Host code here is plumbing; every transform runs in libasx.so (hand-written
sm_100a CUDA behind the C ABI in include/asx.h).  There is no CPU fallback.
"""

from .core import (
    DenseFactor,
    FrequencyGrid,
    IncompatibleAlphaError,
    Signal,
    Spectrum,
    UnsupportedSizeError,
    ValidatedPair,
    bin_frequency,
    density_for_alpha,
    is_power_of_two,
    make_dense_factor,
    validate_pair,
)
from .transforms import (
    LeafKind,
    OpCounter,
    Plan,
    alpha_fft,
    combine,
    dft_matrix,
    leaf_block_sum,
    naive_forward,
    plan,
    predicted_adds,
    predicted_mults,
    transform_samples,
)
from .comparators import (
    PaddedSignal,
    aliased_reconstruct,
    naive_inverse,
    orthogonality_kernel,
    standard_fft,
    zero_pad,
)
from ._lib import AsxCudaError, LIB_PATH

__version__ = "0.1.0"

__all__ = [
    "DenseFactor", "FrequencyGrid", "IncompatibleAlphaError", "Signal", "Spectrum", "UnsupportedSizeError",
    "ValidatedPair", "bin_frequency", "density_for_alpha", "is_power_of_two", "make_dense_factor",
    "validate_pair", "LeafKind", "OpCounter", "Plan", "alpha_fft", "combine", "dft_matrix", "leaf_block_sum",
    "naive_forward", "plan", "predicted_adds", "predicted_mults", "transform_samples", "AsxCudaError",
    "LIB_PATH", "PaddedSignal", "aliased_reconstruct", "naive_inverse", "orthogonality_kernel", "standard_fft",
    "zero_pad",
]
