"""B200-native NNFFT and fast sinc transform (arXiv 2107.02671).

Drop-in for the hot path of the reference package ``sincfft``: the names,
signatures, defaults and exception classes of ``sincfft.nnfft`` and
``sincfft.fast_sinc`` (reference ``pkg/src/sincfft/__init__.py:17-47``), backed
by hand-written sm_100a CUDA kernels behind the C ABI in
``include/sincfft_b200.h``.  Importing the package loads that library and
fails loudly if it has not been built; there is no CPU fallback.
"""

from . import bounds, direct
from .direct import ndft_direct, nndft_direct, sinc_transform_direct
from .nfft import NfftPlan, nfft_adjoint, nfft_plan, nfft_trafo
from .errors import ParameterError, PositivityError
from .fast_sinc import SincMode, SincPlan, fast_sinc_transform, sinc_plan
from .nnfft import (NnfftGeometry, NnfftPlan, WindowSpec, nnfft_adjoint, nnfft_plan,
                    nnfft_trafo, nnfft_trafo_into, rescale_frequencies)
from .quadrature import (CcQuadrature, cc_export_csv, cc_quadrature, cc_weights_direct,
                         cc_weights_fast)
from .sinc_approx import sinc_expsum_eval, sinc_expsum_eval_grid, sinc_expsum_max_error
from .windows import omega_eval, omega_hat_eval, phi_eval, phi_hat_eval, window_kinds

__version__ = "0.1.0"

__all__ = [
    "ParameterError", "PositivityError",
    "WindowSpec", "window_kinds", "omega_eval", "omega_hat_eval", "phi_eval", "phi_hat_eval",
    "NnfftGeometry", "NnfftPlan", "nnfft_plan", "nnfft_trafo", "nnfft_trafo_into", "nnfft_adjoint",
    "rescale_frequencies",
    "CcQuadrature", "cc_quadrature", "cc_weights_direct", "cc_weights_fast",
    "cc_export_csv",
    "SincMode", "SincPlan", "sinc_plan", "fast_sinc_transform",
    "NfftPlan", "nfft_plan", "nfft_trafo", "nfft_adjoint",
    "nndft_direct", "ndft_direct", "sinc_transform_direct",
    "sinc_expsum_eval", "sinc_expsum_eval_grid", "sinc_expsum_max_error",
    "bounds", "direct", "__version__",
]
