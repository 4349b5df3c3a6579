"""Test shim: the reference's ``xft`` namespace served by the GPU package.

The hot-path names (grid, plans/DFT, scaled Fourier kernel,
LctParams/Signal/fast_lct/fast_frft/xft_fourier/lct_b_zero, the Mehler
transform, dense_lct_matrix) come from ``paper_0912_1379_b200`` -- GPU-backed;
the out-of-scope helpers the reference tests also import (exact Hermite zeros,
the eigen-FrFT, analytic/quadrature oracles, calibration constants) come from
the reference itself (oracle/_ref).  Used only by
tests/test_gpu_reference_suite.py to run the reference's own test files.
"""
from .errors import (ConvergenceError, DegenerateParameterError, GridMismatchError, InvalidSizeError,  # noqa
                     ParameterError, ShapeError, SingularParameterError, TruncationWarning, UnsupportedBranchError,
                     XftError)
from .hermite import HermiteGrid, asymptotic_zeros, exact_hermite_zeros, grid_spacing, hermite_function_row  # noqa
from .fftcore import DftPlan, apply_dft, naive_dft, plan_dft  # noqa
from .kernel import DFT_SIGN, apply_scaled_fourier, scaled_fourier_matrix  # noqa
from .lct import (LctParams, Signal, TransformResult, chirp_phase_step, fast_frft, fast_lct, lct_b_zero,  # noqa
                  xft_fourier)
from .dense import (DenseTransform, FrftOrder, dense_lct_matrix, eigenvector_matrix, frft_matrix,  # noqa
                    frft_matrix_asymptotic, mehler_kernel)
from .oracle import (ErrorReport, GaussianParams, QuadratureConfig, compare, direct_quadrature_lct,  # noqa
                     gaussian_lct_closed_form, gaussian_sample, quadrature_on_nodes)

__version__ = "0.1.0"
