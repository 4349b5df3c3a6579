from paper_0912_1379_b200.kernel import (DFT_SIGN, apply_scaled_fourier, boundary_phase,  # noqa: F401
                                         input_chirp, kernel_prefactor, output_chirp, scaled_fourier_matrix)
