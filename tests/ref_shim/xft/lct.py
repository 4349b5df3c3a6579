from paper_0912_1379_b200.lct import (LctParams, Signal, TransformResult, chirp_phase_step, fast_frft,  # noqa
                                      fast_lct, lct_b_zero, xft_fourier)
