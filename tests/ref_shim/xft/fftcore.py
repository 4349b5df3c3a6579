from paper_0912_1379_b200.fft import DftPlan, apply_dft, naive_dft, plan_dft  # noqa: F401
