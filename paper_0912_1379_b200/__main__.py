"""python -m paper_0912_1379_b200 ...  (the reference's `xft` console script, GPU backend)."""
from .cli import entrypoint

entrypoint()
