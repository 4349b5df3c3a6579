from paper_0912_1379_b200.dense import dense_lct_matrix  # noqa: F401
from paper_0912_1379_b200.mehler import DenseTransform, FrftOrder, frft_matrix_asymptotic, mehler_kernel  # noqa
from ._bind import reference

# the exact-zero eigendecomposition FrFT is out of scope: the reference's own
eigenvector_matrix = reference().dense.eigenvector_matrix
frft_matrix = reference().dense.frft_matrix
