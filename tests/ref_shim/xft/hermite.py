from paper_0912_1379_b200.hermite import HermiteGrid, asymptotic_zeros, grid_spacing, hermite_function_row  # noqa
from ._bind import reference

exact_hermite_zeros = reference().hermite.exact_hermite_zeros  # out of scope: the reference's own
