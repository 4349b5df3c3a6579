from paper_0912_1379_b200.errors import *  # noqa: F401,F403
from paper_0912_1379_b200.errors import (ConvergenceError, DegenerateParameterError, GridMismatchError,  # noqa: F401
                                         InvalidSizeError, ParameterError, ShapeError, SingularParameterError,
                                         TruncationWarning, UnsupportedBranchError, XftError)
