# analytic / quadrature oracles are out of scope: the reference's own
from ._bind import reference

_o = reference().oracle
GaussianParams, ErrorReport, QuadratureConfig = _o.GaussianParams, _o.ErrorReport, _o.QuadratureConfig
gaussian_sample, gaussian_lct_closed_form = _o.gaussian_sample, _o.gaussian_lct_closed_form
direct_quadrature_lct, quadrature_on_nodes, compare = _o.direct_quadrature_lct, _o.quadrature_on_nodes, _o.compare
