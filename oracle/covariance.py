"""Covariance functions (oracle; test infrastructure only).

P:968-976 (Matern definition)
    phi(r) = 1/(Gamma(nu) 2^(nu-1)) (sqrt(2 nu) r / rho)^nu K_nu(sqrt(2 nu) r / rho).
P:984-990 gives a half-integer closed form that is garbled in the source (sum from
k = 1, wrong factorials, sqrt(8v)); reading R16 uses the closed forms
implied by the definition itself, with z = sqrt(2 nu) r / rho:
    nu = 1/2: exp(-z);  nu = 3/2: (1 + z) exp(-z);  nu = 5/2: (1 + z + z^2/3) exp(-z).
P:991-995 gives the nu -> infinity limit exp(-r^2/(2 rho^2)); BASELINE.json binds the
Gaussian family as exp(-r^2/rho^2) (reading R17).
C(x, y) = sigma2 * phi(|x - y|) + nugget * [x and y are the same observation]
(reading R18: sigma2 scales, nugget only on the diagonal).

r is formed by direct differences r = sqrt(sum_k (x_k - y_k)^2) -- NOT the Gram
identity -- so that the oracle is independent of the GPU path.
"""
import numpy as np

MATERN_12, MATERN_32, MATERN_52, GAUSSIAN, MATERN_NU = 0, 1, 2, 3, 4
FAMILY_NU = {MATERN_12: 0.5, MATERN_32: 1.5, MATERN_52: 2.5}


def phi(r, family, rho, nu=None):
    """Correlation phi(r) for the supported families (readings R16, R17); MATERN_NU is
    the definition of P:970 for any nu > 0 (NEXT-3: the paper's nu = 1.25, 3/4), by the Bessel
    function itself."""
    r = np.asarray(r)
    if family == MATERN_NU:
        return matern_bessel(r, nu, rho)
    if family == MATERN_12:
        z = r / rho
        return np.exp(-z)
    if family == MATERN_32:
        z = np.sqrt(r.dtype.type(3)) * r / rho
        return (1 + z) * np.exp(-z)
    if family == MATERN_52:
        z = np.sqrt(r.dtype.type(5)) * r / rho
        return (1 + z + z * z / 3) * np.exp(-z)
    if family == GAUSSIAN:
        return np.exp(-(r * r) / (rho * rho))
    raise ValueError("unknown family")


def matern_bessel(r, nu, rho):
    """The Matern definition of P:970 evaluated with scipy's K_nu (used to pin `phi`)."""
    from scipy.special import gammaln, kve

    r = np.asarray(r, dtype=np.float64)
    z = np.sqrt(2 * nu) * r / rho
    out = np.ones_like(z)
    nz = z > 0
    zz = z[nz]
    # log of z^nu K_nu(z) / (Gamma(nu) 2^(nu-1)), with K_nu(z) = kve(nu, z) e^{-z}
    out[nz] = np.exp(nu * np.log(zz) + np.log(kve(nu, zz)) - zz - gammaln(nu)
                     - (nu - 1) * np.log(2.0))
    return out


def distances(Xa, Xb):
    """r_ij = sqrt(sum_k (Xa[i,k] - Xb[j,k])^2) by direct differences."""
    diff = Xa[:, None, :] - Xb[None, :, :]
    return np.sqrt(np.sum(diff * diff, axis=2))


def cov(Xa, Xb, ia, ib, family, rho, sigma2=1.0, nugget=0.0, nu=None):
    """Covariance tile C(X_a, X_b) with global observation indices ia, ib (reading R18)."""
    r = distances(Xa, Xb)
    C = sigma2 * phi(r, family, rho, nu)
    if nugget != 0.0:
        C = C + nugget * (np.asarray(ia)[:, None] == np.asarray(ib)[None, :])
    return C
