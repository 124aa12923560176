"""ZCA whitening oracle — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

"Spyker implements an efficient version of ZCA whitening by taking advantage of routines
from highly optimized linear algebra libraries (BLAS and LAPACK) that operate on symmetric
matrices ... a fit(array, epsilon) and a call function".  The definition, in fp64
with numpy's symmetric eigensolver as the library primitive (reading R-ZCA):

    mu = mean over rows of X[B][F];  Xc = X - mu
    C  = Xc^T Xc / (B - 1)                       (unbiased covariance)
    C  = E diag(lam) E^T                          (symmetric eigendecomposition)
    Wz = E diag((lam + eps)^-1/2) E^T             (symmetric whitening matrix)
    apply(x) = (x - mu) Wz
"""
from __future__ import annotations

import numpy as np


def fit(X: np.ndarray, eps: float):
    X = np.asarray(X, np.float64)
    B, F = X.shape
    assert B >= 2 and eps >= 0
    mu = X.mean(axis=0)
    Xc = X - mu
    C = Xc.T @ Xc / (B - 1)
    lam, E = np.linalg.eigh(C)
    if eps == 0 and lam.min() <= 0:
        raise np.linalg.LinAlgError("singular covariance with eps = 0")
    Wz = (E * (lam + eps) ** -0.5) @ E.T
    return mu, Wz


def apply(X: np.ndarray, mu: np.ndarray, Wz: np.ndarray) -> np.ndarray:
    return (np.asarray(X, np.float64) - mu) @ Wz
