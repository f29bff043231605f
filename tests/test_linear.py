"""Non-SCO environment (picard::linear, linear.hpp / linear.cpp): the spec
generator is checked bit for bit against the unmodified reference (CPU); the
device Picard convergence curve (single-step partitions, one affine time-scan
per iteration) against the reference's picard_convergence_curve (GPU). Real-
valued actions: the reference itself compares them with a 1e-9 relative
tolerance (LinearEnv::actions_equal), and the curve values here are held to
1e-9 relative with identical iteration counts."""
import numpy as np
import pytest

import paper_2406_01939_b200 as P
from oracle.oracle import REF


@pytest.mark.parametrize("n,p,T,rho,seed,coupling", [(4, 4, 60, 0.5, 11, 0.0), (4, 4, 60, 0.5, 11, 0.3),
                                                      (3, 2, 40, 0.9, 5, 0.5), (1, 1, 10, 0.2, 3, 0.0),
                                                      (8, 3, 20, 0.7, 99, 0.6)])
def test_contractive_spec_matches_reference(n, p, T, rho, seed, coupling):
    s = P.make_contractive_spec(n, p, T, rho, seed, coupling)
    A, B, W, G, c = REF.linear_spec(n, p, T, rho, seed, coupling)
    assert np.array_equal(s.dynamics, A) and np.array_equal(s.input, B)
    assert np.array_equal(s.disturbances, W) and np.array_equal(s.gain, G)
    assert s.contraction == c
    assert abs(s.contraction - rho) < 1e-9


def test_contractive_spec_validation():
    with pytest.raises(P.ContractViolation):
        P.make_contractive_spec(2, 2, 5, 0.0, 1)
    with pytest.raises(P.ContractViolation):
        P.make_contractive_spec(2, 2, 5, 0.5, 1, 1.0)


def _same_curve(got, want):
    assert got.size == want.size, (got, want)
    np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,T,rho,coupling", [(4, 4, 300, 0.5, 0.0), (4, 4, 300, 0.5, 0.3), (3, 2, 700, 0.8, 0.5),
                                                (1, 1, 257, 0.3, 0.0), (8, 4, 1000, 0.6, 0.4)])
def test_convergence_curve_matches_reference(n, p, T, rho, coupling):
    spec = P.make_contractive_spec(n, p, T, rho, 7, coupling)
    for norm in ("draft", "reference"):
        want = REF.linear_curve(spec, tolerance=1e-6, normalization=norm)
        got = P.picard_convergence_curve(spec, tolerance=1e-6, normalization=norm)
        _same_curve(got.curve, want)


@pytest.mark.gpu
def test_convergence_curve_warm_start_and_cap():
    spec = P.make_contractive_spec(4, 4, 500, 0.6, 13, 0.2)
    acts, states = REF.linear_sequential(spec)
    rng = np.random.default_rng(1)
    draft = acts + 0.05 * rng.standard_normal(acts.shape)
    want = REF.linear_curve(spec, draft, tolerance=1e-8)
    got = P.picard_convergence_curve(spec, draft, tolerance=1e-8)
    _same_curve(got.curve, want)
    capped = P.picard_convergence_curve(spec, draft, tolerance=1e-12, max_iterations=3)
    _same_curve(capped.curve, REF.linear_curve(spec, draft, tolerance=1e-12, max_iterations=3))
    assert capped.curve.size == 3
    # converged cache = the closed-loop actions (Picard fixed point, Prop. 1)
    full = P.picard_convergence_curve(spec, tolerance=0.0, max_iterations=400)
    np.testing.assert_allclose(full.final_cache, acts, rtol=1e-9, atol=1e-12)


@pytest.mark.gpu
def test_convergence_curve_errors_like_the_reference():
    # a zero reference trajectory (no disturbances) cannot normalise the
    # error (linear.cpp:236-262): both raise ContractViolation
    spec = P.make_contractive_spec(2, 2, 30, 0.5, 3)
    spec.disturbances = np.zeros_like(spec.disturbances)
    for norm in ("reference", "draft"):
        with pytest.raises(Exception):
            REF.linear_curve(spec, normalization=norm)
        with pytest.raises(P.ContractViolation):
            P.picard_convergence_curve(spec, normalization=norm)
    assert P.picard_convergence_curve(P.make_contractive_spec(2, 2, 0, 0.5, 3)).curve.size == 0
