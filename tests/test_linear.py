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
    # the reference's picard_simulate stops at its own 1e-9 equality (stable
    # prefixes are frozen), so its actions equal the fixed point in that sense
    assert _actions_equal(full.final_cache, acts)


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


# ---------------------------------------------------------------- MLP feedback policy
# BASELINE config 4 / SURVEY §8(f)3: the reference's MlpParams::forward as the
# linear env's policy (ref_linear_mlp_* in oracle/ref_harness.cpp run the
# unmodified reference engine, env and MLP with it).
MLP_CASES = [(4, 4, 300, 0.5, 0.0, 20.0), (4, 4, 300, 0.5, 0.3, 40.0), (3, 2, 500, 0.9, 0.5, 30.0),
             (1, 1, 200, 0.3, 0.0, 8.0), (8, 4, 400, 0.6, 0.4, 25.0)]


def _actions_equal(a, b):
    """LinearEnv::actions_equal (linear.hpp:64-71) slot by slot."""
    scale = np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
    return bool(np.all(np.abs(a - b) <= 1e-9 * scale))


def _np_forward(m, s):
    """MlpParams::forward (mlp.cpp:141-169) in numpy (the harness check)."""
    n, H, _, p = m.widths
    h1 = np.tanh(m.b1 + m.w1.reshape(H, n) @ s)
    h2 = np.tanh(m.b2 + m.w2.reshape(H, H) @ h1)
    return m.b3 + m.w3.reshape(p, H) @ h2


def test_mlp_feedback_harness_is_the_reference_forward():
    spec = P.make_contractive_spec(4, 3, 50, 0.5, 7, 0.3)
    pol = P.MlpFeedbackPolicy.seeded(4, 3, 11, 64, 20.0)
    acts, states = REF.linear_mlp_sequential(spec, pol.params)
    for t in range(spec.horizon):
        np.testing.assert_allclose(acts[t], _np_forward(pol.params, states[t]), rtol=1e-12, atol=1e-14)
        nxt = spec.dynamics[t] @ states[t] + spec.input[t] @ acts[t] + spec.disturbances[t]
        np.testing.assert_allclose(states[t + 1], nxt, rtol=1e-12, atol=1e-14)


def test_mlp_feedback_policy_validation():
    spec = P.make_contractive_spec(4, 4, 10, 0.5, 7)
    with pytest.raises(P.InvalidArgument):
        P.picard_convergence_curve(spec, policy=P.MlpFeedbackPolicy.seeded(3, 4, 1))
    bad = P.MlpFeedbackPolicy.seeded(4, 4, 1)
    bad.params.w2 = bad.params.w2[:10]
    with pytest.raises(P.InvalidArgument):
        P.picard_convergence_curve(spec, policy=bad)


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,T,rho,coupling,scale", MLP_CASES)
def test_mlp_convergence_curve_matches_reference(n, p, T, rho, coupling, scale):
    spec = P.make_contractive_spec(n, p, T, rho, 7, coupling)
    pol = P.MlpFeedbackPolicy.seeded(n, p, 3, 64, scale)
    for norm in ("draft", "reference"):
        want = REF.linear_mlp_curve(spec, pol.params, tolerance=1e-6, normalization=norm)
        got = P.picard_convergence_curve(spec, tolerance=1e-6, normalization=norm, policy=pol)
        _same_curve(got.curve, want)
    # picard_simulate's count for the single-step plan, and the fixed point =
    # the sequential trajectory (Prop. 1)
    it, acts = REF.linear_mlp_picard(spec, pol.params)
    seq_a, seq_s = REF.linear_mlp_sequential(spec, pol.params)
    assert got.iterations_to_converged == it
    np.testing.assert_allclose(got.reference_states, seq_s, rtol=1e-9, atol=1e-12)
    full = P.picard_convergence_curve(spec, tolerance=0.0, max_iterations=200, policy=pol)
    np.testing.assert_allclose(full.final_cache, seq_a, rtol=1e-9, atol=1e-12)
    # the reference's picard_simulate stops at its own 1e-9 equality (stable
    # prefixes are frozen), so its actions equal the fixed point in that sense
    assert _actions_equal(full.final_cache, acts)


@pytest.mark.gpu
def test_mlp_convergence_curve_warm_start_and_cap():
    spec = P.make_contractive_spec(4, 4, 600, 0.7, 13, 0.2)
    pol = P.MlpFeedbackPolicy.seeded(4, 4, 5, 64, 30.0)
    acts, _ = REF.linear_mlp_sequential(spec, pol.params)
    rng = np.random.default_rng(1)
    draft = acts + 0.05 * rng.standard_normal(acts.shape)
    want = REF.linear_mlp_curve(spec, pol.params, draft, tolerance=1e-8)
    got = P.picard_convergence_curve(spec, draft, tolerance=1e-8, policy=pol)
    _same_curve(got.curve, want)
    it, _ = REF.linear_mlp_picard(spec, pol.params, draft)
    assert got.iterations_to_converged == it
    capped = P.picard_convergence_curve(spec, draft, tolerance=1e-12, max_iterations=3, policy=pol)
    _same_curve(capped.curve, REF.linear_mlp_curve(spec, pol.params, draft, tolerance=1e-12, max_iterations=3))
    assert capped.curve.size == 3


@pytest.mark.gpu
def test_mlp_convergence_curve_errors_like_the_reference():
    spec = P.make_contractive_spec(2, 2, 30, 0.5, 3)
    spec.disturbances = np.zeros_like(spec.disturbances)
    pol = P.MlpFeedbackPolicy(P.MlpParams.zeros(2, 2))  # zero policy: the zero trajectory
    for norm in ("reference", "draft"):
        with pytest.raises(Exception):
            REF.linear_mlp_curve(spec, pol.params, normalization=norm)
        with pytest.raises(P.ContractViolation):
            P.picard_convergence_curve(spec, normalization=norm, policy=pol)
    empty = P.make_contractive_spec(2, 2, 0, 0.5, 3)
    assert P.picard_convergence_curve(empty, policy=P.MlpFeedbackPolicy.seeded(2, 2, 1)).curve.size == 0
