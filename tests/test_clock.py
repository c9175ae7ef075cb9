"""Relaxed-clock chain rule: clock.hpp:42-55
branch_lengths_from_clock, :140-152 d/d log mu and d/d log eps (likelihood
part), :199-213 node_time_gradient.  The reference's KATs restated:
test_clock.cpp:181-196 (the mu gradient equals the sum of the epsilon
gradients, 1e-12) and :260-295 (node-time gradient vs central finite
differences, 1e-6; near-zero child rates leave only the node's own branch
term).  The oracle (CPU) pins the formulas; the GPU tests run them through the
product (pg_clock_gradient: one kernel after the walk)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_12146_b200 import api

PSI = 0.5


class ClockFixture:
    """test_clock.cpp:14-35: coalescent tree with times, mu = 0.8, lognormal
    effects of mean one and variance psi^2 (clock.hpp:28-33), JC69
    alignment simulated down the clock lengths."""

    def __init__(self, tips, seed, sites=80):
        rng = O.Rng(seed)
        ot = O.Tree.coalescent(rng, tips, 0.6)
        self.otree = ot
        times = ot.node_time if ot.node_time is not None else ot.assign_times()
        self.tree = api.Tree(ot.tip_count, ot.parent, ot.children, np.concatenate([[0.0], ot.branch_lengths, [0.0]]),
                             ot.labels, ot.post_order, node_time=times)
        self.mu = 0.8
        v = np.log1p(PSI * PSI)
        z = np.random.default_rng(seed).standard_normal(self.tree.branch_count())
        self.eps = np.exp(-v / 2.0 + np.sqrt(v) * z)
        self.model = O.Model.jc69()
        b = api.branch_lengths_from_clock(self.tree, self.mu, self.eps)
        cols = O.simulate_states(ot, self.model, [1.0], [1.0], b, sites, seed + 1)
        self.oaln = O.Alignment.from_codes(cols, 4, ot.labels[1:ot.tip_count + 1])

    def lengths(self, tree=None, mu=None, eps=None):
        return api.branch_lengths_from_clock(tree or self.tree, self.mu if mu is None else mu,
                                             self.eps if eps is None else eps)

    def oracle_engine(self, lengths):
        t = O.Tree.from_arrays(self.otree.tip_count, self.otree.parent, self.otree.children, lengths,
                               self.otree.post_order)
        e = O.Engine(t, self.oaln, self.model, [1.0], [1.0])
        e._keep = (t,)
        return e

    def product_engine(self):
        aln = api.SitePatternAlignment(self.oaln.taxa, 4, self.oaln.pattern_codes().astype(np.int8),
                                       self.oaln.weights)
        model = api.SubstitutionModel(_jc_q(), np.full(4, 0.25), True)
        return api.LikelihoodEngine(self.tree, aln, model, api.RateCategories(np.ones(1), np.ones(1)))


def _jc_q():
    q = np.full((4, 4), 1.0 / 3.0)
    np.fill_diagonal(q, -1.0)
    return q


def _node_time_fd(fix, loglik_at_times, k, h=1e-6):
    node = fix.tree.tip_count + 1 + k
    t0 = fix.tree.node_time.copy()

    def at(shift):
        t = t0.copy()
        t[node] += shift
        tree = api.Tree(fix.tree.tip_count, fix.tree.parent, fix.tree.children, fix.tree.branch_length,
                        fix.tree.labels, fix.tree.post_order, node_time=t)
        return loglik_at_times(fix.lengths(tree))

    return (at(h) - at(-h)) / (2.0 * h)


def _node_time_formula(tree, rates, g):
    """clock.hpp:199-213 restated (independent of the product)."""
    out = np.zeros(tree.tip_count - 1)
    for node in range(tree.tip_count + 1, tree.node_count() + 1):
        v = rates[node - 1] * g[node - 1] if node != tree.root() else 0.0
        for c in tree.children[node]:
            v -= rates[c - 1] * g[c - 1]
        out[node - tree.tip_count - 1] = v
    return out


# ------------------------------------------------------------------- CPU
def test_branch_lengths_from_clock_contract():  # clock.hpp:42-55
    fix = ClockFixture(6, 11)
    b = fix.lengths()
    t = fix.tree.node_time
    for i in range(1, fix.tree.node_count()):
        assert b[i - 1] == pytest.approx(fix.mu * fix.eps[i - 1] * (t[i] - t[fix.tree.parent[i]]), rel=1e-15)
    no_times = api.Tree(fix.tree.tip_count, fix.tree.parent, fix.tree.children, fix.tree.branch_length)
    with pytest.raises(api.InvalidArgument, match="no node times"):
        api.branch_lengths_from_clock(no_times, 1.0, fix.eps)
    with pytest.raises(api.InvalidArgument, match="one epsilon per branch"):
        api.branch_lengths_from_clock(fix.tree, 1.0, fix.eps[:-1])
    with pytest.raises(api.InvalidArgument, match="positive"):
        api.branch_lengths_from_clock(fix.tree, 0.0, fix.eps)
    bad = fix.eps.copy()
    bad[2] = -1.0
    with pytest.raises(api.InvalidArgument, match="positive"):
        api.branch_lengths_from_clock(fix.tree, 1.0, bad)


def test_oracle_node_time_gradient_vs_fd():  # test_clock.cpp:260-280 on the oracle
    fix = ClockFixture(7, 104, 60)
    _, g, _ = fix.oracle_engine(fix.lengths()).branch_gradient(False)
    analytic = _node_time_formula(fix.tree, fix.mu * fix.eps, g)
    for k in range(fix.tree.tip_count - 1):
        fd = _node_time_fd(fix, lambda b: fix.oracle_engine(b).log_likelihood(), k)
        assert analytic[k] == pytest.approx(fd, rel=1e-6, abs=1e-6)


# ------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_mu_gradient_is_sum_of_epsilon_gradients():  # test_clock.cpp:181-196
    fix = ClockFixture(10, 55)
    eng = fix.product_engine()
    rng = np.random.default_rng(2)
    for _ in range(10):
        x = 0.3 * rng.standard_normal(1 + fix.tree.branch_count())
        x[0] -= 0.5
        mu, eps = float(np.exp(x[0])), np.exp(x[1:])
        dmu, deps = api.clock_likelihood_gradient(eng, fix.tree, mu, eps)
        assert dmu == pytest.approx(float(np.sum(deps)), rel=1e-12, abs=1e-12)
        # and d/d log eps_i = b_i g_i against the oracle's branch gradient
        b = fix.lengths(mu=mu, eps=eps)
        _, g, _ = fix.oracle_engine(b).branch_gradient(False)
        np.testing.assert_allclose(deps, b * g, rtol=1e-9, atol=1e-12 * np.abs(b * g).max())


@pytest.mark.gpu
def test_node_time_gradient_vs_fd():  # test_clock.cpp:260-280
    fix = ClockFixture(7, 104, 60)
    eng = fix.product_engine()
    analytic = api.node_time_gradient(eng, fix.tree, fix.mu, fix.eps)
    _, g, _ = fix.oracle_engine(fix.lengths()).branch_gradient(False)
    np.testing.assert_allclose(analytic, _node_time_formula(fix.tree, fix.mu * fix.eps, g), rtol=1e-9,
                               atol=1e-12 * np.abs(g).max())
    probe = fix.product_engine()

    def loglik(b):
        probe.set_branch_lengths(b)
        return probe.log_likelihood()

    for k in range(fix.tree.tip_count - 1):
        fd = _node_time_fd(fix, loglik, k)
        assert analytic[k] == pytest.approx(fd, rel=1e-6, abs=1e-6)


@pytest.mark.gpu
def test_node_time_gradient_muted_children():  # test_clock.cpp:282-294
    fix = ClockFixture(7, 104, 60)
    eng = fix.product_engine()
    tree = fix.tree
    root_child = int(tree.children[tree.root()][0])
    if root_child <= tree.tip_count:
        root_child = int(tree.children[tree.root()][1])
    assert root_child > tree.tip_count
    eps = fix.eps.copy()
    for c in tree.children[root_child]:
        eps[c - 1] = 1e-12
    g_nt = api.node_time_gradient(eng, tree, fix.mu, eps)
    eng.set_branch_lengths(fix.lengths(eps=eps))
    rep = eng.branch_gradient()
    own = fix.mu * eps[root_child - 1] * rep.branch_gradient[root_child - 1]
    assert g_nt[root_child - tree.tip_count - 1] == pytest.approx(own, abs=1e-6)


@pytest.mark.gpu
def test_clock_gradient_rates_from_durations():
    """rates=None derives r_i = b_i / dt_i from pg_set_clock_durations."""
    fix = ClockFixture(9, 21)
    eng = fix.product_engine()
    t = fix.tree.node_time
    dt = np.array([t[i] - t[fix.tree.parent[i]] for i in range(1, fix.tree.node_count())])
    eng.set_branch_lengths(fix.lengths())
    eng.set_clock_durations(dt)
    a = eng.clock_gradient()
    b = eng.clock_gradient(fix.mu * fix.eps)
    np.testing.assert_allclose(a.node_time, b.node_time, rtol=1e-12, atol=1e-14 * np.abs(b.node_time).max())
    assert a.dlog_mu == b.dlog_mu and np.array_equal(a.dlog_epsilon, b.dlog_epsilon)
    with pytest.raises(api.InvalidArgument):
        eng.clock_gradient(np.ones(3))
