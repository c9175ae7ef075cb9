"""GPU parity of every DMMA walkm instantiation and of the engine routes,
against the CPU oracle: MP = 8 / 16 / 20 (odd k-step chains) / 24 / 32 / 64, one and many rate categories (operand staging on and off),
per-branch generators (non-homogeneous Q, Padé path), ambiguous and missing
tips, the likelihood-only route (engine.hpp:146-149) against the gradient
route (test_engine.cpp:161: routes agree), and a traversal-order change
(test_engine.cpp:185).  Tolerances: tests/helpers.py (1e-9 relative)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import assert_logl, assert_vec, oracle_for

pytestmark = pytest.mark.gpu

pg = pytest.importorskip("paper_1905_12146_b200")
from workloads import synth  # noqa: E402
from paper_1905_12146_b200.api import (EngineOptions, LikelihoodEngine, RateCategories,  # noqa: E402
                                       SitePatternAlignment, SubstitutionModel, Tree)


def _reversible(m, rng, conc=2.0):
    pi = rng.dirichlet(np.ones(m) * conc)
    s = rng.lognormal(0, 0.7, (m, m))
    s = (s + s.T) / 2
    q = s * pi[None, :]
    np.fill_diagonal(q, 0)
    np.fill_diagonal(q, -q.sum(1))
    q /= -np.sum(pi * np.diag(q))
    return q, pi


def _general(m, rng):
    q = rng.lognormal(0, 0.5, (m, m))
    np.fill_diagonal(q, 0)
    np.fill_diagonal(q, -q.sum(1))
    return q


def _pair(m, L, taxa, sites, seed, branch_q=(), gaps=0.0, post_order=None, **opts):
    rng = np.random.default_rng(seed)
    q, pi = _reversible(m, rng)
    mo = O.Model(q, pi, True)
    for br, g in branch_q:
        mo.set_branch_generator(br, g)
    r = O.Rng(seed)
    tree_o = O.Tree.random(r, taxa, 0.03, 0.8)
    rates, probs = O.discrete_gamma(0.5, L) if L > 1 else ([1.0], [1.0])
    codes = O.simulate_states(tree_o, mo, rates, probs, tree_o.branch_lengths, sites, seed + 1)
    if gaps:
        codes = np.where(rng.random(codes.shape) < gaps, -1, codes)
    labels = [tree_o.labels[i] for i in range(1, tree_o.tip_count + 1)]
    aln_o = O.Alignment.from_codes(codes, m, labels)
    ref = O.Engine(tree_o, aln_o, mo, rates, probs, **opts)
    po = tree_o.post_order if post_order is None else post_order(tree_o)
    tree = Tree(tree_o.tip_count, tree_o.parent, tree_o.children,
                np.concatenate([[0.0], tree_o.branch_lengths, [0.0]]), tree_o.labels, po)
    aln = SitePatternAlignment.from_codes(labels, codes, m)
    model = SubstitutionModel(q, pi, True)
    for br, g in branch_q:
        model.set_branch_generator(br, g)
    eng = LikelihoodEngine(tree, aln, model, RateCategories(np.asarray(rates), np.asarray(probs)),
                           EngineOptions(force_rescaling=opts.get("force_rescaling", False)))
    return eng, ref


def _check(eng, ref, hess=True):
    ll, g, h = ref.branch_gradient(hess)
    rep = eng.branch_gradient(hess)
    assert_logl(rep.log_likelihood, ll)
    assert_vec(rep.branch_gradient, g)
    if hess:
        assert_vec(rep.hessian_diagonal, h, rtol=1e-8, what="hessian")
    return rep


@pytest.mark.parametrize("m,L", [(5, 2), (7, 4), (8, 1), (9, 1), (12, 4), (16, 3), (17, 4), (19, 1), (20, 5), (21, 2), (24, 4), (25, 1),
                                 (31, 4), (33, 2), (48, 4), (64, 1), (64, 3)])
def test_walkm_instantiations(m, L):
    eng, ref = _pair(m, L, 13, 300, 97 * m + L, gaps=0.05)
    _check(eng, ref)
    assert eng.info()["kernel"] == "walkm_kernel"  # geometry of the last evaluation


@pytest.mark.parametrize("m", [20, 61])
def test_walkm_per_branch_generators(m):
    """Non-homogeneous Q (engine.hpp:384-394; substitution.hpp:131-143): Padé
    P(t) per branch, generators read from global fragment tables, tip Q e
    from Q_branch P columns."""
    rng = np.random.default_rng(m)
    bq = [(1, _general(m, rng)), (4, _general(m, rng)), (9, _general(m, rng))]
    eng, ref = _pair(m, 4, 11, 200, 5 * m, branch_q=bq)
    _check(eng, ref)


@pytest.mark.parametrize("m", [4, 6, 20, 61])
def test_likelihood_route_matches_gradient_route(m):
    """logL-only evaluation (post pass, engine.hpp:146-149) equals the logL of
    the gradient evaluation (test_engine.cpp:161 asks 1e-14)."""
    eng, ref = _pair(m, 4, 15, 250, 3 * m + 1)
    ll_only = eng.log_likelihood()
    eng.invalidate_caches()
    rep = eng.branch_gradient()
    assert abs(ll_only - rep.log_likelihood) <= 1e-14 * abs(rep.log_likelihood)
    assert_logl(ll_only, ref.log_likelihood())


@pytest.mark.parametrize("m", [4, 20])
def test_traversal_order_invariance(m):
    """A different valid post-order for the same tree (test_engine.cpp:185)
    gives the same results to 1e-12 (the engine schedules its own order)."""
    def right_first(t):
        order = []

        def visit(k):
            if k > t.tip_count:
                a, b = t.children[k]
                visit(b)
                visit(a)
            order.append(k)
        visit(t.root)
        return np.asarray(order, np.int32)

    e1, ref = _pair(m, 4, 14, 200, 77 + m)
    e2, _ = _pair(m, 4, 14, 200, 77 + m, post_order=right_first)
    r1, r2 = e1.branch_gradient(True), e2.branch_gradient(True)
    assert abs(r1.log_likelihood - r2.log_likelihood) <= 1e-12 * abs(r1.log_likelihood)
    assert np.allclose(r1.branch_gradient, r2.branch_gradient, rtol=1e-12, atol=1e-12 * np.abs(r1.branch_gradient).max())
    _check(e1, ref)


def test_walkm_forced_rescaling_neutral():  # test_engine.cpp:324-340 on the DMMA kernel
    eng, ref = _pair(20, 4, 12, 150, 404, force_rescaling=True)
    _check(eng, ref)


def test_walkm_many_tiles_and_ragged_tail():
    """Pattern counts that are not multiples of the 32-pattern CTA tile, at a
    size that runs several tiles per CTA."""
    for sites in (33, 1001):
        inst = synth.generate("C4", sites=sites)
        eng = synth.engine_for(inst)
        ref = oracle_for(inst, blocks=4)
        ll, g, _ = ref.branch_gradient(False)
        rep = eng.branch_gradient()
        assert_logl(rep.log_likelihood, ll)
        assert_vec(rep.branch_gradient, g)


@pytest.mark.parametrize("m,L", [(2, 1), (3, 2), (4, 1), (4, 4), (4, 8), (5, 4), (8, 2), (20, 4), (61, 2)])
def test_gaps_every_kernel(m, L):
    """Missing data (code -1 -> all-ones class column, alignment.hpp:223-224)
    through every kernel family: generic walk_kernel, walk4, walkm."""
    eng, ref = _pair(m, L, 10, 220, 1234 + 10 * m + L, gaps=0.15)
    _check(eng, ref)


@pytest.mark.parametrize("m,L", [(4, 4), (4, 1), (20, 4), (61, 4)])
@pytest.mark.parametrize("taxa", [2, 3])
def test_smallest_trees(m, L, taxa):
    """Two- and three-taxon trees (a root-only schedule; test_engine.cpp:24-35)."""
    eng, ref = _pair(m, L, taxa, 40, 55 + taxa * m + L, gaps=0.1)
    _check(eng, ref)


@pytest.mark.parametrize("m,L", [(4, 4), (6, 2), (20, 4), (61, 1)])
@pytest.mark.parametrize("sites", [1, 5])
def test_single_and_few_patterns(m, L, sites):
    """P smaller than one warp / CTA tile (every lane but a few idle)."""
    eng, ref = _pair(m, L, 9, sites, 700 + m + sites)
    _check(eng, ref)


def _caterpillar_pair(m, L, tips, sites, seed, blen, **opts):
    rng = np.random.default_rng(seed)
    q, pi = _reversible(m, rng)
    mo = O.Model(q, pi, True)
    tree_o = O.Tree.caterpillar(tips, blen)
    rates, probs = O.discrete_gamma(0.5, L) if L > 1 else ([1.0], [1.0])
    codes = O.simulate_states(tree_o, mo, rates, probs, tree_o.branch_lengths, sites, seed + 1)
    labels = [tree_o.labels[i] for i in range(1, tree_o.tip_count + 1)]
    ref = O.Engine(tree_o, O.Alignment.from_codes(codes, m, labels), mo, rates, probs)
    tree = Tree(tree_o.tip_count, tree_o.parent, tree_o.children,
                np.concatenate([[0.0], tree_o.branch_lengths, [0.0]]), tree_o.labels, tree_o.post_order)
    eng = LikelihoodEngine(tree, SitePatternAlignment.from_codes(labels, codes, m), SubstitutionModel(q, pi, True),
                           RateCategories(np.asarray(rates), np.asarray(probs)), EngineOptions(**opts))
    return eng, ref


@pytest.mark.parametrize("m,L,tips,sites", [(20, 4, 400, 24), (61, 2, 300, 12), (4, 4, 700, 6000)])
def test_deep_caterpillar_rescaling(m, L, tips, sites):
    """Caterpillars whose site likelihoods underflow double precision without
    rescaling (test_engine.cpp:341-361) through walkm (20, 61 states) and
    walk4 (4 states, enough patterns for the pipelined kernel)."""
    eng, ref = _caterpillar_pair(m, L, tips, sites, 31 + m, 0.3)
    ll, g, _ = ref.branch_gradient(False)
    assert ll / max(1, sites) < -700.0 or ll < -5000.0  # far below the double range per site
    rep = eng.branch_gradient()
    assert_logl(rep.log_likelihood, ll)
    assert_vec(rep.branch_gradient, g)
    off, _ = _caterpillar_pair(m, L, tips, sites, 31 + m, 0.3, disable_rescaling=True)
    with pytest.raises(pg.RuntimeFailure, match="underflow"):
        off.log_likelihood()


@pytest.mark.parametrize("m", [4, 20, 61])
def test_extreme_branch_lengths(m):
    """Zero-length branches (P = I exactly, substitution.hpp:151: indicator
    tip vectors, zero lanes) and very long ones (P -> stationary rows) through
    every kernel family."""
    rng = np.random.default_rng(5 + m)
    q, pi = _reversible(m, rng)
    mo = O.Model(q, pi, True)
    r = O.Rng(40 + m)
    tree_o = O.Tree.random(r, 12, 0.02, 0.5)
    bl = tree_o.branch_lengths.copy()
    bl[::4] = 0.0
    bl[1::5] = 40.0
    rates, probs = O.discrete_gamma(0.5, 4)
    codes = O.simulate_states(tree_o, mo, rates, probs, bl, 120, 9 + m)  # data consistent with P = I
    labels = [tree_o.labels[i] for i in range(1, tree_o.tip_count + 1)]
    tree_x = O.Tree.from_arrays(tree_o.tip_count, tree_o.parent, tree_o.children, bl, tree_o.post_order)
    ref = O.Engine(tree_x, O.Alignment.from_codes(codes, m, labels), mo, rates, probs)
    tree = Tree(tree_o.tip_count, tree_o.parent, tree_o.children, np.concatenate([[0.0], bl, [0.0]]),
                tree_o.labels, tree_o.post_order)
    eng = LikelihoodEngine(tree, SitePatternAlignment.from_codes(labels, codes, m), SubstitutionModel(q, pi, True),
                           RateCategories(np.asarray(rates), np.asarray(probs)), EngineOptions())
    ll, g, h = ref.branch_gradient(True)
    rep = eng.branch_gradient(True)
    assert_logl(rep.log_likelihood, ll)
    assert_vec(rep.branch_gradient, g)
    assert_vec(rep.hessian_diagonal, h, rtol=1e-8, what="hessian")


@pytest.mark.parametrize("m,L,A", [(20, 4, 2), (20, 4, 6), (20, 4, 14), (12, 4, 3), (16, 2, 1), (24, 4, 5),
                                   (32, 3, 2), (61, 2, 3)])
def test_walkm_ambiguity_classes_table_staging(m, L, A):
    """Tip column tables (NC = MP + A columns) are bulk-copied into shared
    memory when they fit (P x and Q P tables; pg_walkm.cuh `tstage`,
    `qstage`) and gathered per lane otherwise: class counts on both sides of
    each limit, every tip code kind (state, missing, class) mixed."""
    rng = np.random.default_rng(1000 * m + 10 * L + A)
    q, pi = _reversible(m, rng)
    mo = O.Model(q, pi, True)
    r = O.Rng(m + A)
    tree_o = O.Tree.random(r, 11, 0.03, 0.8)
    rates, probs = O.discrete_gamma(0.5, L) if L > 1 else ([1.0], [1.0])
    sites = 157
    codes = np.asarray(O.simulate_states(tree_o, mo, rates, probs, tree_o.branch_lengths, sites, 5 + m))
    u = rng.random(codes.shape)
    codes = np.where(u < 0.15, m + rng.integers(0, A, codes.shape), codes)
    codes = np.where(u > 0.95, -1, codes)
    amb = (rng.random((A, m)) < 0.3).astype(np.float64)
    amb[:, 0] = 1.0  # every class admits at least one state
    w = rng.integers(1, 4, sites)
    labels = [tree_o.labels[i] for i in range(1, tree_o.tip_count + 1)]
    ref = O.Engine(tree_o, O.Alignment.from_patterns(codes, m, w, amb, labels), mo, rates, probs)
    tree = Tree(tree_o.tip_count, tree_o.parent, tree_o.children,
                np.concatenate([[0.0], tree_o.branch_lengths, [0.0]]), tree_o.labels, tree_o.post_order)
    aln = SitePatternAlignment(labels, m, codes, w, amb)
    eng = LikelihoodEngine(tree, aln, SubstitutionModel(q, pi, True),
                           RateCategories(np.asarray(rates), np.asarray(probs)))
    _check(eng, ref)
    assert eng.info()["kernel"] == "walkm_kernel"
