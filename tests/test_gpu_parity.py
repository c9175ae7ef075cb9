"""GPU parity: the sm_100a engine (through the C-ABI) against the CPU oracle
and the reference's known-answer tests (proj/tests/test_engine.cpp cited per
test).  Tolerances are the north star's: 1e-9 relative on logL and on every
gradient component (tests/helpers.py)."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import assert_logl, assert_vec, oracle_for

pytestmark = pytest.mark.gpu

pg = pytest.importorskip("paper_1905_12146_b200")
from workloads import synth  # noqa: E402
from paper_1905_12146_b200.api import (EngineOptions, LikelihoodEngine, RateCategories,  # noqa: E402
                                       SitePatternAlignment, SubstitutionModel, Tree, discrete_gamma_categories,
                                       parse_fasta, parse_newick)


def jc_same(b):
    return 0.25 + 0.75 * math.exp(-4.0 * b / 3.0)


def jc_diff(b):
    return (1.0 - jc_same(b)) / 3.0


SINGLE = RateCategories.single()


def fasta_engine(newick, fasta, model, cats=SINGLE, **opts):
    tree = parse_newick(newick)
    aln = SitePatternAlignment.compress(parse_fasta(fasta))
    return LikelihoodEngine(tree, aln, model, cats, EngineOptions(**opts))


def oracle_pair(tree_o, model_o, cats, sites, seed, capture=False, **opts):
    """Simulate with the oracle (reference draw order), build both engines."""
    rates, probs = cats
    codes = O.simulate_states(tree_o, model_o, rates, probs, tree_o.branch_lengths, sites, seed)
    labels = [tree_o.labels[i] for i in range(1, tree_o.tip_count + 1)]
    aln_o = O.Alignment.from_codes(codes, model_o.m, labels)
    ref = O.Engine(tree_o, aln_o, model_o, rates, probs, **opts)
    tree = Tree(tree_o.tip_count, tree_o.parent, tree_o.children,
                np.concatenate([[0.0], tree_o.branch_lengths, [0.0]]), tree_o.labels, tree_o.post_order)
    aln = SitePatternAlignment.from_codes(labels, codes, model_o.m)
    model = SubstitutionModel(model_o.q, model_o.pi, model_o.reversible)
    for br, q in model_o.branch_q.items():
        model.set_branch_generator(br, q)
    eopts = EngineOptions(capture_partials=capture,
                          force_rescaling=opts.get("force_rescaling", False),
                          disable_rescaling=opts.get("disable_rescaling", False))
    eng = LikelihoodEngine(tree, aln, model, RateCategories(np.asarray(rates), np.asarray(probs)), eopts)
    # integer pattern compression must be bit-exact with the oracle's std::map order
    assert np.array_equal(aln.weights(), aln_o.weights)
    assert np.array_equal(aln.codes.astype(np.int32), aln_o.pattern_codes())
    return eng, ref


# -------------------------------------------------------------- closed forms
def test_two_taxon_closed_form():  # test_engine.cpp:24-35, :189-204
    eng = fasta_engine("(A:0.1,B:0.2);", ">A\nA\n>B\nC\n", SubstitutionModel.jc69())
    site = 0.25 * jc_diff(0.3)
    assert abs(eng.log_likelihood() - math.log(site)) < 1e-14
    rep = eng.branch_gradient()
    b = 0.3
    expected = math.exp(-4 * b / 3) / (0.75 * (1 - math.exp(-4 * b / 3)))
    assert rep.branch_gradient[0] == pytest.approx(expected, rel=1e-12)
    assert rep.branch_gradient[1] == pytest.approx(expected, rel=1e-12)


def test_fig1_partials():  # test_engine.cpp:37-72
    model = SubstitutionModel.hky85(2.0, [0.3, 0.2, 0.2, 0.3])
    eng = fasta_engine("((A:0.1,B:0.2):0.05,C:0.3);", ">A\nA\n>B\nC\n>C\nG\n", model, capture_partials=True)
    mo = O.Model.hky85(2.0, [0.3, 0.2, 0.2, 0.3])
    p = lambda br, b: mo.transition_matrix(br, b)
    e = np.eye(4)
    p4 = (p(1, 0.1) @ e[0]) * (p(2, 0.2) @ e[1])
    p5 = (p(4, 0.05) @ p4) * (p(3, 0.3) @ e[2])
    assert abs(eng.log_likelihood() - math.log(model.root_distribution() @ p5)) < 1e-13
    eng.branch_gradient()
    np.testing.assert_allclose(eng.post_partial(4, 0)[:, 0], p4, rtol=1e-14)
    assert np.array_equal(eng.pre_partial(5, 0)[:, 0], model.root_distribution())
    q4 = p(4, 0.05).T @ (model.root_distribution() * (p(3, 0.3) @ e[2]))
    np.testing.assert_allclose(eng.pre_partial(4, 0)[:, 0], q4, rtol=1e-14)


def test_zero_length_indicator_and_all_gap():  # test_engine.cpp:74-90
    eng = fasta_engine("((A:0.0,B:0.0):0.0,C:0.0);", ">A\nG\n>B\nG\n>C\nG\n", SubstitutionModel.jc69())
    assert abs(eng.log_likelihood() - math.log(0.25)) < 1e-14
    eng = fasta_engine("((A:0.4,B:0.9):0.2,C:0.3);", ">A\n-\n>B\n-\n>C\n-\n",
                       SubstitutionModel.hky85(3.0, [0.4, 0.1, 0.3, 0.2]), discrete_gamma_categories(0.5, 4))
    assert abs(eng.log_likelihood()) < 1e-12


def test_iupac_ambiguity_matches_oracle():  # test_alignment.cpp:38-50 through the engine
    fasta = ">A\nRAC-NY\n>B\nAAGTCC\n>C\nGWCTAS\n"
    eng = fasta_engine("((A:0.1,B:0.2):0.05,C:0.3);", fasta, SubstitutionModel.hky85(2.0, [0.3, 0.2, 0.2, 0.3]),
                       discrete_gamma_categories(0.8, 4))
    tree = O.Tree.parse("((A:0.1,B:0.2):0.05,C:0.3);")
    ref = O.Engine(tree, O.Alignment.from_fasta(fasta), O.Model.hky85(2.0, [0.3, 0.2, 0.2, 0.3]),
                   *O.discrete_gamma(0.8, 4))
    ll, g, h = ref.branch_gradient(True)
    rep = eng.branch_gradient(True)
    assert_logl(rep.log_likelihood, ll)
    assert_vec(rep.branch_gradient, g)
    assert_vec(rep.hessian_diagonal, h, what="hessian")


# ---------------------------------------------------------- random instances
def test_brute_force_random_instances():  # test_engine.cpp:92-105
    rng = O.Rng(2024)
    mo = O.Model.hky85(2.0, [0.3, 0.25, 0.25, 0.2])
    for trial in range(25):
        tips = 2 + rng.next() % 4
        tree = O.Tree.random(rng, tips, 0.0, 2.0)
        cats = ([1.0], [1.0]) if trial % 2 == 0 else O.discrete_gamma(0.7, 4)
        eng, ref = oracle_pair(tree, mo, cats, 30, 100 + trial)
        exact = O.brute_force_log_likelihood(tree, ref.aln, mo, *cats, tree.branch_lengths)
        assert abs(eng.log_likelihood() - exact) <= 1e-12 * abs(exact)


@pytest.mark.parametrize("trial", range(12))
def test_gradient_matches_oracle_random(trial):  # test_engine.cpp:219-239 (engine vs oracle, then FD)
    rng = O.Rng(404 + trial)
    mo = O.Model.gtr([1.2, 2.8, 0.7, 1.1, 3.5, 1.0], [0.35, 0.2, 0.15, 0.3])
    tips = 3 + rng.next() % 30
    tree = O.Tree.random(rng, tips, 0.02, 1.2)
    cats = ([1.0], [1.0]) if trial % 2 == 0 else O.discrete_gamma(0.8, 4)
    eng, ref = oracle_pair(tree, mo, cats, 60, 900 + trial)
    ll, g, h = ref.branch_gradient(True)
    rep = eng.branch_gradient(True)
    assert_logl(rep.log_likelihood, ll)
    assert_vec(rep.branch_gradient, g)
    assert_vec(rep.hessian_diagonal, h, rtol=1e-8, what="hessian")


def test_likelihood_at_every_node():  # test_engine.cpp:133-147 (Eq. 8)
    rng = O.Rng(77)
    mo = O.Model.hky85(2.5, [0.35, 0.15, 0.25, 0.25])
    for trial in range(20):
        tips = 3 + rng.next() % 14
        tree = O.Tree.random(rng, tips, 0.0, 1.5)
        cats = O.discrete_gamma(0.6, 4) if trial % 3 == 0 else ([1.0], [1.0])
        eng, _ = oracle_pair(tree, mo, cats, 20, 500 + trial, capture=True)
        ref = eng.log_likelihood()
        for node in range(1, tree.node_count + 1):
            v = eng.log_likelihood_at_node(node)
            assert abs(v - ref) <= 1e-12 + 1e-10 * abs(ref), (trial, node, v, ref)


def test_nonreversible_branch_generator():  # test_engine.cpp:241-253 (Pade path on the GPU)
    q = np.array([[-3, 1, 1, 1], [2, -4, 1, 1], [1, 1, -2, 0], [3, 1, 2, -6]], float)
    fasta = ">A\nACGTA\n>B\nACGGC\n>C\nATG-C\n"
    model = SubstitutionModel.jc69()
    model.set_branch_generator(2, q)
    eng = fasta_engine("((A:0.2,B:0.4):0.1,C:0.3);", fasta, model)
    mo = O.Model.jc69()
    mo.set_branch_generator(2, q)
    ref = O.Engine(O.Tree.parse("((A:0.2,B:0.4):0.1,C:0.3);"), O.Alignment.from_fasta(fasta), mo, [1.0], [1.0])
    ll, g, h = ref.branch_gradient(True)
    rep = eng.branch_gradient(True)
    assert_logl(rep.log_likelihood, ll)
    assert_vec(rep.branch_gradient, g)
    assert_vec(rep.hessian_diagonal, h, rtol=1e-8, what="hessian")
    fd = O.fd_branch_gradient(ref, 1e-5)
    assert np.all(np.abs(rep.branch_gradient - fd) <= 1e-8 + 1e-6 * np.abs(fd))


def test_single_category_equals_degenerate_mixture():  # test_engine.cpp:284-300
    rng = O.Rng(15)
    tree = O.Tree.random(rng, 5, 0.05, 0.7)
    mo = O.Model.jc69()
    a, _ = oracle_pair(tree, mo, ([1.0], [1.0]), 30, 5)
    b, _ = oracle_pair(tree, mo, ([1.0, 1.0], [0.5, 0.5]), 30, 5)
    assert a.log_likelihood() == pytest.approx(b.log_likelihood(), rel=1e-14)
    ra, rb = a.branch_gradient(True), b.branch_gradient(True)
    assert np.linalg.norm(ra.branch_gradient - rb.branch_gradient) <= 1e-13 * np.linalg.norm(ra.branch_gradient)
    assert np.linalg.norm(ra.hessian_diagonal - rb.hessian_diagonal) <= 1e-13 * np.linalg.norm(ra.hessian_diagonal)


def test_node_visits_and_caching():  # test_engine.cpp:302-322; engine.hpp:116-124
    rng = O.Rng(52)
    mo = O.Model.jc69()
    for tips in (4, 9, 17):
        tree = O.Tree.random(rng, tips, 0.05, 0.6)
        eng, _ = oracle_pair(tree, mo, ([1.0], [1.0]), 25, tips)
        eng.reset_node_visits()
        eng.branch_gradient()
        assert eng.node_visits() == 2 * (2 * tips - 1)
        eng.branch_gradient()  # cached: no new visits
        assert eng.node_visits() == 2 * (2 * tips - 1)
        eng.set_branch_lengths(eng.branch_lengths())  # bit-identical: caches stay valid
        eng.branch_gradient()
        assert eng.node_visits() == 2 * (2 * tips - 1)
        eng.invalidate_caches()
        eng.branch_gradient()
        assert eng.node_visits() == 4 * (2 * tips - 1)


def test_rescaling_neutral_and_deep_trees():  # test_engine.cpp:324-361
    rng = O.Rng(99)
    tree = O.Tree.random(rng, 12, 0.1, 1.5)
    mo = O.Model.jc69()
    cats = O.discrete_gamma(0.8, 4)
    plain, ref = oracle_pair(tree, mo, cats, 40, 3)
    forced, _ = oracle_pair(tree, mo, cats, 40, 3, force_rescaling=True)
    off, _ = oracle_pair(tree, mo, cats, 40, 3, disable_rescaling=True)
    r = plain.log_likelihood()
    assert_logl(r, ref.log_likelihood())
    assert forced.log_likelihood() == pytest.approx(r, rel=1e-12)
    assert off.log_likelihood() == pytest.approx(r, rel=1e-12)
    a, b = plain.branch_gradient(True), forced.branch_gradient(True)
    assert np.linalg.norm(a.branch_gradient - b.branch_gradient) <= 1e-12 * np.linalg.norm(a.branch_gradient)
    assert np.linalg.norm(a.hessian_diagonal - b.hessian_diagonal) <= 1e-10 * np.linalg.norm(a.hessian_diagonal)

    deep = O.Tree.caterpillar(600, 0.4)
    eng, ref = oracle_pair(deep, mo, ([1.0], [1.0]), 3, 12)
    dll = eng.log_likelihood()
    assert math.isfinite(dll) and dll < -1000.0
    assert_logl(dll, ref.log_likelihood())
    ll, g, _ = ref.branch_gradient()
    assert_vec(eng.branch_gradient().branch_gradient, g)
    broken, _ = oracle_pair(deep, mo, ([1.0], [1.0]), 3, 12, disable_rescaling=True)
    with pytest.raises(pg.RuntimeFailure, match="underflow"):
        broken.log_likelihood()


def test_binding_and_staleness_errors():  # test_engine.cpp:363-382
    model = SubstitutionModel.jc69()
    aln = SitePatternAlignment.compress(parse_fasta(">A\nAC\n>B\nGT\n"))
    with pytest.raises(pg.InvalidArgument, match="not found"):
        LikelihoodEngine(parse_newick("(A:0.1,Mismatch:0.2);"), aln, model, SINGLE)
    extra = SitePatternAlignment.compress(parse_fasta(">A\nAC\n>B\nGT\n>C\nGG\n"))
    with pytest.raises(pg.InvalidArgument, match="one record per tree tip"):
        LikelihoodEngine(parse_newick("(A:0.1,B:0.2);"), extra, model, SINGLE)
    eng = LikelihoodEngine(parse_newick("(A:0.1,B:0.2);"), aln, model, SINGLE)
    eng.log_likelihood()
    eng.set_branch_lengths([0.3, 0.1])
    with pytest.raises(pg.LogicError):
        eng.pre_order_pass()
    with pytest.raises(pg.InvalidArgument):
        eng.set_branch_lengths([-0.1, 0.2])
    eng.post_order_pass()
    eng.pre_order_pass()


# ------------------------------------------------------ state / category zoo
@pytest.mark.parametrize("m,L", [(2, 1), (3, 2), (4, 3), (4, 8), (6, 1), (6, 4), (20, 4), (20, 1), (32, 2), (61, 4)])
def test_state_and_category_layouts(m, L):
    rng = np.random.default_rng(1000 * m + L)
    pi = rng.dirichlet(np.ones(m) * 3)
    s = rng.lognormal(0, 0.5, (m, m))
    s = (s + s.T) / 2
    q = s * pi[None, :]
    np.fill_diagonal(q, 0)
    np.fill_diagonal(q, -q.sum(1))
    q /= -np.sum(pi * np.diag(q))
    mo = O.Model(q, pi, True)
    r = O.Rng(m * 31 + L)
    tree = O.Tree.random(r, 9, 0.02, 0.6)
    cats = O.discrete_gamma(0.6, L) if L > 1 else ([1.0], [1.0])
    eng, ref = oracle_pair(tree, mo, cats, 70, 17)
    ll, g, h = ref.branch_gradient(True)
    rep = eng.branch_gradient(True)
    assert_logl(rep.log_likelihood, ll)
    assert_vec(rep.branch_gradient, g)
    assert_vec(rep.hessian_diagonal, h, rtol=1e-8, what="hessian")


# --------------------------------------------------------- config workloads
def _check_instance(inst, blocks=8, hess=True):
    eng = synth.engine_for(inst)
    ref = oracle_for(inst, blocks=blocks)
    ll, g, h = ref.branch_gradient(hess)
    rep = eng.branch_gradient(hess)
    assert_logl(rep.log_likelihood, ll)
    assert_vec(rep.branch_gradient, g)
    if hess:
        assert_vec(rep.hessian_diagonal, h, rtol=1e-8, what="hessian")
    return eng, rep, (ll, g, h)


def test_config_c1_full():
    _check_instance(synth.generate("C1"))


def test_config_c2_full():  # 512 taxa, GTR+G4, 2% gaps, 20k columns
    _check_instance(synth.generate("C2"))


def test_config_c3_sample_rates():  # non-reversible Pade path + clock chain rule
    inst = synth.generate("C3", sites=3000)
    eng, rep, (ll, g, h) = _check_instance(inst, hess=False)
    rr = eng.rate_gradient()
    assert_vec(rr.branch_gradient, inst.durations * g, what="rate gradient")


def test_config_c4_sample():  # 20-state
    _check_instance(synth.generate("C4", sites=1500, tips=200), hess=False)


def test_config_c5_sample():  # 61-state codon
    _check_instance(synth.generate("C5", sites=300, tips=64), hess=False)


def test_pattern_split_linearity_full_c3():
    """Size-independent property at full C3 size: logL and the gradient are
    sums over patterns, so two shards evaluated separately add up to the whole
    (the multi-GPU contract)."""
    inst = synth.generate("C3", sites=200000)
    whole = synth.engine_for(inst).branch_gradient()
    P = inst.patterns
    a = synth.engine_for(inst.slice_patterns(0, P // 3)).branch_gradient()
    b = synth.engine_for(inst.slice_patterns(P // 3, P)).branch_gradient()
    assert_logl(a.log_likelihood + b.log_likelihood, whole.log_likelihood, rtol=1e-12)
    assert_vec(a.branch_gradient + b.branch_gradient, whole.branch_gradient, rtol=1e-11, what="sharded gradient")


def test_compressed_equals_raw_sites_gpu():  # test_engine.cpp:107-131 through the product
    rng = O.Rng(31)
    tree_o = O.Tree.random(rng, 6, 0.05, 0.8)
    mo = O.Model.jc69()
    cats = O.discrete_gamma(0.9, 4)
    codes = O.simulate_states(tree_o, mo, *cats, tree_o.branch_lengths, 400, 9)
    labels = [tree_o.labels[i] for i in range(1, 7)]
    tree = Tree(6, tree_o.parent, tree_o.children, np.concatenate([[0.0], tree_o.branch_lengths, [0.0]]),
                tree_o.labels, tree_o.post_order)
    model = SubstitutionModel.jc69()
    rc = RateCategories(np.asarray(cats[0]), np.asarray(cats[1]))
    comp = SitePatternAlignment.from_codes(labels, codes, 4)
    assert comp.pattern_count() < 400
    whole = LikelihoodEngine(tree, comp, model, rc).log_likelihood()
    raw = SitePatternAlignment(labels, 4, codes.astype(np.int8), np.ones(400, np.int64))
    assert LikelihoodEngine(tree, raw, model, rc).log_likelihood() == pytest.approx(whole, rel=1e-12)


def test_linear_time_scaling_exponent():
    """acceptance.cpp:172-217 / SPEC.md:575: analytic-gradient wall time grows
    linearly in N (fitted log-log exponent < 1.3) at 1000 sites."""
    import time

    ns, ts = [], []
    for tips in (64, 128, 256, 512, 1024):
        inst = synth.generate("C1", seed=tips, sites=1000, tips=tips)
        eng = synth.engine_for(inst)
        eng.branch_gradient()
        best = 1e9
        for _ in range(5):
            eng.invalidate_caches()
            t0 = time.perf_counter()
            eng.branch_gradient()
            best = min(best, time.perf_counter() - t0)
        ns.append(tips)
        ts.append(best)
    slope = np.polyfit(np.log(ns), np.log(ts), 1)[0]
    assert slope < 1.3, (slope, ts)


@pytest.mark.parametrize("m,L", [(4, 1), (4, 4), (20, 4), (61, 2)])
def test_zero_patterns(m, L):
    """An alignment with no columns (alignment.hpp:186-229 gives no patterns):
    logL 0 and a zero gradient / Hessian on every kernel family, like the
    oracle (sums over an empty pattern set, engine.hpp:206-218, :267-268)."""
    r = O.Rng(5)
    tree_o = O.Tree.random(r, 6, 0.05, 0.5)
    rng = np.random.default_rng(m)
    pi = rng.dirichlet(np.ones(m))
    q = rng.lognormal(0, 0.5, (m, m)) * pi[None, :]
    np.fill_diagonal(q, 0)
    np.fill_diagonal(q, -q.sum(1))
    rates, probs = O.discrete_gamma(0.5, L) if L > 1 else ([1.0], [1.0])
    labels = [tree_o.labels[i] for i in range(1, tree_o.tip_count + 1)]
    codes = np.zeros((tree_o.tip_count, 0), np.int8)
    ref = O.Engine(tree_o, O.Alignment.from_patterns(codes.astype(np.int32), m, np.zeros(0, np.int64), None, labels),
                   O.Model(q, pi, False), rates, probs)
    ll, g, h = ref.branch_gradient(True)
    tree = Tree(tree_o.tip_count, tree_o.parent, tree_o.children,
                np.concatenate([[0.0], tree_o.branch_lengths, [0.0]]), tree_o.labels, tree_o.post_order)
    eng = LikelihoodEngine(tree, SitePatternAlignment(labels, m, codes, np.zeros(0, np.int64)),
                           SubstitutionModel(q, pi, False), RateCategories(np.asarray(rates), np.asarray(probs)))
    rep = eng.branch_gradient(True)
    assert ll == 0.0 and rep.log_likelihood == 0.0
    assert np.all(rep.branch_gradient == 0.0) and np.all(g == 0.0)
    assert np.all(rep.hessian_diagonal == 0.0) and rep.pattern_count == 0
