"""Pins the CPU oracle against the reference's own known-answer tests.

Each test restates one TEST_CASE from /root/reference/proj/tests/*.cpp (cited
per test) with the same constants and tolerances.  Passing these is what makes
the oracle a *pinned* restatement of the reference.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O


def jc_same(b):
    return 0.25 + 0.75 * math.exp(-4.0 * b / 3.0)


def jc_diff(b):
    return (1.0 - jc_same(b)) / 3.0


def taylor_expm(a, terms=60):
    s = np.eye(a.shape[0])
    pw = s.copy()
    for k in range(1, terms + 1):
        pw = pw @ a / k
        s = s + pw
    return s


def random_alignment(tree, model, rates, probs, sites, seed):
    """test_engine.cpp:121-128: compress(simulate_alignment(...)); from_codes keys
    the same first-occurrence pattern order as the character-column compress."""
    codes = O.simulate_states(tree, model, rates, probs, tree.branch_lengths, sites, seed)
    labels = [tree.labels[i] for i in range(1, tree.tip_count + 1)]
    return O.Alignment.from_codes(codes, model.m, labels)


SINGLE = ([1.0], [1.0])


# ----------------------------------------------------------------- engine KATs
def test_two_taxon_closed_form_likelihood():  # test_engine.cpp:24-35
    tree = O.Tree.parse("(A:0.1,B:0.2);")
    aln = O.Alignment.from_fasta(">A\nA\n>B\nC\n")
    eng = O.Engine(tree, aln, O.Model.jc69(), *SINGLE)
    site = 0.25 * jc_diff(0.3)
    assert abs(site - 0.0206050) < 5e-8
    assert abs(eng.log_likelihood() - math.log(site)) < 1e-14
    assert abs(math.log(site) - (-3.8822216538)) < 5e-10


def test_fig1_post_order_update():  # test_engine.cpp:37-55
    tree = O.Tree.parse("((A:0.1,B:0.2):0.05,C:0.3);")
    model = O.Model.hky85(2.0, [0.3, 0.2, 0.2, 0.3])
    aln = O.Alignment.from_fasta(">A\nA\n>B\nC\n>C\nG\n")
    eng = O.Engine(tree, aln, model, *SINGLE)
    eng.post_order_pass()
    p = lambda br: model.transition_matrix(br, tree.branch_lengths[br - 1])
    p1, p2, p3 = (aln.tip_partials(aln.taxon_index(x))[:, 0] for x in "ABC")
    p4 = (p(1) @ p1) * (p(2) @ p2)
    np.testing.assert_allclose(eng.post_partial(4, 0)[:, 0], p4, rtol=1e-14)
    p5 = (p(4) @ p4) * (p(3) @ p3)
    assert abs(eng.log_likelihood() - math.log(model.pi @ p5)) < 1e-13


def test_pre_order_root_and_fig1():  # test_engine.cpp:57-72
    tree = O.Tree.parse("((A:0.1,B:0.2):0.05,C:0.3);")
    model = O.Model.hky85(2.0, [0.3, 0.2, 0.2, 0.3])
    aln = O.Alignment.from_fasta(">A\nA\n>B\nC\n>C\nG\n")
    eng = O.Engine(tree, aln, model, *SINGLE)
    eng.branch_gradient()
    assert np.array_equal(eng.pre_partial(5, 0)[:, 0], model.pi)
    p = lambda br: model.transition_matrix(br, tree.branch_lengths[br - 1])
    p3 = aln.tip_partials(aln.taxon_index("C"))[:, 0]
    q4 = p(4).T @ (model.pi * (p(3) @ p3))
    np.testing.assert_allclose(eng.pre_partial(4, 0)[:, 0], q4, rtol=1e-14)


def test_zero_length_indicator():  # test_engine.cpp:74-82
    tree = O.Tree.parse("((A:0.0,B:0.0):0.0,C:0.0);")
    aln = O.Alignment.from_fasta(">A\nG\n>B\nG\n>C\nG\n")
    eng = O.Engine(tree, aln, O.Model.jc69(), *SINGLE)
    eng.post_order_pass()
    assert np.array_equal(eng.post_partial(5, 0)[:, 0], [0, 0, 1, 0])
    assert abs(eng.log_likelihood() - math.log(0.25)) < 1e-14


def test_all_gap_zero():  # test_engine.cpp:84-90
    tree = O.Tree.parse("((A:0.4,B:0.9):0.2,C:0.3);")
    model = O.Model.hky85(3.0, [0.4, 0.1, 0.3, 0.2])
    aln = O.Alignment.from_fasta(">A\n-\n>B\n-\n>C\n-\n")
    eng = O.Engine(tree, aln, model, *O.discrete_gamma(0.5, 4))
    assert abs(eng.log_likelihood()) < 1e-12


def test_brute_force_random_instances():  # test_engine.cpp:92-105
    rng = O.Rng(2024)
    model = O.Model.hky85(2.0, [0.3, 0.25, 0.25, 0.2])
    for trial in range(25):
        tips = 2 + rng.next() % 4
        tree = O.Tree.random(rng, tips, 0.0, 2.0)
        cats = SINGLE if trial % 2 == 0 else O.discrete_gamma(0.7, 4)
        aln = random_alignment(tree, model, *cats, 30, 100 + trial)
        eng = O.Engine(tree, aln, model, *cats)
        exact = O.brute_force_log_likelihood(tree, aln, model, *cats, eng.branch_lengths)
        assert abs(eng.log_likelihood() - exact) <= 1e-12 * abs(exact)


def test_compressed_equals_raw_sites():  # test_engine.cpp:107-131
    rng = O.Rng(31)
    tree = O.Tree.random(rng, 6, 0.05, 0.8)
    model = O.Model.jc69()
    cats = O.discrete_gamma(0.9, 4)
    codes = O.simulate_states(tree, model, *cats, tree.branch_lengths, 400, 9)
    labels = [tree.labels[i] for i in range(1, 7)]
    comp = O.Alignment.from_codes(codes, 4, labels)
    assert comp.pattern_count < 400
    raw_total = sum(O.Engine(tree, O.Alignment.from_codes(codes[:, s:s + 1], 4, labels), model, *cats).log_likelihood()
                    for s in range(400))
    ll = O.Engine(tree, comp, model, *cats).log_likelihood()
    assert ll == pytest.approx(raw_total, rel=1e-12)


def test_likelihood_recoverable_at_every_node():  # test_engine.cpp:133-147 (Eq. 8)
    rng = O.Rng(77)
    model = O.Model.hky85(2.5, [0.35, 0.15, 0.25, 0.25])
    for trial in range(100):
        tips = 3 + rng.next() % 14
        tree = O.Tree.random(rng, tips, 0.0, 1.5)
        cats = O.discrete_gamma(0.6, 4) if trial % 3 == 0 else SINGLE
        aln = random_alignment(tree, model, *cats, 20, 500 + trial)
        eng = O.Engine(tree, aln, model, *cats)
        ref = eng.log_likelihood()
        for node in range(1, tree.node_count + 1):
            v = eng.log_likelihood_at_node(node)
            assert abs(v - ref) <= 1e-12 + 1e-10 * abs(ref)


def test_scratch_route_matches_cached_and_shuffled():  # test_engine.cpp:149-187
    rng = O.Rng(271)
    model = O.Model.hky85(2.0, [0.3, 0.25, 0.25, 0.2])
    for trial in range(10):
        tips = 3 + rng.next() % 20
        tree = O.Tree.random(rng, tips, 0.01, 1.0)
        cats = SINGLE if trial % 2 == 0 else O.discrete_gamma(0.7, 4)
        aln = random_alignment(tree, model, *cats, 50, 40 + trial)
        eng = O.Engine(tree, aln, model, *cats)
        scratch = eng.log_likelihood()
        eng.post_order_pass()
        assert eng.log_likelihood() == pytest.approx(scratch, rel=1e-14)
        order = tree.random_post_order(rng)
        variant = O.Tree.from_arrays(tree.tip_count, tree.parent, tree.children, tree.branch_lengths, order)
        shuffled = O.Engine(variant, aln, model, *cats)
        assert shuffled.log_likelihood() == pytest.approx(scratch, rel=1e-12)


def test_two_taxon_gradient_closed_form():  # test_engine.cpp:189-204
    tree = O.Tree.parse("(A:0.1,B:0.2);")
    aln = O.Alignment.from_fasta(">A\nA\n>B\nC\n")
    eng = O.Engine(tree, aln, O.Model.jc69(), *SINGLE)
    _, g, _ = eng.branch_gradient()
    b = 0.3
    expected = math.exp(-4 * b / 3) / (0.75 * (1 - math.exp(-4 * b / 3)))
    assert g[0] == pytest.approx(expected, rel=1e-12)
    assert g[1] == pytest.approx(expected, rel=1e-12)
    fd = O.fd_branch_gradient(eng, 1e-5)
    assert abs(g[0] - fd[0]) < 1e-7


def test_root_children_gradients_coincide():  # test_engine.cpp:206-217
    rng = O.Rng(8)
    tree = O.Tree.random(rng, 6, 0.05, 0.9)
    model = O.Model.hky85(2.0, [0.3, 0.2, 0.3, 0.2])
    aln = random_alignment(tree, model, *SINGLE, 50, 21)
    _, g, _ = O.Engine(tree, aln, model, *SINGLE).branch_gradient()
    left, right = tree.children[tree.root]
    assert g[left - 1] == pytest.approx(g[right - 1], rel=1e-10)


def test_gradient_vs_finite_differences():  # test_engine.cpp:219-239
    rng = O.Rng(404)
    model = O.Model.gtr([1.2, 2.8, 0.7, 1.1, 3.5, 1.0], [0.35, 0.2, 0.15, 0.3])
    for trial in range(12):
        tips = 3 + rng.next() % 14
        tree = O.Tree.random(rng, tips, 0.02, 1.2)
        cats = SINGLE if trial % 2 == 0 else O.discrete_gamma(0.8, 4)
        aln = random_alignment(tree, model, *cats, 40, 900 + trial)
        eng = O.Engine(tree, aln, model, *cats)
        _, g, _ = eng.branch_gradient()
        fd = O.fd_branch_gradient(eng, 1e-5)
        for i in range(len(fd)):
            if abs(fd[i]) > 1e-3:
                assert g[i] == pytest.approx(fd[i], rel=1e-5)
            else:
                assert abs(g[i] - fd[i]) < 1e-5


def test_nonreversible_branch_generator_gradient():  # test_engine.cpp:241-253
    tree = O.Tree.parse("((A:0.2,B:0.4):0.1,C:0.3);")
    model = O.Model.jc69()
    q = np.array([[-3, 1, 1, 1], [2, -4, 1, 1], [1, 1, -2, 0], [3, 1, 2, -6]], float)
    model.set_branch_generator(2, q)
    aln = O.Alignment.from_fasta(">A\nACGTA\n>B\nACGGC\n>C\nATG-C\n")
    eng = O.Engine(tree, aln, model, *SINGLE)
    _, g, _ = eng.branch_gradient()
    fd = O.fd_branch_gradient(eng, 1e-5)
    for i in range(len(fd)):
        assert abs(g[i] - fd[i]) <= 1e-8 + 1e-6 * abs(fd[i])


def test_hessian_vs_fd():  # test_engine.cpp:255-282
    rng = O.Rng(606)
    tree = O.Tree.parse("(A:0.15,B:0.2);")
    aln = O.Alignment.from_fasta(">A\nA\n>B\nC\n")
    eng = O.Engine(tree, aln, O.Model.jc69(), *SINGLE)
    _, _, h = eng.branch_gradient(True)
    fd = O.fd_branch_hessian_diagonal(eng, 1e-4)
    np.testing.assert_allclose(h, fd, rtol=1e-4)

    tree = O.Tree.random(rng, 8, 0.05, 0.8)
    model = O.Model.gtr([0.9, 2.2, 1.4, 0.8, 2.9, 1.0], [0.3, 0.25, 0.2, 0.25])
    cats = O.discrete_gamma(0.5, 4)
    aln = random_alignment(tree, model, *cats, 80, 77)
    eng = O.Engine(tree, aln, model, *cats)
    _, _, h = eng.branch_gradient(True)
    fd = O.fd_branch_hessian_diagonal(eng, 1e-4)
    np.testing.assert_allclose(h, fd, rtol=1e-3)


def test_single_category_equals_degenerate_mixture():  # test_engine.cpp:284-300
    rng = O.Rng(15)
    tree = O.Tree.random(rng, 5, 0.05, 0.7)
    model = O.Model.jc69()
    aln = random_alignment(tree, model, *SINGLE, 30, 5)
    a = O.Engine(tree, aln, model, *SINGLE)
    b = O.Engine(tree, aln, model, [1.0, 1.0], [0.5, 0.5])
    assert a.log_likelihood() == pytest.approx(b.log_likelihood(), rel=1e-14)
    _, ga, ha = a.branch_gradient(True)
    _, gb, hb = b.branch_gradient(True)
    assert np.linalg.norm(ga - gb) <= 1e-13 * min(np.linalg.norm(ga), np.linalg.norm(gb))
    assert np.linalg.norm(ha - hb) <= 1e-13 * min(np.linalg.norm(ha), np.linalg.norm(hb))


def test_node_visit_counts_linear():  # test_engine.cpp:302-322
    rng = O.Rng(52)
    model = O.Model.jc69()
    for tips in (4, 9, 17):
        tree = O.Tree.random(rng, tips, 0.05, 0.6)
        aln = random_alignment(tree, model, *SINGLE, 25, tips)
        eng = O.Engine(tree, aln, model, *SINGLE)
        eng.reset_node_visits()
        eng.branch_gradient()
        assert eng.node_visits() == 2 * (2 * tips - 1)


def test_rescaling_neutral_and_deep_trees():  # test_engine.cpp:324-361
    rng = O.Rng(99)
    tree = O.Tree.random(rng, 12, 0.1, 1.5)
    model = O.Model.jc69()
    cats = O.discrete_gamma(0.8, 4)
    aln = random_alignment(tree, model, *cats, 40, 3)
    plain = O.Engine(tree, aln, model, *cats)
    scaled = O.Engine(tree, aln, model, *cats, force_rescaling=True)
    unscaled = O.Engine(tree, aln, model, *cats, disable_rescaling=True)
    ref = plain.log_likelihood()
    assert scaled.log_likelihood() == pytest.approx(ref, rel=1e-12)
    assert unscaled.log_likelihood() == pytest.approx(ref, rel=1e-12)
    _, ga, ha = plain.branch_gradient(True)
    _, gb, hb = scaled.branch_gradient(True)
    assert np.linalg.norm(ga - gb) <= 1e-12 * np.linalg.norm(ga)
    assert np.linalg.norm(ha - hb) <= 1e-10 * np.linalg.norm(ha)

    deep = O.Tree.caterpillar(600, 0.4)
    codes = O.simulate_states(deep, model, *SINGLE, np.full(deep.branch_count, 0.4), 3, 12)
    labels = [deep.labels[i] for i in range(1, 601)]
    daln = O.Alignment.from_codes(codes, 4, labels)
    dll = O.Engine(deep, daln, model, *SINGLE).log_likelihood()
    assert math.isfinite(dll) and dll < -1000.0
    with pytest.raises(O.OracleError, match="underflow"):
        O.Engine(deep, daln, model, *SINGLE, disable_rescaling=True).log_likelihood()


def test_binding_errors():  # test_engine.cpp:363-382
    model = O.Model.jc69()
    aln = O.Alignment.from_fasta(">A\nAC\n>B\nGT\n")
    with pytest.raises(O.OracleInvalidArgument, match="not found"):
        O.Engine(O.Tree.parse("(A:0.1,Mismatch:0.2);"), aln, model, *SINGLE)
    extra = O.Alignment.from_fasta(">A\nAC\n>B\nGT\n>C\nGG\n")
    with pytest.raises(O.OracleInvalidArgument, match="one record per tree tip"):
        O.Engine(O.Tree.parse("(A:0.1,B:0.2);"), extra, model, *SINGLE)
    eng = O.Engine(O.Tree.parse("(A:0.1,B:0.2);"), aln, model, *SINGLE)
    eng.log_likelihood()
    eng.set_branch_lengths([0.3, 0.1])
    with pytest.raises(O.OracleLogicError):
        eng.pre_order_pass()
    with pytest.raises(O.OracleInvalidArgument):
        eng.set_branch_lengths([-0.1, 0.2])


# ----------------------------------------------------------- substitution KATs
def test_jc_generator_and_degeneracies():  # test_substitution.cpp:10-26
    q = O.Model.jc69().q
    np.testing.assert_allclose(q, np.where(np.eye(4) > 0, -1.0, 1.0 / 3.0), atol=1e-14)
    np.testing.assert_allclose(O.Model.hky85(1.0, [0.25] * 4).q, q, atol=1e-14)
    np.testing.assert_allclose(O.Model.gtr([2.5] * 6, [0.25] * 4).q, q, atol=1e-14)


def test_named_generator_invariants():  # test_substitution.cpp:28-50
    rng = O.Rng(3)
    for _ in range(20):
        exch = [rng.uniform(0.2, 3.0) for _ in range(6)]
        f = np.array([rng.uniform(0.2, 3.0) for _ in range(4)])
        f /= f.sum()
        m = O.Model.gtr(exch, f)
        assert np.all(np.abs(m.q.sum(1)) < 1e-12)
        assert -np.sum(f * np.diag(m.q)) == pytest.approx(1.0, rel=1e-12)
        assert np.linalg.norm(m.pi @ m.q) < 1e-12


def test_transition_matrix_closed_forms():  # test_substitution.cpp:52-71
    m = O.Model.jc69()
    assert np.array_equal(m.transition_matrix(1, 0.0), np.eye(4))
    p = m.transition_matrix(1, 0.3)
    np.testing.assert_allclose(p, np.where(np.eye(4) > 0, jc_same(0.3), jc_diff(0.3)), rtol=1e-12)
    np.testing.assert_allclose(m.transition_matrix(1, 100.0), 0.25, atol=1e-10)
    with pytest.raises(O.OracleInvalidArgument):
        m.transition_matrix(1, -0.1)
    with pytest.raises(O.OracleInvalidArgument):
        m.transition_matrix(1, 0.1, 0.0)


def test_row_stochastic():  # test_substitution.cpp:73-89
    rng = O.Rng(5)
    for _ in range(10):
        exch = [rng.uniform(0.2, 3.0) for _ in range(6)]
        f = np.array([rng.uniform(0.2, 3.0) for _ in range(4)])
        f /= f.sum()
        m = O.Model.gtr(exch, f)
        for b in (0.0, 1e-8, 0.05, 0.7, 5.0, 40.0):
            p = m.transition_matrix(1, b, 1.3)
            assert np.all(p >= 0)
            np.testing.assert_allclose(p.sum(1), 1.0, atol=1e-10)


def test_expm_vs_taylor():  # test_substitution.cpp:91-115
    assert np.array_equal(O.expm(np.zeros((3, 3))), np.eye(3))
    d = np.array([-0.2, 0.0, 1.4, -3.0])
    np.testing.assert_allclose(np.diag(O.expm(np.diag(d))), np.exp(d), rtol=1e-14)
    rng = O.Rng(9)
    for _ in range(20):
        q = np.array([[0.0 if i == j else rng.uniform(0.0, 1.0) for j in range(4)] for i in range(4)])
        np.fill_diagonal(q, -q.sum(1))
        a = q * 0.3
        ref = taylor_expm(a)
        assert np.linalg.norm(O.expm(a) - ref) <= 1e-12 * np.linalg.norm(ref)
    with pytest.raises(O.OracleInvalidArgument):
        O.expm(np.array([[0.0, np.inf], [0.0, 0.0]]))


def test_derivative_and_composition():  # test_substitution.cpp:117-142
    m = O.Model.hky85(2.5, [0.35, 0.15, 0.2, 0.3])
    b, h = 0.4, 1e-5
    fd = (m.transition_matrix(1, b + h) - m.transition_matrix(1, b - h)) / (2 * h)
    p = m.transition_matrix(1, b)
    assert np.abs(fd - m.q @ p).max() < 1e-6 and np.abs(fd - p @ m.q).max() < 1e-6
    g = O.Model.gtr([1.1, 2.4, 0.8, 1.7, 3.2, 1.0], [0.4, 0.1, 0.25, 0.25])
    ck = g.transition_matrix(1, 0.3) @ g.transition_matrix(1, 0.4)
    assert np.abs(g.transition_matrix(1, 0.7) - ck).max() < 1e-10
    k = O.Model.hky85(3.0, [0.1, 0.45, 0.25, 0.2])
    flow = np.diag(k.pi) @ k.transition_matrix(1, 0.6)
    assert np.abs(flow - flow.T).max() < 1e-10


def test_raw_branch_generator_verbatim():  # test_substitution.cpp:144-158
    m = O.Model.jc69()
    q = np.array([[-3, 1, 1, 1], [2, -4, 1, 1], [1, 1, -2, 0], [3, 1, 2, -6]], float)
    m.set_branch_generator(2, q)
    p = m.transition_matrix(2, 0.2)
    assert np.abs(p - taylor_expm(q * 0.2)).max() < 1e-12
    np.testing.assert_allclose(p.sum(1), 1.0, atol=1e-10)
    bad = q.copy()
    bad[0, 1] = -1
    with pytest.raises(O.OracleInvalidArgument):
        m.set_branch_generator(3, bad)


def test_discrete_gamma():  # test_substitution.cpp:160-184
    r, p = O.discrete_gamma(0.7, 1)
    assert r[0] == 1.0 and p[0] == 1.0
    r, _ = O.discrete_gamma(1e6, 4)
    assert np.all(np.abs(r - 1) < 1.2e-3)
    r, _ = O.discrete_gamma(1e8, 4)
    assert np.all(np.abs(r - 1) < 1.2e-4)
    r, p = O.discrete_gamma(0.5, 4)
    assert abs(p.sum() - 1) < 1e-14 and abs(r @ p - 1) < 1e-12
    orc = np.array([O.gamma_quantile(0.5, 0.5, (2 * l + 1) / 8) for l in range(4)])
    orc *= 4 / orc.sum()
    np.testing.assert_allclose(r, orc, rtol=1e-9)
    with pytest.raises(O.OracleInvalidArgument):
        O.discrete_gamma(0.0, 4)
    with pytest.raises(O.OracleInvalidArgument):
        O.discrete_gamma(0.5, 0)


def test_model_rejects_invalid():  # test_substitution.cpp:186-197
    with pytest.raises(O.OracleInvalidArgument):
        O.Model.hky85(-1.0, [0.25] * 4)
    with pytest.raises(O.OracleInvalidArgument):
        O.Model.hky85(2.0, [0.5, 0.5, 0.2, -0.2])
    with pytest.raises(O.OracleInvalidArgument):
        O.Model.gtr([-1.0] * 6, [0.25] * 4)
    with pytest.raises(O.OracleInvalidArgument):
        O.Model(np.ones((4, 4)), [0.25] * 4, False)


# ------------------------------------------------------------------- tree KATs
def test_three_taxon_numbering():  # test_tree.cpp:10-24, :59-61
    t = O.Tree.parse("((A:0.1,B:0.2):0.05,C:0.3);")
    assert t.tip_count == 3 and t.root == 5
    assert t.labels[1:4] == ["A", "B", "C"]
    assert list(t.parent[1:5]) == [4, 4, 5, 5]
    assert t.branch_lengths[0] == 0.1 and t.branch_lengths[3] == 0.05
    assert list(t.post_order) == [1, 2, 4, 3, 5]
    t2 = O.Tree.parse("(A:0.1,B:0.2);")
    assert list(t2.post_order) == [1, 2, 3]


def test_newick_errors():  # test_tree.cpp:36-52
    for bad, frag in [("((A:0.1,B:0.2,C:0.3):0.05,D:0.4);", "polytomy"), ("((A:0.1):0.2,B:0.3);", "unifurcation"),
                      ("(A:-0.1,B:0.2);", "negative")]:
        with pytest.raises(O.OracleNewickError, match=frag):
            O.Tree.parse(bad)
    for bad in ["((A,B),(A,C));", "(A:0.1,B:0.2)", "(A:0.1,B:0.2();", "A;"]:
        with pytest.raises(O.OracleNewickError):
            O.Tree.parse(bad)
    assert O.Tree.newick_error_position("(A:0.1,B:bad);") == 9


def test_serialize_round_trip():  # test_tree.cpp:76-92
    text = "((A:0.1,B:0.2):0.05,C:0.3);"
    assert O.Tree.parse(text).serialize() == text
    assert O.Tree.parse("((A:0.1,B:0.2)inner:0.05,C:0.3)root;").serialize() == text


def test_times_from_durations():  # test_tree.cpp:124-132
    t = O.Tree.parse("((A:0.1,B:0.2):0.05,C:0.3);")
    times = t.assign_times()
    assert times[5] == 0.0 and times[4] == pytest.approx(0.05) and times[1] == pytest.approx(0.15)


# --------------------------------------------------------------- alignment KATs
def test_iupac_and_gaps():  # test_alignment.cpp:38-50
    aln = O.Alignment.from_fasta(">A\nR-N\n>B\nAAA\n")
    a = aln.taxon_index("A")
    tp = aln.tip_partials(a)
    assert list(tp[:, 0]) == [1, 0, 1, 0]
    assert list(tp[:, 1]) == [1, 1, 1, 1] and list(tp[:, 2]) == [1, 1, 1, 1]
    assert aln.pattern_count == 3


def test_compression_counts():  # test_alignment.cpp:52-70
    two = O.Alignment.from_fasta(">x\nAAC\n>y\nAAG\n")
    assert list(two.weights) == [2, 1] and two.pattern_column(0) == "AA"
    one = O.Alignment.from_fasta(">x\n" + "A" * 100 + "\n>y\n" + "A" * 100 + "\n")
    assert one.pattern_count == 1 and one.weights[0] == 100
    four = O.Alignment.from_fasta(">x\nACGT\n>y\nCAGT\n")
    assert four.pattern_count == 4 and four.weights.sum() == 4


def test_generic_state_count():  # test_alignment.cpp:72-80
    aln = O.Alignment.from_codes([[0, 5, -1], [1, 5, 2]], 6, ["a", "b"])
    assert aln.state_count == 6 and aln.pattern_count == 3
    assert np.array_equal(aln.tip_partials(0)[:, 2], np.ones(6))
    assert aln.tip_partials(1)[2, 2] == 1.0
    with pytest.raises(O.OracleInvalidArgument):
        O.Alignment.from_codes([[7]], 4, ["a"])


def test_brute_force_fig1_bracketed_sum():  # test_validation.cpp:11-32
    tree = O.Tree.parse("((A:0.1,B:0.2):0.05,C:0.3);")
    model = O.Model.hky85(2.0, [0.3, 0.2, 0.25, 0.25])
    aln = O.Alignment.from_fasta(">A\nA\n>B\nC\n>C\nG\n")
    lengths = [0.1, 0.2, 0.3, 0.05]
    v = O.brute_force_log_likelihood(tree, aln, model, *SINGLE, lengths)
    p = lambda br, b: model.transition_matrix(br, b)
    total = 0.0
    for y5 in range(4):
        inner = sum(p(4, 0.05)[y5, y4] * p(1, 0.1)[y4, 0] * p(2, 0.2)[y4, 1] for y4 in range(4))
        total += model.pi[y5] * inner * p(3, 0.3)[y5, 2]
    assert abs(v - math.log(total)) < 1e-14


@pytest.mark.parametrize("name,sites", [("C4", 4000), ("C5", 2000)])
def test_oracle_p_method_spread(name, sites):
    """The fp64 uncertainty the parity bar must allow for: the reference
    computes P(t) by a symmetric eigensystem for reversible models and by
    Pade scaling-and-squaring otherwise (substitution.hpp:153-156).  Running
    the SAME reversible instance through both paths moves cancelling gradient
    components by more than 1e-9 relative, but by < 1e-10 of each component's
    condition (oracle gradient_condition) -- the condition-aware bound of
    tests/helpers.py (COND_RTOL)."""
    import dataclasses

    from tests.helpers import COND_RTOL, oracle_for
    from workloads import synth

    inst = synth.generate(name, seed=12146, sites=sites)
    a = oracle_for(inst, blocks=8)
    lla, ga, _ = a.branch_gradient(False)
    cond = a.gradient_condition()
    b = oracle_for(dataclasses.replace(inst, reversible=False), blocks=8)
    llb, gb, _ = b.branch_gradient(False)
    err = np.abs(ga - gb)
    assert abs(lla - llb) <= 1e-12 * abs(lla)
    assert np.max(err / np.abs(ga)) > 1e-9        # the plain relative bar is below the method spread
    assert np.max(err / cond) < COND_RTOL          # the condition-aware bar is above it
