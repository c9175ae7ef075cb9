"""Direct oracle parity of every 4-state kernel variant (the C2/C3 bench
kernels): the per-warp walk4_kernel<HOMOG, HESS, NC, LCV> with one lane per
pattern (LCV=4) or two (LCV=2) forced through PG_WALK4_LCV, and the
level-scheduled walkl_kernel<L, HOMOG, HESS> (PG_WALKL=1; the small-P
default); homogeneous and per-branch generators, with and without the
Hessian, gaps only (NC=5) and IUPAC ambiguity classes (NC=16)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import assert_logl, assert_vec

pytestmark = pytest.mark.gpu

pg = pytest.importorskip("paper_1905_12146_b200")
from workloads import synth  # noqa: E402
from paper_1905_12146_b200.api import (EngineOptions, LikelihoodEngine, RateCategories,  # noqa: E402
                                       SitePatternAlignment, SubstitutionModel, Tree, parse_fasta, parse_newick)


@pytest.fixture(params=["lvl", "4t", "4s", 4, 2], ids=["walkl", "lcv4t", "lcv4s", "lcv4", "lcv2"])
def lcv(request, monkeypatch):
    """The kernel variant under test; returns (kernel name, lanes per pattern)."""
    if request.param == "lvl":
        monkeypatch.setenv("PG_WALKL", "1")
        return "walkl_kernel", 4
    monkeypatch.setenv("PG_WALKL", "0")
    if request.param == "4t":
        # tensor-core (DMMA) walk: lane = (pattern, state)
        monkeypatch.setenv("PG_WALK4_LCV", "4")
        monkeypatch.setenv("PG_WALK4T", "1")
        return "walk4t_kernel", 1
    monkeypatch.setenv("PG_WALK4T", "0")
    if request.param == "4s":
        # single-buffered one-lane-per-pattern walk (chosen by padded wave
        # work at large P; forced here)
        monkeypatch.setenv("PG_WALK4_LCV", "4")
        monkeypatch.setenv("PG_WALK4S", "1")
        return "walk4s_kernel", 1
    monkeypatch.setenv("PG_WALK4S", "0")
    monkeypatch.setenv("PG_WALK4_LCV", str(request.param))
    return "walk4_kernel", 4 // request.param


def _branch_q(seed, B, k=5):
    rng = np.random.default_rng(seed)
    out = []
    for br in rng.choice(np.arange(1, B + 1), size=k, replace=False):
        q = rng.lognormal(0, 0.6, (4, 4))
        np.fill_diagonal(q, 0)
        np.fill_diagonal(q, -q.sum(1))
        out.append((int(br), q))
    return out


def _instance_pair(inst, branch_q=()):
    labels = inst.labels()
    tree = Tree(inst.tip_count, inst.parent, inst.children, np.concatenate([[0.0], inst.branch_lengths, [0.0]]),
                labels, inst.post_order)
    aln = SitePatternAlignment(labels[1:inst.tip_count + 1], inst.states, inst.codes, inst.weights)
    model = SubstitutionModel(inst.q, inst.pi, inst.reversible)
    for br, q in branch_q:
        model.set_branch_generator(br, q)
    eng = LikelihoodEngine(tree, aln, model, RateCategories(inst.cat_rates, inst.cat_probs), EngineOptions())
    tree_o = O.Tree.from_arrays(inst.tip_count, inst.parent, inst.children, inst.branch_lengths, inst.post_order)
    aln_o = O.Alignment.from_patterns(inst.codes.astype(np.int32), inst.states, inst.weights)
    model_o = O.Model(inst.q, inst.pi, inst.reversible)
    for br, q in branch_q:
        model_o.set_branch_generator(br, q)
    ref = O.Engine(tree_o, aln_o, model_o, inst.cat_rates, inst.cat_probs, blocks=16)
    ref._keep = (tree_o, aln_o, model_o)
    return eng, ref


@pytest.mark.parametrize("homog", [True, False], ids=["homog", "per_branch_q"])
@pytest.mark.parametrize("hess", [False, True], ids=["grad", "hess"])
def test_walk4_variants_c3_shape(lcv, homog, hess):
    # C3 model family (raw non-reversible Q, Pade P(t)) on a 256-taxon Yule tree
    inst = synth.generate("C3", sites=40000, tips=256)
    bq = () if homog else _branch_q(3, inst.branches)
    eng, ref = _instance_pair(inst, bq)
    ll, g, h = ref.branch_gradient(hess)
    rep = eng.branch_gradient(hess)
    assert eng.info()["kernel"] == lcv[0]
    assert eng.info()["lanes_per_pattern"] == lcv[1]
    assert_logl(rep.log_likelihood, ll)
    assert_vec(rep.branch_gradient, g)
    if hess:
        assert_vec(rep.hessian_diagonal, h, rtol=1e-8, what="hessian")


def test_walk4_gaps_c2_shape(lcv):
    inst = synth.generate("C2", sites=12000)  # GTR + 2 % gaps
    eng, ref = _instance_pair(inst)
    ll, g, _ = ref.branch_gradient(False)
    rep = eng.branch_gradient()
    assert eng.info()["kernel"] == lcv[0]
    assert_logl(rep.log_likelihood, ll)
    assert_vec(rep.branch_gradient, g)


def test_walk4_iupac_classes(lcv):
    """IUPAC ambiguity classes (alignment.hpp:50-70) widen the TC table to
    NC = 16 columns."""
    rng = np.random.default_rng(8)
    taxa, sites = 24, 9000
    alphabet = np.array(list("ACGT"))
    amb = np.array(list("RYKMSWBDHVN-?"))
    cols = alphabet[rng.integers(0, 4, size=(taxa, sites))]
    mask = rng.random((taxa, sites)) < 0.08
    cols = np.where(mask, amb[rng.integers(0, amb.size, size=(taxa, sites))], cols)
    tree_o = O.Tree.random(O.Rng(4), taxa, 0.02, 0.3)
    names = [tree_o.labels[k] for k in range(1, taxa + 1)]
    fasta = "".join(f">{names[i]}\n{''.join(cols[i])}\n" for i in range(taxa))
    newick = tree_o.serialize()
    model = SubstitutionModel.hky85(2.0, [0.3, 0.2, 0.2, 0.3])
    cats = pg.discrete_gamma_categories(0.5, 4)
    tree = parse_newick(newick)
    aln = SitePatternAlignment.compress(parse_fasta(fasta))
    eng = LikelihoodEngine(tree, aln, model, cats, EngineOptions())
    ref = O.Engine(O.Tree.parse(newick), O.Alignment.from_fasta(fasta), O.Model.hky85(2.0, [0.3, 0.2, 0.2, 0.3]),
                   list(cats.rates), list(cats.probs), blocks=8)
    ll, g, h = ref.branch_gradient(True)
    rep = eng.branch_gradient(True)
    assert eng.info()["kernel"] == lcv[0]
    assert_logl(rep.log_likelihood, ll)
    assert_vec(rep.branch_gradient, g)
    assert_vec(rep.hessian_diagonal, h, rtol=1e-8, what="hessian")


def _gtr(rng):
    pi = rng.dirichlet(np.ones(4) * 5)
    s = rng.lognormal(0, 0.5, (4, 4))
    s = (s + s.T) / 2
    q = s * pi[None, :]
    np.fill_diagonal(q, 0)
    np.fill_diagonal(q, -q.sum(1))
    q /= -np.sum(pi * np.diag(q))
    return q, pi


@pytest.mark.parametrize("L", [1, 2, 3, 8])
@pytest.mark.parametrize("homog", [True, False], ids=["homog", "per_branch_q"])
@pytest.mark.parametrize("level", [False, True], ids=["walk4", "walkl"])
def test_walk4_other_category_counts(L, homog, level, monkeypatch):
    """The pipelined kernel for 1, 2, 3 rate categories (one lane per pattern)
    and 8 (two lanes per pattern), and the level-scheduled one for 1, 2, 8
    (L = 3 has no level-scheduled instance: walk4 runs), with gaps,
    per-branch generators and the Hessian."""
    monkeypatch.setenv("PG_WALKL", "1" if level else "0")
    want_kernel = "walkl_kernel" if level and L != 3 else "walk4_kernel"
    rng = np.random.default_rng(60 + L)
    q, pi = _gtr(rng)
    mo = O.Model(q, pi, True)
    taxa = 40
    tree_o = O.Tree.random(O.Rng(70 + L), taxa, 0.01, 0.2)
    bq = [] if homog else _branch_q(9, 2 * taxa - 2, k=4)
    for br, g in bq:
        mo.set_branch_generator(br, g)
    rates, probs = ([1.0], [1.0]) if L == 1 else O.discrete_gamma(0.6, L)
    codes = O.simulate_states(tree_o, mo, rates, probs, tree_o.branch_lengths, 9000, 80 + L)
    codes = np.where(rng.random(codes.shape) < 0.04, -1, codes)
    labels = [tree_o.labels[i] for i in range(1, tree_o.tip_count + 1)]
    ref = O.Engine(tree_o, O.Alignment.from_codes(codes, 4, labels), mo, rates, probs, blocks=16)
    tree = Tree(tree_o.tip_count, tree_o.parent, tree_o.children,
                np.concatenate([[0.0], tree_o.branch_lengths, [0.0]]), tree_o.labels, tree_o.post_order)
    model = SubstitutionModel(q, pi, True)
    for br, g in bq:
        model.set_branch_generator(br, g)
    eng = LikelihoodEngine(tree, SitePatternAlignment.from_codes(labels, codes, 4), model,
                           RateCategories(np.asarray(rates), np.asarray(probs)), EngineOptions())
    for hess in (False, True):
        ll, g, h = ref.branch_gradient(hess)
        rep = eng.branch_gradient(hess)
        assert eng.info()["kernel"] == want_kernel
        assert_logl(rep.log_likelihood, ll)
        assert_vec(rep.branch_gradient, g)
        if hess:
            assert_vec(rep.hessian_diagonal, h, rtol=1e-8, what="hessian")


@pytest.mark.parametrize("sites", [2500, 600])
def test_walkl_small_pattern_counts(sites, monkeypatch):
    """The small-P regime the level-scheduled traversal is for (C2 sliced to
    one GPU's share at 8 GPUs, and smaller), against the oracle, and
    bit-reproducible run to run."""
    monkeypatch.setenv("PG_WALKL", "1")
    inst = synth.generate("C2", sites=sites)
    eng, ref = _instance_pair(inst)
    ll, g, h = ref.branch_gradient(True)
    rep = eng.branch_gradient(True)
    assert eng.info()["kernel"] == "walkl_kernel"
    assert_logl(rep.log_likelihood, ll)
    assert_vec(rep.branch_gradient, g)
    assert_vec(rep.hessian_diagonal, h, rtol=1e-8, what="hessian")
    eng.invalidate_caches()
    rep2 = eng.branch_gradient(True)
    assert rep2.log_likelihood == rep.log_likelihood and np.array_equal(rep2.branch_gradient, rep.branch_gradient)


def test_walk4s_table_width_and_kernel_agree(monkeypatch):
    """A gapless 4-state alignment runs walk4s with 4-column TC blocks; the
    5-column blocks (PG_WALK4S_NC5=1) and walk4 (PG_WALK4S=0) give the same
    result to rounding, and all match the oracle (C3 model family, clock
    rates, Hessian)."""
    inst = synth.generate("C3", seed=21, sites=40000, tips=192)
    assert int(inst.codes.min()) >= 0  # no missing / ambiguous codes
    monkeypatch.setenv("PG_WALKL", "0")
    monkeypatch.setenv("PG_WALK4_LCV", "4")
    reps = {}
    for name, env in (("nc4", {}), ("nc5", {"PG_WALK4S_NC5": "1"}), ("walk4", {"PG_WALK4S": "0"})):
        for k in ("PG_WALK4S_NC5", "PG_WALK4S"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        eng, ref = _instance_pair(inst)
        reps[name] = eng.branch_gradient(True)
        assert eng.info()["kernel"] == ("walk4_kernel" if name == "walk4" else "walk4s_kernel")
    ll, g, h = ref.branch_gradient(True)
    for rep in reps.values():
        assert_logl(rep.log_likelihood, ll)
        assert_vec(rep.branch_gradient, g)
        assert_vec(rep.hessian_diagonal, h, rtol=1e-8, what="hessian")
    a, b = reps["nc4"], reps["nc5"]
    # the post-order pass is the same arithmetic (the cherry tables of the
    # 4-column kernel are exact); the fused cherry steps of its pre-order pass
    # share the parent's denominator, so the gradients agree to rounding
    assert a.log_likelihood == b.log_likelihood
    np.testing.assert_allclose(a.branch_gradient, b.branch_gradient, rtol=1e-12,
                               atol=1e-14 * np.abs(b.branch_gradient).max())
    np.testing.assert_allclose(reps["walk4"].branch_gradient, a.branch_gradient, rtol=1e-12,
                               atol=1e-14 * np.abs(a.branch_gradient).max())


def test_walk4_deep_caterpillar(lcv):
    """A 700-taxon caterpillar whose site likelihoods underflow double
    precision without rescaling (test_engine.cpp:341-361), through every
    4-state kernel variant: the pre-partials' exponents (consumer-side scaling
    in walk4s, per-quad normalisation in walk4t) over 700 levels."""
    from tests.test_gpu_parity_walkm import _caterpillar_pair

    eng, ref = _caterpillar_pair(4, 4, 700, 6000, 35, 0.3)
    ll, g, h = ref.branch_gradient(True)
    assert ll < -5000.0
    rep = eng.branch_gradient(True)
    assert eng.info()["kernel"] == lcv[0]
    assert_logl(rep.log_likelihood, ll)
    assert_vec(rep.branch_gradient, g)
    assert_vec(rep.hessian_diagonal, h, rtol=1e-8, what="hessian")


def _newick_pair(newick, sites, seed, hess_model_seed=3, branch_q=False):
    """Engine + oracle on a Newick tree with simulated gapless 4-state data
    (non-reversible generator, Γ4) and enough patterns for walk4s."""
    rng = np.random.default_rng(hess_model_seed)
    q = rng.uniform(0.2, 1.5, (4, 4))
    np.fill_diagonal(q, 0.0)
    np.fill_diagonal(q, -q.sum(1))
    pi = np.array([0.3, 0.2, 0.2, 0.3])
    tree_o = O.Tree.parse(newick)
    mo = O.Model(q, pi, False)
    rates, probs = O.discrete_gamma(0.5, 4)
    codes = O.simulate_states(tree_o, mo, rates, probs, tree_o.branch_lengths, sites, seed)
    labels = [tree_o.labels[i] for i in range(1, tree_o.tip_count + 1)]
    model = SubstitutionModel(q, pi, False)
    if branch_q:
        for br, qb in _branch_q(7, len(tree_o.branch_lengths), k=3):
            mo.set_branch_generator(br, qb)
            model.set_branch_generator(br, qb)
    ref = O.Engine(tree_o, O.Alignment.from_codes(codes, 4, labels), mo, rates, probs)
    ref._keep = (tree_o, mo)
    tree = Tree(tree_o.tip_count, tree_o.parent, tree_o.children,
                np.concatenate([[0.0], tree_o.branch_lengths, [0.0]]), tree_o.labels, tree_o.post_order)
    eng = LikelihoodEngine(tree, SitePatternAlignment.from_codes(labels, codes, 4), model,
                           RateCategories(np.asarray(rates), np.asarray(probs)), EngineOptions())
    return eng, ref


def _balanced(depth, rng, prefix="t"):
    if depth == 0:
        return f"{prefix}:{rng.uniform(0.02, 0.3):.6f}"
    return (f"({_balanced(depth - 1, rng, prefix + 'a')},{_balanced(depth - 1, rng, prefix + 'b')})"
            f":{rng.uniform(0.02, 0.3):.6f}")


def _caterpillar_newick(tips, rng):
    s = f"(c0:{rng.uniform(0.02, 0.3):.6f},c1:{rng.uniform(0.02, 0.3):.6f})"
    for i in range(2, tips):
        s = f"({s}:{rng.uniform(0.02, 0.3):.6f},c{i}:{rng.uniform(0.02, 0.3):.6f})"
    return s + ";"


@pytest.mark.parametrize("shape", ["balanced", "caterpillar", "root_cherry", "mixed"])
@pytest.mark.parametrize("branch_q", [False, True], ids=["homog", "per_branch_q"])
def test_walk4s_cherry_tables(shape, branch_q, monkeypatch):
    """walk4s with cherry tables (a node with two tip children tabulated per
    code pair, its pre-order step fused into its parent's; pg_walk4s.cuh CH
    instances) against the oracle and against the same kernel without them,
    gradient only and with the Hessian: a balanced tree (every tip in a
    cherry, parents of two cherries), a caterpillar (one cherry at the
    bottom), a small tree with a cherry directly under the root and a random
    Yule tree."""
    rng = np.random.default_rng(11)
    if shape == "balanced":
        nw = _balanced(6, rng)
        nw = nw[:nw.rfind(":")] + ";"
    elif shape == "caterpillar":
        nw = _caterpillar_newick(40, rng)
    elif shape == "root_cherry":
        nw = ("((x:0.11,y:0.07):0.05,((((a:0.2,b:0.1):0.07,c:0.3):0.04,(d:0.12,(e:0.08,f:0.25):0.1):0.06):0.09,"
              "(g:0.3,(h:0.1,(i:0.2,j:0.15):0.05):0.1):0.2):0.13);")
    else:
        inst = synth.generate("C3", seed=5, sites=30000, tips=100)
        nw = None
    monkeypatch.setenv("PG_WALKL", "0")
    monkeypatch.setenv("PG_WALK4_LCV", "4")
    monkeypatch.setenv("PG_WALK4S", "1")
    reps, grads = {}, {}
    for ch in ("1", "0"):
        monkeypatch.setenv("PG_WALK4S_CHERRY", ch)
        if nw is None:
            eng, ref = _instance_pair(inst, _branch_q(3, inst.branches) if branch_q else ())
        else:
            eng, ref = _newick_pair(nw, 30000, 17, branch_q=branch_q)
        # gradient only (cherry steps fused through the W tables) and with the
        # Hessian (fused through the tips' TC blocks, or unfused per-branch)
        grads[ch] = eng.branch_gradient(False)
        # K1 + cherry tables + walk + reduce with the tables, K1 + walk + reduce without
        assert eng.info()["launches"] == (4 if ch == "1" else 3)
        reps[ch] = eng.branch_gradient(True)
        assert eng.info()["kernel"] == "walk4s_kernel"
    ll, g, h = ref.branch_gradient(True)
    for rep in reps.values():
        assert_logl(rep.log_likelihood, ll)
        assert_vec(rep.branch_gradient, g)
        assert_vec(rep.hessian_diagonal, h, rtol=1e-8, what="hessian")
    for rep in grads.values():
        assert_logl(rep.log_likelihood, ll)
        assert_vec(rep.branch_gradient, g)
    a, b = reps["1"], reps["0"]
    np.testing.assert_allclose(a.log_likelihood, b.log_likelihood, rtol=1e-14)
    np.testing.assert_allclose(a.branch_gradient, b.branch_gradient, rtol=1e-11,
                               atol=1e-13 * np.abs(b.branch_gradient).max())
    # the logL-only route runs the post-order pass alone
    monkeypatch.setenv("PG_WALK4S_CHERRY", "1")
    eng, ref = (_instance_pair(inst) if nw is None else _newick_pair(nw, 30000, 17))
    assert_logl(eng.log_likelihood(), ref.branch_gradient(False)[0])


@pytest.mark.parametrize("branch_q", [False, True], ids=["homog", "per_branch_q"])
def test_walk4s_cherry_tables_with_missing_data(branch_q, monkeypatch):
    """Data with missing characters (5-column TC blocks): the cherries' e_k
    tables over the 25 code pairs (the cherry keeps its own pre-order step),
    against the oracle and the table-free kernel, gradient and Hessian."""
    inst = synth.generate("C2", seed=9, sites=40000, tips=96)
    assert int(inst.codes.min()) < 0  # missing characters present
    monkeypatch.setenv("PG_WALKL", "0")
    monkeypatch.setenv("PG_WALK4_LCV", "4")
    monkeypatch.setenv("PG_WALK4S", "1")
    reps = {}
    for ch in ("1", "0"):
        monkeypatch.setenv("PG_WALK4S_CHERRY", ch)
        eng, ref = _instance_pair(inst, _branch_q(3, inst.branches) if branch_q else ())
        g_only = eng.branch_gradient(False)
        assert eng.info()["kernel"] == "walk4s_kernel"
        assert eng.info()["launches"] == (4 if ch == "1" else 3)
        reps[ch] = (g_only, eng.branch_gradient(True))
    ll, g, h = ref.branch_gradient(True)
    for g_only, rep in reps.values():
        assert_logl(rep.log_likelihood, ll)
        assert_vec(g_only.branch_gradient, g)
        assert_vec(rep.branch_gradient, g)
        assert_vec(rep.hessian_diagonal, h, rtol=1e-8, what="hessian")
    # unfused cherry steps: the same arithmetic as the table-free kernel
    assert reps["1"][1].log_likelihood == reps["0"][1].log_likelihood
    assert np.array_equal(reps["1"][1].branch_gradient, reps["0"][1].branch_gradient)
