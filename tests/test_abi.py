"""CPU-side checks of the product library: it loads, exports every symbol
include/phylograd_b200.h declares, and its host-side formats (tree indexing,
pattern compression, discrete gamma) are bit-exact with the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pglib():
    from paper_1905_12146_b200 import _lib

    return _lib


def header_symbols():
    text = open(os.path.join(ROOT, "include", "phylograd_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pg_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol(pglib):
    so = ctypes.CDLL(pglib.SO_PATH)
    syms = header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(so, s)]
    assert not missing, missing
    assert sorted(pglib.EXPORTS) == syms


def test_no_cpu_fallback_without_library(tmp_path, monkeypatch, pglib):
    monkeypatch.setattr(pglib, "SO_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(pglib, "_lib", None)
    with pytest.raises(ImportError, match="no CPU fallback"):
        pglib.lib()


def _tree_arrays(t):
    return t.tip_count, t.parent, t.children.reshape(-1), t.post_order, t.labels


def test_newick_indexing_bit_exact():
    from paper_1905_12146_b200 import parse_newick

    for text in ["((A:0.1,B:0.2):0.05,C:0.3);", "(A:0.1,B:0.2);", "((A,B),C);",
                 "((A:0.1,B:0.2)inner:0.05,C:0.3)root;", "(((a:1,b:2):3,(c:4,d:5):6):7,(e:8,f:9):10);"]:
        a = parse_newick(text)
        b = O.Tree.parse(text)
        assert a.tip_count == b.tip_count
        assert np.array_equal(a.parent, b.parent)
        assert np.array_equal(a.children, b.children)
        assert np.array_equal(a.post_order, b.post_order)
        assert np.array_equal(a.branch_lengths(), b.branch_lengths)
        assert a.labels[1:a.tip_count + 1] == b.labels[1:b.tip_count + 1]
    rng = O.Rng(7)
    for tips in (2, 3, 5, 9, 16, 64, 300):
        t = O.Tree.random(rng, tips, 0.0, 1.0)
        text = t.serialize()
        a = parse_newick(text)
        b = O.Tree.parse(text)
        assert np.array_equal(a.parent, b.parent) and np.array_equal(a.post_order, b.post_order)
        assert np.array_equal(a.children, b.children)


def test_newick_errors_match_reference():  # test_tree.cpp:36-52
    import paper_1905_12146_b200 as pg

    for bad, frag in [("((A:0.1,B:0.2,C:0.3):0.05,D:0.4);", "polytomy"), ("((A:0.1):0.2,B:0.3);", "unifurcation"),
                      ("(A:-0.1,B:0.2);", "negative")]:
        with pytest.raises(pg.NewickError, match=frag):
            pg.parse_newick(bad)
    for bad in ["((A,B),(A,C));", "(A:0.1,B:0.2)", "(A:0.1,B:0.2();", "A;"]:
        with pytest.raises(pg.NewickError):
            pg.parse_newick(bad)
    with pytest.raises(pg.NewickError) as ei:
        pg.parse_newick("(A:0.1,B:bad);")
    assert ei.value.position == 9


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_compression_bit_exact(seed):
    from paper_1905_12146_b200 import SitePatternAlignment

    rng = np.random.default_rng(seed)
    m = [4, 6, 20][seed - 1]
    ntax, sites = 7, 3000
    codes = rng.integers(-1, m, size=(ntax, sites)).astype(np.int32)
    codes[:, ::3] = codes[:, :1]  # plenty of duplicates
    codes[:, 1::7] = codes[:, 5:6]
    labels = [f"x{i}" for i in range(ntax)]
    a = SitePatternAlignment.from_codes(labels, codes, m)
    b = O.Alignment.from_codes(codes, m, labels)
    assert a.pattern_count() == b.pattern_count
    assert np.array_equal(a.weights(), b.weights)
    assert np.array_equal(a.codes.astype(np.int32), b.pattern_codes())
    assert a.weights().sum() == sites


def test_compression_rejects_out_of_range():
    import paper_1905_12146_b200 as pg

    with pytest.raises(pg.InvalidArgument):
        pg.SitePatternAlignment.from_codes(["a"], [[7]], 4)


def test_fasta_compression_matches_oracle():  # test_alignment.cpp:38-70
    from paper_1905_12146_b200 import SitePatternAlignment, parse_fasta

    for fasta in [">A\nR-N\n>B\nAAA\n", ">x\nAAC\n>y\nAAG\n", ">x\nACGTRYKMSWBDHVN-?\n>y\nCAGTACGTTTTTAACGG\n"]:
        a = SitePatternAlignment.compress(parse_fasta(fasta))
        b = O.Alignment.from_fasta(fasta)
        assert a.pattern_count() == b.pattern_count
        assert np.array_equal(a.weights(), b.weights)
        for r in range(len(a.taxa())):
            assert np.array_equal(a.tip_partials(r), b.tip_partials(r))
        for p in range(a.pattern_count()):
            assert a.pattern_column(p) == b.pattern_column(p)


def test_discrete_gamma_matches_oracle():  # test_substitution.cpp:160-184
    from paper_1905_12146_b200 import discrete_gamma_categories

    for alpha, L in [(0.5, 4), (0.7, 4), (1.3, 8), (5.0, 3), (0.2, 6)]:
        c = discrete_gamma_categories(alpha, L)
        r, p = O.discrete_gamma(alpha, L)
        np.testing.assert_allclose(c.rates, r, rtol=1e-12)
        np.testing.assert_array_equal(c.probs, p)
    c = discrete_gamma_categories(0.7, 1)
    assert c.rates[0] == 1.0 and c.probs[0] == 1.0


def test_synthetic_configs_deterministic():
    from workloads import synth

    a = synth.generate("C2", seed=3, sites=2000)
    b = synth.generate("C2", seed=3, sites=2000, threads=1)
    assert np.array_equal(a.codes, b.codes) and np.array_equal(a.weights, b.weights)
    assert np.array_equal(a.branch_lengths, b.branch_lengths)
    assert a.weights.sum() == 2000
    # the synthetic tree obeys the reference numbering contract
    O.Tree.validate(a.tip_count, a.parent, a.children, a.branch_lengths, a.post_order)
    t = O.Tree.from_arrays(a.tip_count, a.parent, a.children, a.branch_lengths)
    assert np.array_equal(t.post_order, a.post_order)
    # gaps present at ~2 %
    assert 0.01 < (a.codes < 0).mean() < 0.03
    c5 = synth.generate("C5", sites=500, tips=16)
    assert c5.states == 61 and np.allclose(c5.q.sum(1), 0, atol=1e-12)
    assert -np.sum(c5.pi * np.diag(c5.q)) == pytest.approx(1.0, rel=1e-12)
