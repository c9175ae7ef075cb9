"""Committed golden fixtures (tests/golden/*.npz, made by
tests/golden/make_golden.py from the KAT-pinned oracle): the oracle must keep
reproducing them (CPU), and the sm_100a engine must match them within the
north star's 1e-9 (GPU)."""
import glob
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import assert_logl, assert_vec

# complete small evaluations (inputs + outputs); the full-size fixtures
# (full_*.npz: digest + outputs only) are checked by tests/test_gpu_fullsize.py
FIXTURES = sorted(f for f in glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "*.npz"))
                  if not os.path.basename(f).startswith("full_"))
IDS = [os.path.basename(f)[:-4] for f in FIXTURES]


def _load(path):
    z = np.load(path)
    return {k: z[k] for k in z.files}


def _oracle(fx):
    tree = O.Tree.from_arrays(int(fx["tip_count"]), fx["parent"], fx["children"], fx["branch_lengths"],
                              fx["post_order"])
    aln = O.Alignment.from_patterns(fx["codes"].astype(np.int32), int(fx["states"]), fx["weights"])
    model = O.Model(fx["q"], fx["pi"], bool(fx["reversible"]))
    for br, g in zip(fx["branch_q_index"], fx["branch_q"]):
        model.set_branch_generator(int(br), g)
    eng = O.Engine(tree, aln, model, fx["cat_rates"], fx["cat_probs"], blocks=8)
    eng._keep = (tree, aln, model)
    return eng


def test_fixtures_present():
    assert len(FIXTURES) >= 6


@pytest.mark.parametrize("path", FIXTURES, ids=IDS)
def test_oracle_reproduces_golden(path):
    fx = _load(path)
    ll, g, h = _oracle(fx).branch_gradient(True)
    assert ll == pytest.approx(float(fx["logL"]), rel=1e-13)
    np.testing.assert_allclose(g, fx["gradient"], rtol=1e-11, atol=1e-13 * np.abs(fx["gradient"]).max())
    np.testing.assert_allclose(h, fx["hessian"], rtol=1e-10, atol=1e-12 * np.abs(fx["hessian"]).max())


@pytest.mark.gpu
@pytest.mark.parametrize("path", FIXTURES, ids=IDS)
def test_engine_matches_golden(path):
    from paper_1905_12146_b200.api import (EngineOptions, LikelihoodEngine, RateCategories, SitePatternAlignment,
                                           SubstitutionModel, Tree)

    fx = _load(path)
    n = int(fx["tip_count"])
    labels = [""] + [f"t{i}" for i in range(1, n + 1)] + [""] * (n - 1)
    tree = Tree(n, fx["parent"], fx["children"], np.concatenate([[0.0], fx["branch_lengths"], [0.0]]), labels,
                fx["post_order"])
    aln = SitePatternAlignment(labels[1:n + 1], int(fx["states"]), fx["codes"], fx["weights"])
    model = SubstitutionModel(fx["q"], fx["pi"], bool(fx["reversible"]))
    for br, g in zip(fx["branch_q_index"], fx["branch_q"]):
        model.set_branch_generator(int(br), g)
    eng = LikelihoodEngine(tree, aln, model, RateCategories(fx["cat_rates"], fx["cat_probs"]), EngineOptions())
    rep = eng.branch_gradient(True)
    assert_logl(rep.log_likelihood, float(fx["logL"]))
    assert_vec(rep.branch_gradient, fx["gradient"])
    assert_vec(rep.hessian_diagonal, fx["hessian"], rtol=1e-8, what="hessian")
    assert eng.log_likelihood() == pytest.approx(float(fx["logL"]), rel=1e-9)
