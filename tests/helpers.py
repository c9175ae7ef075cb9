"""Shared test helpers: build the product engine and the CPU oracle over the
same seeded instance, and compare with the north-star tolerances."""
import numpy as np

from oracle import oracle as O

# BASELINE.json north star: relative error <= 1e-9 on logL and every gradient
# component.  Components that cancel to ~0 are judged against the vector
# scale (condition-aware variant).
RTOL = 1e-9
ATOL_REL_SCALE = 1e-12
# condition-aware bound: a component whose terms cancel is
# judged against its condition (the oracle's gradient_condition: the same
# sums over absolute values, inside Q e and over patterns).  The scale is set
# by the reference itself: switching ONLY its P(t) method (symmetric eigen vs
# Pade, both substitution.hpp:153-156) moves such components by up to ~7e-11
# of their condition (2e-8 relative on codon components;
# tests/test_oracle_kats.py::test_oracle_p_method_spread), so 1e-10 of the
# condition is the fp64 uncertainty of the quantity, not an error.
COND_RTOL = 1e-10


def oracle_for(inst, blocks=1, **opts):
    tree = O.Tree.from_arrays(inst.tip_count, inst.parent, inst.children, inst.branch_lengths, inst.post_order)
    aln = O.Alignment.from_patterns(inst.codes.astype(np.int32), inst.states, inst.weights)
    model = O.Model(inst.q, inst.pi, inst.reversible)
    eng = O.Engine(tree, aln, model, inst.cat_rates, inst.cat_probs, blocks=blocks, **opts)
    eng._keep = (tree, aln, model)
    return eng


def assert_logl(a, b, rtol=RTOL):
    assert np.isfinite(a), f"logL {a!r} is not finite"
    assert abs(a - b) <= rtol * max(abs(b), 1e-300), f"logL {a!r} vs oracle {b!r} (rel {abs(a - b) / abs(b):.3e})"


def assert_vec(a, b, rtol=RTOL, what="gradient", cond=None):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape
    assert np.all(np.isfinite(a)), f"{what}: {int(np.sum(~np.isfinite(a)))} non-finite components"
    assert np.all(np.isfinite(b)), f"{what} (oracle): non-finite components"
    scale = np.max(np.abs(b)) if b.size else 0.0
    err = np.abs(a - b)
    tol = rtol * np.abs(b) + ATOL_REL_SCALE * scale
    if cond is not None:
        tol = np.maximum(tol, COND_RTOL * np.asarray(cond))
    bad = np.nonzero(~(err <= tol))[0]
    assert bad.size == 0, (f"{what}: {bad.size} components off; worst idx {bad[np.argmax(err[bad])]} "
                           f"got {a[bad[0]]!r} want {b[bad[0]]!r}; max rel {np.max(err / np.maximum(np.abs(b), 1e-300)):.3e}")


def rel_report(a, b, cond=None):
    a = np.asarray(a)
    b = np.asarray(b)
    scale = np.max(np.abs(b))
    out = {"max_rel": float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))),
           "max_rel_to_scale": float(np.max(np.abs(a - b)) / scale)}
    if cond is not None:
        out["max_rel_to_condition"] = float(np.max(np.abs(a - b) / np.maximum(np.asarray(cond), 1e-300)))
    return out
