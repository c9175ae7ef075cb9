"""Parity of the exact workloads bench.py times: the
BASELINE.json configs C2 (20,000 patterns, 512 taxa, 2 % gaps), C3 (906,622
patterns on the 2,048-taxon tree, the benchmarked walk4 geometry: one lane
per pattern, 4 categories), C4 (20 states, 1,000 taxa) and C5 (61-state
codons, 256 taxa) at FULL size, seed 12146, against the committed oracle
fixtures tests/golden/full_*.npz (made by tests/golden/make_fullsize.py: the
KAT-pinned CPU oracle in pattern chunks).  North star: relative error <= 1e-9
on logL and on every gradient component; components whose terms cancel are
judged against their condition (tests/helpers.py COND_RTOL, set by the
oracle's own eigen-vs-Pade spread).

Also: results are bit-reproducible whatever the free device memory (the
grid, and with it the fixed-order reduction, does not depend on it), and the
device error flags are sticky across back-to-back device evaluations."""
import os

import numpy as np
import pytest

from tests.helpers import assert_logl, assert_vec
from workloads import synth

HERE = os.path.dirname(os.path.abspath(__file__))
SEED = 12146


def _fixture(name):
    path = os.path.join(HERE, "golden", f"full_{name}.npz")
    if not os.path.exists(path):
        pytest.fail(f"missing full-size fixture {path} (tests/golden/make_fullsize.py)")
    return np.load(path)


@pytest.mark.gpu
@pytest.mark.parametrize("name,kernel,lanes", [("C2", "walk4_kernel", 2), ("C3", "walk4s_kernel", 1),
                                               ("C4", "walkm_kernel", 4), ("C5", "walkm_kernel", 4)])
def test_full_size_workload_matches_oracle(name, kernel, lanes):
    fx = _fixture(name)
    inst = synth.generate(name, seed=SEED, threads=os.cpu_count() or 1)
    assert inst.patterns == int(fx["patterns"])
    assert synth.instance_digest(inst) == str(fx["digest"]), "bench instance differs from the fixture's"
    eng = synth.engine_for(inst)
    rep = eng.rate_gradient() if inst.clock else eng.branch_gradient()
    info = eng.info()
    assert info["kernel"] == kernel and info["lanes_per_pattern"] == lanes, info
    want = fx["rate_gradient"] if inst.clock else fx["gradient"]
    ckey = "rate_gradient_condition" if inst.clock else "gradient_condition"
    cond = fx[ckey] if ckey in fx.files else None
    assert_logl(rep.log_likelihood, float(fx["logL"]))
    # 1e-9 relative per component; a component whose 10^5..10^6 per-pattern
    # terms cancel is judged against its condition sum_s w_s |term_s|
    assert_vec(rep.branch_gradient, want, what=f"{name} full-size gradient", cond=cond)
    if inst.clock:
        # the plain branch-length gradient of the same evaluation route
        assert_vec(eng.branch_gradient().branch_gradient, fx["gradient"], what=f"{name} branch-length gradient",
                   cond=fx["gradient_condition"] if "gradient_condition" in fx.files else None)


@pytest.mark.gpu
def test_bit_reproducible_across_free_memory():
    import torch

    inst = synth.generate("C3", seed=4, sites=60000)
    a = synth.engine_for(inst).rate_gradient()
    free, _ = torch.cuda.mem_get_info()
    hog = torch.empty(int(free * 0.6), dtype=torch.uint8, device="cuda")
    try:
        b = synth.engine_for(inst).rate_gradient()
    finally:
        del hog
    assert a.log_likelihood == b.log_likelihood
    assert np.array_equal(a.branch_gradient, b.branch_gradient)


@pytest.mark.gpu
def test_error_flags_sticky_across_device_evaluations():
    """An underflow in an earlier back-to-back device evaluation is still
    reported at the next pg_check_errors (the bench checks after its timed
    region)."""
    import torch

    from paper_1905_12146_b200 import _lib as _L
    from paper_1905_12146_b200.api import EngineOptions

    inst = synth.generate("C2", seed=2, sites=200, tips=800)
    eng = synth.engine_for(inst, EngineOptions(disable_rescaling=True))
    L = _L.lib()
    out = torch.zeros(1 + inst.branches, dtype=torch.float64, device="cuda")
    _L.check(L.pg_set_stream(eng.handle, torch.cuda.current_stream().cuda_stream))
    # 800 tips near stationarity in every Gamma category, no rescaling: ~4^-800 underflows
    eng.set_branch_lengths(np.full(inst.branches, 300.0))
    _L.check(L.pg_evaluate_device(eng.handle, _L.EVAL_GRAD, out.data_ptr()))
    eng.set_branch_lengths(np.full(inst.branches, 1e-3))
    _L.check(L.pg_evaluate_device(eng.handle, _L.EVAL_GRAD, out.data_ptr()))
    with pytest.raises(_L.RuntimeFailure, match="underflow"):
        _L.check(L.pg_check_errors(eng.handle))
    # the next window starts clean
    _L.check(L.pg_evaluate_device(eng.handle, _L.EVAL_GRAD, out.data_ptr()))
    _L.check(L.pg_check_errors(eng.handle))
