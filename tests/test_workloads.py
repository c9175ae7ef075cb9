"""The synthetic workload generator (workloads/, input generation only):
C1/C2 are simulated in the reference's draw order (alignment.hpp:243-286), so
the oracle's restated simulate_states regenerates their columns; the library
is separate from the product library."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from workloads import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _oracle_sim(inst, sites, seed):
    tree = O.Tree.from_arrays(inst.tip_count, inst.parent, inst.children, inst.branch_lengths, inst.post_order)
    model = O.Model(inst.q, inst.pi, inst.reversible)
    return O.simulate_states(tree, model, inst.cat_rates, inst.cat_probs, inst.branch_lengths, sites, seed)


@pytest.mark.parametrize("name,sites", [("C1", 1000), ("C2", 3000)])
def test_reference_draw_order_matches_oracle(name, sites):
    inst = synth.generate(name, seed=12146, sites=sites)
    got = synth.simulate_states(inst.tip_count, inst.parent, inst.post_order, inst.q, inst.pi, inst.reversible,
                                inst.cat_rates, inst.cat_probs, inst.branch_lengths, sites, 12146)
    want = _oracle_sim(inst, sites, 12146)
    assert np.array_equal(got.astype(np.int32), want)


def test_reference_configs_regenerate_from_simulate_states():
    # C1 (no gaps): compressing the oracle's simulate_states output with the
    # oracle's from_codes gives exactly the generated patterns and weights
    inst = synth.generate("C1", seed=12146)
    cols = _oracle_sim(inst, 1000, 12146)
    aln = O.Alignment.from_codes(cols, inst.states)
    assert np.array_equal(aln.pattern_codes(), inst.codes.astype(np.int32))
    assert np.array_equal(aln.weights, inst.weights)


def test_blocked_simulation_independent_of_threads():
    a = synth.generate("C4", seed=5, sites=9000, tips=12, threads=1)
    b = synth.generate("C4", seed=5, sites=9000, tips=12, threads=5)
    assert np.array_equal(a.codes, b.codes) and np.array_equal(a.weights, b.weights)
    assert a.weights.sum() == 9000


def test_simulate_rejects_bad_input():
    inst = synth.generate("C1", seed=1, sites=50)
    with pytest.raises(ValueError, match="site_count"):
        synth.simulate_states(inst.tip_count, inst.parent, inst.post_order, inst.q, inst.pi, True, inst.cat_rates,
                              inst.cat_probs, inst.branch_lengths, 0, 1)
    bad = inst.branch_lengths.copy()
    bad[3] = -1.0
    with pytest.raises(ValueError, match="negative branch length"):
        synth.simulate_states(inst.tip_count, inst.parent, inst.post_order, inst.q, inst.pi, True, inst.cat_rates,
                              inst.cat_probs, bad, 10, 1)


def test_generator_does_not_map_the_product_library():
    # the CPU reference arm builds its inputs here; it must not load
    # libphylograd_b200.so (checked in a fresh interpreter)
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from workloads import synth\n"
            "synth.generate('C2', sites=500)\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert 'libpg_workloads.so' in maps\n"
            "assert 'libphylograd_b200' not in maps, 'product library mapped'\n") % ROOT
    subprocess.check_call([sys.executable, "-c", code])


def test_counter_simulation_independent_of_threads_and_compressed_consistently():
    """C3-C5 use the counter-based per-site stream (pg_simulate.hpp): the
    columns do not depend on the thread count, and the instance's patterns are
    the first-occurrence compression of exactly those columns."""
    inst = synth.generate("C3", seed=21, sites=3000, tips=40, threads=1)
    cols1 = synth.simulate_states_counter(inst.tip_count, inst.parent, inst.post_order, inst.q, inst.pi,
                                          inst.reversible, inst.cat_rates, inst.cat_probs, inst.branch_lengths, 3000,
                                          21, threads=1)
    cols7 = synth.simulate_states_counter(inst.tip_count, inst.parent, inst.post_order, inst.q, inst.pi,
                                          inst.reversible, inst.cat_rates, inst.cat_probs, inst.branch_lengths, 3000,
                                          21, threads=7)
    assert np.array_equal(cols1, cols7)
    aln = O.Alignment.from_codes(cols1.astype(np.int32), inst.states)
    assert np.array_equal(aln.pattern_codes(), inst.codes.astype(np.int32))
    assert np.array_equal(aln.weights, inst.weights)
    assert synth.CONFIGS["C3"]["sim"] == synth.SIM_COUNTER


def test_counter_simulation_gaps_and_states():
    inst = synth.generate("C4", seed=3, sites=100, tips=12)
    cols = synth.simulate_states_counter(inst.tip_count, inst.parent, inst.post_order, inst.q, inst.pi, True,
                                         inst.cat_rates, inst.cat_probs, inst.branch_lengths, 20000, 9, gap=0.05)
    assert cols.min() == -1 and cols.max() <= 19
    assert 0.04 < (cols < 0).mean() < 0.06
    with pytest.raises(ValueError, match="gap fraction"):
        synth.simulate_states_counter(inst.tip_count, inst.parent, inst.post_order, inst.q, inst.pi, True,
                                      inst.cat_rates, inst.cat_probs, inst.branch_lengths, 10, 9, gap=1.5)
