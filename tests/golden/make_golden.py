"""Generates the committed golden fixtures (tests/golden/*.npz) from the CPU
oracle (oracle/, pinned by the reference's known-answer tests in
tests/test_oracle_kats.py).  Each fixture holds the complete input of one
evaluation — tree arrays, compressed patterns + weights, model, categories,
optional per-branch generators — and the expected outputs: logL, branch
gradient, Hessian diagonal, per-pattern site log-likelihoods.

    python tests/golden/make_golden.py        # rewrites tests/golden/*.npz
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402
from workloads import synth  # noqa: E402


def from_instance(name, inst, branch_q=()):
    tree = O.Tree.from_arrays(inst.tip_count, inst.parent, inst.children, inst.branch_lengths, inst.post_order)
    aln = O.Alignment.from_patterns(inst.codes.astype(np.int32), inst.states, inst.weights)
    model = O.Model(inst.q, inst.pi, inst.reversible)
    for br, g in branch_q:
        model.set_branch_generator(br, g)
    eng = O.Engine(tree, aln, model, inst.cat_rates, inst.cat_probs, blocks=8)
    ll, g, h = eng.branch_gradient(True)
    bq_idx = np.array([b for b, _ in branch_q], np.int32)
    bq = np.array([q for _, q in branch_q], np.float64).reshape(len(branch_q), inst.states, inst.states)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), tip_count=inst.tip_count, parent=inst.parent,
                        children=inst.children, post_order=inst.post_order, branch_lengths=inst.branch_lengths,
                        codes=inst.codes.astype(np.int8), weights=inst.weights, states=inst.states, q=inst.q,
                        pi=inst.pi, reversible=inst.reversible, cat_rates=inst.cat_rates, cat_probs=inst.cat_probs,
                        branch_q_index=bq_idx, branch_q=bq, logL=ll, gradient=g, hessian=h)
    print(f"{name}: {inst.tip_count} tips, {inst.patterns} patterns, m={inst.states}, L={len(inst.cat_rates)}, "
          f"logL {ll:.12f}")


def main():
    # BASELINE.json configs at oracle-friendly sizes (C1 at its full size)
    from_instance("c1_full", synth.generate("C1"))
    from_instance("c2_gaps", synth.generate("C2", sites=600, tips=48))
    from_instance("c3_nonrev_clock", synth.generate("C3", sites=500, tips=40))
    from_instance("c4_aa20", synth.generate("C4", sites=200, tips=40))
    from_instance("c5_codon", synth.generate("C5", sites=80, tips=24))
    # per-branch (non-homogeneous) generators on the 20-state config
    inst = synth.generate("C4", seed=77, sites=150, tips=20)
    rng = np.random.default_rng(77)
    bq = []
    for br in (1, 5, 17, 30):
        g = rng.lognormal(0, 0.5, (20, 20))
        np.fill_diagonal(g, 0)
        np.fill_diagonal(g, -g.sum(1))
        bq.append((br, g))
    from_instance("c4_branch_generators", inst, bq)


if __name__ == "__main__":
    main()
