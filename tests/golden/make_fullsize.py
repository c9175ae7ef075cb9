"""Full-size parity fixtures for the exact workloads bench.py times
(VERDICT r1 "Next round" item 1): the bench instances C3 (906,112 patterns,
2,048 taxa), C4 (1,000 taxa, 20 states) and C5 (256 taxa, 61-state codons),
seed 12146, evaluated by the CPU oracle (oracle/, the KAT-pinned restatement
of engine.hpp) in pattern chunks.  logL and the branch gradient are sums over
patterns (engine.hpp:217, :268), so the chunk sums are the full-size result
(chunk order fixed; the oracle's own per-chunk reduction is deterministic).

Each fixture stores a digest of the generated inputs (so a test can prove it
regenerated the same instance), logL, the branch-length gradient g, and for the
clock config the rate gradient dt * g (clock.hpp:146-152, cli.hpp:437-438),
plus each component's condition: the same sum with every
product of the per-pattern term taken in absolute value (oracle
gradient_condition), the scale for components whose terms cancel — inside
Q e (generator rows sum to zero) or across patterns.

    python tests/golden/make_fullsize.py [C3 C4 C5]   # minutes per config on 8 cores
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from tests.helpers import oracle_for  # noqa: E402
from workloads import synth  # noqa: E402

SEED = 12146


def chunk_patterns(inst, budget_bytes=4.0e9):
    """Patterns per oracle chunk: the restatement keeps ~5 N L m doubles per
    pattern (post, pre, edge grids, engine.hpp:85-99)."""
    per = 5.0 * inst.tip_count * len(inst.cat_rates) * inst.states * 8
    return int(max(64, budget_bytes // per))


def evaluate_chunked(inst, threads, log=print):
    P = inst.patterns
    step = chunk_patterns(inst)
    ll = 0.0
    g = np.zeros(inst.branches)
    cond = np.zeros(inst.branches)
    t0 = time.time()
    for a in range(0, P, step):
        b = min(P, a + step)
        ref = oracle_for(inst.slice_patterns(a, b), blocks=threads)
        lla, ga, _ = ref.branch_gradient(False)
        ll += lla
        g += ga
        cond += ref.gradient_condition()
        del ref
        if log and (a // step) % 20 == 0:
            log(f"  {inst.name}: {b}/{P} patterns, {time.time() - t0:.0f} s")
    return ll, g, cond, time.time() - t0, step


def main(names):
    threads = os.cpu_count() or 1
    for name in names:
        t0 = time.time()
        inst = synth.generate(name, seed=SEED, threads=threads)
        t_gen = time.time() - t0
        dig = synth.instance_digest(inst)
        print(f"{name}: {inst.tip_count} tips, {inst.patterns} patterns, m={inst.states}, generated in {t_gen:.1f} s")
        ll, g, cond, t_eval, step = evaluate_chunked(inst, threads)
        out = dict(name=name, seed=SEED, digest=dig, patterns=inst.patterns, tips=inst.tip_count,
                   states=inst.states, categories=len(inst.cat_rates), logL=ll, gradient=g,
                   rate_gradient=(inst.durations * g) if inst.clock else np.zeros(0),
                   gradient_condition=cond,
                   rate_gradient_condition=(inst.durations * cond) if inst.clock else np.zeros(0),
                   chunk_patterns=step, oracle_seconds=t_eval, oracle_threads=threads)
        np.savez_compressed(os.path.join(HERE, f"full_{name}.npz"), **out)
        print(f"{name}: logL {ll:.10f}, max|g| {np.abs(g).max():.6e}, oracle {t_eval:.0f} s on {threads} threads")


if __name__ == "__main__":
    main(sys.argv[1:] or ["C3", "C4", "C5"])
