"""Small driver for ncu: builds one engine on a config sample and runs a few
full evaluations (launch order per evaluation: tc_kernel, walk_kernel, reduce)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--sites", type=int, default=100000)
ap.add_argument("--evals", type=int, default=2)
ap.add_argument("--hess", action="store_true")
a = ap.parse_args()
inst = synth.generate(a.config, sites=a.sites or None)
eng = synth.engine_for(inst)
for i in range(a.evals):
    eng.invalidate_caches()
    t = time.perf_counter()
    rep = eng.branch_gradient(a.hess)
    print(f"eval {i}: logL {rep.log_likelihood:.6f} {1e3 * (time.perf_counter() - t):.2f} ms, walk/total ms "
          f"{eng.last_times_ms()}, {inst.patterns} patterns, geometry {eng.info()}", flush=True)
