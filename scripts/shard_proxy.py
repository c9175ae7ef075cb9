"""Single-GPU proxy of the multi-GPU scaling of a config: the per-rank work at
G GPUs is exactly the contiguous pattern block sharding.shard_range(P, r, G)
of the full bench instance, so timing those blocks on one GPU gives each
rank's evaluation time (the 32 KB all-reduce excluded).  Prints one JSON line
per (G, rank): device ms per evaluation (CUDA events, 3 warm-up, 10 timed)
and the implied efficiency T_1 / (G * max_r T_r).

  python scripts/shard_proxy.py [--config C3] [--gpus 1 2 4 8]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_12146_b200 import _lib as _L  # noqa: E402
from paper_1905_12146_b200.sharding import shard_range  # noqa: E402
from workloads import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--gpus", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
full = synth.generate(a.config, threads=os.cpu_count() or 1)
L = _L.lib()
flags = _L.EVAL_GRAD | _L.EVAL_FORCE | (_L.EVAL_RATE_GRAD if full.clock else 0)


def time_block(p0, p1):
    inst = full.slice_patterns(p0, p1)
    eng = synth.engine_for(inst)
    stream = torch.cuda.current_stream()
    _L.check(L.pg_set_stream(eng.handle, stream.cuda_stream))
    out = torch.zeros(1 + inst.branches, dtype=torch.float64, device="cuda")
    for _ in range(3):
        _L.check(L.pg_evaluate_device(eng.handle, flags, out.data_ptr()))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        L.pg_evaluate_device(eng.handle, flags, out.data_ptr())
    e1.record(stream)
    torch.cuda.synchronize()
    _L.check(L.pg_check_errors(eng.handle))
    return e0.elapsed_time(e1) / a.steps, eng.info()


t1 = None
for G in a.gpus:
    ranks = sorted({0, G - 1})  # the first and the last block (sizes differ by at most one pattern)
    worst = 0.0
    for r in ranks:
        p0, p1 = shard_range(full.patterns, r, G)
        ms, info = time_block(p0, p1)
        worst = max(worst, ms)
        print(json.dumps({"config": a.config, "gpus": G, "rank": r, "patterns": p1 - p0, "ms_per_eval": ms,
                          "kernel": info["kernel"], "warps": info["total_warps"]}), flush=True)
    if G == 1:
        t1 = worst
    if t1:
        print(json.dumps({"config": a.config, "gpus": G, "max_rank_ms": worst,
                          "implied_efficiency": t1 / (G * worst)}), flush=True)
