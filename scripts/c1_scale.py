"""Generic-kernel check: the C1 model (HKY85, one rate category) at 10^6
columns, timed like bench.py's device leg."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_12146_b200 import _lib as _L  # noqa: E402
from workloads import synth  # noqa: E402

for tips in (64, 512):
    inst = synth.generate("C1", sites=1_000_000, tips=tips)
    eng = synth.engine_for(inst)
    L = _L.lib()
    stream = torch.cuda.current_stream()
    _L.check(L.pg_set_stream(eng.handle, stream.cuda_stream))
    out = torch.zeros(1 + inst.branches, dtype=torch.float64, device="cuda")
    for _ in range(3):
        _L.check(L.pg_evaluate_device(eng.handle, _L.EVAL_GRAD | _L.EVAL_FORCE, out.data_ptr()))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5):
        _L.check(L.pg_evaluate_device(eng.handle, _L.EVAL_GRAD | _L.EVAL_FORCE, out.data_ptr()))
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    P, N, m = inst.patterns, inst.tip_count, 4
    balg = 40 * 1 * m * (N - 2) * P + 2 * N * P
    print(f"tips {tips} patterns {P}: {ms:.2f} ms, {P * inst.branches / ms / 1e-3:.3e} pattern-branch/s, "
          f"B_alg frac {balg / (ms * 1e-3) / 6550.4e9:.3f}, kernel {eng.info()['kernel']}", flush=True)
