"""Time consecutive full evaluations through the device path and the host
API, to see whether per-evaluation time drifts with sustained load."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1905_12146_b200 import _lib as _L
from workloads import synth
inst = synth.generate("C3", sites=int(os.environ.get("SITES", "1000000")))
eng = synth.engine_for(inst)
L = _L.lib()
stream = torch.cuda.current_stream()
_L.check(L.pg_set_stream(eng.handle, stream.cuda_stream))
out = torch.zeros(1 + inst.branches, dtype=torch.float64, device="cuda")
flags = _L.EVAL_RATE_GRAD | _L.EVAL_FORCE
for rnd in range(3):
    for mode in ("device", "host"):
        ts = []
        for i in range(6):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0.record(stream)
            if mode == "device":
                _L.check(L.pg_evaluate_device(eng.handle, flags, out.data_ptr()))
            else:
                eng.set_branch_lengths(inst.branch_lengths * (1 + 1e-12 * (i % 2)))
                eng.rate_gradient()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append((round(e0.elapsed_time(e1), 1), round(1e3 * (time.perf_counter() - t0), 1), eng.last_times_ms()[0]))
        print(rnd, mode, ts, flush=True)
