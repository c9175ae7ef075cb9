"""Device time of one full evaluation (K1+K2+K3) for a config, without the
error check (used to time deliberately broken variants in A/B experiments)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_12146_b200 import _lib as _L  # noqa: E402
from workloads import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
inst = synth.generate(cfg)
eng = synth.engine_for(inst)
L = _L.lib()
stream = torch.cuda.current_stream()
_L.check(L.pg_set_stream(eng.handle, stream.cuda_stream))
out = torch.zeros(1 + inst.branches, dtype=torch.float64, device="cuda")
flags = _L.EVAL_GRAD | _L.EVAL_FORCE
for _ in range(3):
    L.pg_evaluate_device(eng.handle, flags, out.data_ptr())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(5):
    L.pg_evaluate_device(eng.handle, flags, out.data_ptr())
e1.record(stream)
torch.cuda.synchronize()
print(f"{cfg} {e0.elapsed_time(e1) / 5:.2f} ms/eval", flush=True)
