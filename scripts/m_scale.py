"""5..8-state models (e.g. 6-state) at 256 taxa x 2e5 columns, Gamma-4:
device time per evaluation with the DMMA kernel walkm<8> (default) vs the
generic kernel (PG_NO_WALKM=1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1905_12146_b200 import _lib as _L  # noqa: E402
from paper_1905_12146_b200.api import (EngineOptions, LikelihoodEngine, RateCategories,  # noqa: E402
                                       SitePatternAlignment, SubstitutionModel, Tree)

m = int(sys.argv[1]) if len(sys.argv) > 1 else 6
rng = np.random.default_rng(2)
pi = rng.dirichlet(np.ones(m) * 3)
s = rng.lognormal(0, 0.5, (m, m))
s = (s + s.T) / 2
q = s * pi[None, :]
np.fill_diagonal(q, 0)
np.fill_diagonal(q, -q.sum(1))
q /= -np.sum(pi * np.diag(q))
tr = O.Tree.random(O.Rng(3), 256, 0.005, 0.1)
codes = rng.integers(0, m, size=(256, 200_000)).astype(np.int32)
labels = [tr.labels[i] for i in range(1, 257)]
aln = SitePatternAlignment.from_codes(labels, codes, m)
tree = Tree(256, tr.parent, tr.children, np.concatenate([[0.0], tr.branch_lengths, [0.0]]), tr.labels, tr.post_order)
rates, probs = O.discrete_gamma(0.5, 4)
for env in (None, "1"):
    if env:
        os.environ["PG_NO_WALKM"] = "1"
    eng = LikelihoodEngine(tree, aln, SubstitutionModel(q, pi, True), RateCategories(np.asarray(rates), np.asarray(probs)),
                           EngineOptions())
    Lb = _L.lib()
    stream = torch.cuda.current_stream()
    _L.check(Lb.pg_set_stream(eng.handle, stream.cuda_stream))
    out = torch.zeros(1 + 510, dtype=torch.float64, device="cuda")
    for _ in range(2):
        _L.check(Lb.pg_evaluate_device(eng.handle, _L.EVAL_GRAD | _L.EVAL_FORCE, out.data_ptr()))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(3):
        _L.check(Lb.pg_evaluate_device(eng.handle, _L.EVAL_GRAD | _L.EVAL_FORCE, out.data_ptr()))
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"m={m} {'generic' if env else 'default'}: {e0.elapsed_time(e1) / 3:.2f} ms, kernel {eng.info()['kernel']}",
          flush=True)
    del eng
