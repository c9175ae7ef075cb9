"""4-state model with L = 1, 2, 3, 4, 8 rate categories at 512 taxa x 4e5
columns: device time of one evaluation and the kernel the engine picks."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1905_12146_b200 import _lib as _L  # noqa: E402
from paper_1905_12146_b200.api import (EngineOptions, LikelihoodEngine, RateCategories,  # noqa: E402
                                       SitePatternAlignment, SubstitutionModel, Tree)

base = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
inst_tree = O.Tree.random(O.Rng(3), 512, 0.005, 0.1)
rng = np.random.default_rng(1)
codes = rng.integers(0, 4, size=(512, base)).astype(np.int32)
labels = [inst_tree.labels[i] for i in range(1, 513)]
aln = SitePatternAlignment.from_codes(labels, codes, 4)
tree = Tree(512, inst_tree.parent, inst_tree.children, np.concatenate([[0.0], inst_tree.branch_lengths, [0.0]]),
            inst_tree.labels, inst_tree.post_order)
model = SubstitutionModel.hky85(2.0, [0.3, 0.2, 0.2, 0.3])
for L in (1, 2, 3, 4, 8):
    for env in (None, "1"):
        if env:
            os.environ["PG_NO_WALK4"] = "1"
        else:
            os.environ.pop("PG_NO_WALK4", None)
        rates, probs = ([1.0], [1.0]) if L == 1 else O.discrete_gamma(0.5, L)
        eng = LikelihoodEngine(tree, aln, model, RateCategories(np.asarray(rates), np.asarray(probs)), EngineOptions())
        Lb = _L.lib()
        stream = torch.cuda.current_stream()
        _L.check(Lb.pg_set_stream(eng.handle, stream.cuda_stream))
        out = torch.zeros(1 + 1022, dtype=torch.float64, device="cuda")
        for _ in range(2):
            _L.check(Lb.pg_evaluate_device(eng.handle, _L.EVAL_GRAD | _L.EVAL_FORCE, out.data_ptr()))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            _L.check(Lb.pg_evaluate_device(eng.handle, _L.EVAL_GRAD | _L.EVAL_FORCE, out.data_ptr()))
        e1.record(stream)
        torch.cuda.synchronize()
        print(f"L={L} {'generic' if env else 'default'}: {e0.elapsed_time(e1) / 3:.2f} ms, kernel {eng.info()['kernel']}",
              flush=True)
        del eng
