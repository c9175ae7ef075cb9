"""Pattern sharding across GPUs (one process per GPU, torch.distributed).

Site patterns are independent and logL / gradient / Hessian diagonal are sums
over patterns (engine.hpp:217, :268), so rank r owns the
contiguous block [floor(r P / G), floor((r+1) P / G)) and runs both traversals
locally.  The only collective on the path is one all-reduce of
[logL, g (2N-2), H (2N-2)] per evaluation; over NCCL it is issued on the
engine's stream straight from the device output buffer.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np


def shard_range(patterns: int, rank: int, world: int):
    """Contiguous block of patterns owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: bad rank/world")
    return patterns * rank // world, patterns * (rank + 1) // world


def slice_alignment(aln, p0: int, p1: int):
    from .api import SitePatternAlignment

    return SitePatternAlignment(aln.taxa(), aln.state_count(), aln.codes[:, p0:p1], aln.weights()[p0:p1],
                                aln.ambiguity, None, None)


class ShardedEngine:
    """LikelihoodEngine over this rank's pattern shard + one all-reduce.

    ``engine_factory`` builds the local engine (default: the GPU
    LikelihoodEngine); tests substitute the CPU oracle to exercise the
    sharding and reduction logic on gloo without a GPU.
    """

    def __init__(self, tree, alignment, model, categories, options=None, group=None,
                 engine_factory: Optional[Callable] = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.p0, self.p1 = shard_range(alignment.pattern_count(), self.rank, self.world)
        local_aln = slice_alignment(alignment, self.p0, self.p1)
        if engine_factory is None:
            from .api import LikelihoodEngine

            engine_factory = LikelihoodEngine
        self.local = engine_factory(tree, local_aln, model, categories, options)
        self.B = tree.branch_count()
        self._device_path = dist.get_backend(group) == "nccl" and hasattr(self.local, "handle")

    def set_branch_lengths(self, b):
        self.local.set_branch_lengths(b)

    def invalidate_caches(self):
        self.local.invalidate_caches()

    def _reduce_host(self, vec: np.ndarray) -> np.ndarray:
        import torch

        t = torch.from_numpy(np.ascontiguousarray(vec, dtype=np.float64))
        self.dist.all_reduce(t, group=self.group)
        return t.numpy()

    def set_clock_durations(self, dt):
        if hasattr(self.local, "set_clock_durations"):
            self.local.set_clock_durations(dt)
        self.durations = np.asarray(dt, dtype=np.float64).copy()

    def enqueue_device(self, flags, out):
        """Asynchronous step of the NCCL path: this rank's evaluation into the
        CUDA tensor `out` ([logL, g (, h)]) on the current stream, then the
        all-reduce on the same stream.  pg_check_errors (check_errors) reports
        a failure of any step enqueued since the last check (sticky flags)."""
        import torch

        from . import _lib as _L

        L = _L.lib()
        _L.check(L.pg_set_stream(self.local.handle, torch.cuda.current_stream().cuda_stream))
        _L.check(L.pg_evaluate_device(self.local.handle, flags, out.data_ptr()))
        self.dist.all_reduce(out, group=self.group)

    def check_errors(self):
        from . import _lib as _L

        _L.check(_L.lib().pg_check_errors(self.local.handle))

    def _device_eval(self, flags):
        import torch

        from . import _lib as _L

        width = 1 + self.B * (2 if flags & _L.EVAL_HESS else 1)
        out = torch.zeros(width, dtype=torch.float64, device="cuda")
        self.enqueue_device(flags, out)
        self.check_errors()
        return out.cpu().numpy()

    def branch_gradient(self, with_hessian_diagonal=False):
        from .api import GradientReport

        if self._device_path:
            from . import _lib as _L

            v = self._device_eval(_L.EVAL_GRAD | (_L.EVAL_HESS if with_hessian_diagonal else 0))
        else:
            rep = self.local.branch_gradient(with_hessian_diagonal)
            ll, g, h = (rep if isinstance(rep, tuple) else
                        (rep.log_likelihood, rep.branch_gradient, rep.hessian_diagonal))
            parts = [np.array([ll]), np.asarray(g)]
            if with_hessian_diagonal:
                parts.append(np.asarray(h))
            v = self._reduce_host(np.concatenate(parts))
        return GradientReport(float(v[0]), v[1:1 + self.B].copy(),
                              v[1 + self.B:].copy() if with_hessian_diagonal else np.zeros(0),
                              self.p1 - self.p0, 0)

    def rate_gradient(self, with_hessian_diagonal=False):
        """d logL / d r_i = dt_i g_i for b_i = r_i dt_i (clock.hpp:146-152,
        cli.hpp:437-438): on the device path the chain rule runs in the
        engine's reduction kernel; on the host path it scales the reduced g."""
        from .api import GradientReport

        if self._device_path:
            from . import _lib as _L

            v = self._device_eval(_L.EVAL_RATE_GRAD | (_L.EVAL_HESS if with_hessian_diagonal else 0))
            return GradientReport(float(v[0]), v[1:1 + self.B].copy(),
                                  v[1 + self.B:].copy() if with_hessian_diagonal else np.zeros(0),
                                  self.p1 - self.p0, 0)
        rep = self.branch_gradient(with_hessian_diagonal)
        dt = self.durations
        return GradientReport(rep.log_likelihood, dt * rep.branch_gradient,
                              dt * dt * rep.hessian_diagonal if with_hessian_diagonal else np.zeros(0),
                              rep.pattern_count, 0)

    def log_likelihood(self):
        ll = self.local.log_likelihood()
        return float(self._reduce_host(np.array([ll]))[0])
