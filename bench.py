#!/usr/bin/env python
"""phylograd-b200 benchmark: pattern x branch gradient updates per second of a
full logL + branch(-rate) gradient evaluation (BASELINE.json metric).

One step = one full evaluation of the hot path over the whole synthetic
workload: P(t) build (K1), post-order + pre-order walk with the fused gradient
(K2), fixed-order reduction with the clock chain rule (K3), and for N > 1 the
NCCL all-reduce of [logL, grad].  Patterns are sharded contiguously over ranks
(weak in the per-GPU sense: each rank owns P/N patterns of the same job; the
job itself is fixed, so scaling is reported as "strong").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl reference]

Default workload: C3 (BASELINE.json configs[2]): 2048-taxon Yule tree,
general non-reversible 4-state Q + Gamma4, 1,000,000 simulated columns,
gradient w.r.t. 4,094 branch-specific clock rates — the largest config and the
one BASELINE.json quotes "1/2/4/8 GPUs" on.  --impl reference times the CPU
restatement of the reference engine (oracle/, "port": the reference itself needs
Eigen + Boost, absent here) on the host cores on a bounded pattern sample.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 12146


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--sites", type=int, default=None, help="override column count (testing only)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=None, help="patterns in the CPU baseline sample")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU work timed for the cpu_baseline (s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--clock-ms", type=int, default=100, help="nvidia-smi sampling period in the timed region (0: off)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def bytes_alg(inst, patterns):
    """B_alg = 40 L m (N-2) P + 2 N P (5 fp64 m-vectors per
    internal non-root node per pattern-category + uint8 tip codes per pass)."""
    L = len(inst.cat_rates)
    m = inst.states
    N = inst.tip_count
    return 40.0 * L * m * (N - 2) * patterns + 2.0 * N * patterns


def flops_alg(inst, patterns):
    L = len(inst.cat_rates)
    return 6.0 * inst.states ** 2 * (inst.tip_count - 2) * L * patterns


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def fp64_tensor_peak():
    """DMMA (mma.sync m8n8k4 f64) peak measured on this pool's B200 by
    scripts/fp64_peak.cu (profiles/fp64_peak_b200.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak_b200.json")) as f:
            for line in f:
                d = json.loads(line)
                if d.get("kernel", "").startswith("dmma"):
                    return float(d["tflops"]), "measured (scripts/fp64_peak.cu)"
    except Exception:
        pass
    return 37.0, "fallback (datasheet)"


def profiled_traffic(config):
    """DRAM bytes per walk launch from the committed ncu capture, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_walk_summary.json")) as f:
            d = json.load(f)
        rec = d.get(config)
        if rec:
            return rec
    except Exception:
        pass
    return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index, period_ms=100):
        self.index = index
        self.period = period_ms
        self.samples = []
        self.proc = None
        self.first = 0
        self.after = False

    def __enter__(self):
        if self.period <= 0:
            return self
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.period)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # the sampler is live before the region starts (nvidia-smi start-up
            # takes longer than a short region)
            t0 = time.time()
            while not self.samples and time.time() - t0 < 10:
                time.sleep(0.005)
            self.first = len(self.samples)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            n = len(self.samples)
            # a region shorter than the period: keep the first sample taken after it
            t0 = time.time()
            while n <= self.first and len(self.samples) <= self.first and time.time() - t0 < 2:
                time.sleep(0.002)
            self.after = n <= self.first
            self.samples = self.samples[self.first:self.first + 1] if self.after else self.samples[self.first:n]
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples),
                **({"note": "region shorter than the sampling period: first sample after it"} if self.after else {})}


def cpu_baseline(inst, sample, threads, target_s=10.0):
    """Oracle (CPU restatement of engine.hpp) timed with the reference's
    `invalidate_caches(); branch_gradient()` idiom (validation.hpp:281-286).
    One evaluation costs a + b P: a fixed part (the B x L transition
    matrices) and a part linear in the pattern count.  The oracle keeps full
    per-node partial grids, so a sample is capped in memory (`sample`
    patterns); two sample sizes (S and S/4) are timed repeatedly until about
    target_s seconds of CPU work, and the full-workload time is a + b P
    (time full-tree chunks, extrapolate linearly in P).
    Returns (pattern-branch/s, description)."""
    from tests.helpers import oracle_for

    P = inst.patterns
    S = min(sample, P)
    big = oracle_for(inst.slice_patterns(0, S), blocks=threads)
    small = None if S == P else oracle_for(inst.slice_patterns(0, max(1, S // 4)), blocks=threads)
    s1 = max(1, S // 4)

    def timed(ref):
        ref.invalidate_caches()
        t0 = time.perf_counter()
        ref.branch_gradient()
        return time.perf_counter() - t0

    timed(big)  # warm-up
    if small is not None:
        timed(small)
    tb, ts, total = [], [], 0.0
    while len(tb) < 3 or total < target_s:
        tb.append(timed(big))
        total += tb[-1]
        if small is not None:
            ts.append(timed(small))
            total += ts[-1]
        if len(tb) >= 50:
            break
    t_big = statistics.median(tb)
    if small is None:
        t_full, how = t_big, f"all {P} patterns, median of {len(tb)}"
    else:
        t_small = statistics.median(ts)
        slope = max(0.0, (t_big - t_small) / (S - s1))
        fixed = max(0.0, t_big - slope * S)
        t_full = fixed + slope * P
        how = (f"samples of {S} and {s1} of {P} patterns (median of {len(tb)} each), fitted "
               f"{fixed * 1e3:.1f} ms + {slope * 1e6:.3f} us/pattern, extrapolated to {P}")
    return P * inst.branches / t_full, f"{how}; {total:.1f} s of CPU time"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def default_sample(inst):
    """Bounded CPU sample: the restated reference keeps full per-node partial
    grids (post, pre, edge: ~5 N L m doubles per pattern, engine.hpp:85-99), so
    the sample is capped at ~6 GB of host memory; cost is exactly linear in P."""
    per_pattern = 5.0 * inst.tip_count * len(inst.cat_rates) * inst.states * 8
    return int(max(32, min(inst.patterns, 6.0e9 / per_pattern)))


def run_reference(args, inst):
    threads = os.cpu_count() or 1
    sample = args.cpu_sample or default_sample(inst)
    B = inst.branches
    rates = []
    from tests.helpers import oracle_for

    sub = inst.slice_patterns(0, min(sample, inst.patterns))
    ref = oracle_for(sub, blocks=threads)
    for _ in range(max(args.warmup, 1)):
        ref.invalidate_caches()
        ref.branch_gradient()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ref.invalidate_caches()
        ref.branch_gradient()
    t = (time.perf_counter() - t0) / args.steps
    # one evaluation is a + b P (fixed transition-matrix build + per pattern):
    # the fixed part is measured on a quarter sample and the step time is
    # extrapolated to the full pattern count, so the sample
    # does not charge the fixed part to too few patterns
    how = f"{sub.patterns} of {inst.patterns} patterns per step"
    value = sub.patterns * B / t
    if sub.patterns < inst.patterns and sub.patterns >= 8:
        small = oracle_for(inst.slice_patterns(0, sub.patterns // 4), blocks=threads)
        ts = []
        for _ in range(3):
            small.invalidate_caches()
            t1 = time.perf_counter()
            small.branch_gradient()
            ts.append(time.perf_counter() - t1)
        t_small = statistics.median(ts)
        slope = max(0.0, (t - t_small) / (sub.patterns - sub.patterns // 4))
        fixed = max(0.0, t - slope * sub.patterns)
        value = inst.patterns * B / (fixed + slope * inst.patterns)
        how += (f", extrapolated to all {inst.patterns} ({fixed * 1e3:.1f} ms fixed + "
                f"{slope * 1e6:.3f} us/pattern, fixed part from a {sub.patterns // 4}-pattern sample)")
    line = {
        "impl": "reference", "metric": "pattern x branch gradient updates/s (full logL + grad eval)",
        "value": value, "unit": "pattern-branch/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded; BASELINE.json config)",
        "config": {"workload": args.config, "sample_patterns": sub.patterns, "full_patterns": inst.patterns,
                   "branches": B, "tips": inst.tip_count, "states": inst.states,
                   "categories": len(inst.cat_rates)},
        "cpu_baseline": {"value": value, "unit": "pattern-branch/s", "cores": threads, "kind": "port",
                         "sample": f"{how}, full tree, {threads} pattern blocks on std::threads; {cpu_model()}"},
        "e2e": {"value": value, "unit": "pattern-branch/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    rank, world, local = dist_env()
    from paper_1905_12146_b200 import synth

    if args.impl == "reference":
        if rank != 0:
            return 0
        inst = synth.generate(args.config, seed=SEED, sites=args.sites)
        run_reference(args, inst)
        return 0

    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    t_gen = time.perf_counter()
    inst = synth.generate_shared(args.config, rank, world, (lambda: torch.distributed.barrier()) if world > 1 else None,
                                 tag=str(os.getppid()), seed=SEED, sites=args.sites)
    t_gen = time.perf_counter() - t_gen
    P_total = inst.patterns
    p0, p1 = P_total * rank // world, P_total * (rank + 1) // world
    shard = inst.slice_patterns(p0, p1)
    from paper_1905_12146_b200 import _lib as _L
    from paper_1905_12146_b200.api import EngineOptions

    eng = synth.engine_for(shard, EngineOptions(device=local))
    L = _L.lib()
    B = inst.branches
    stream = torch.cuda.current_stream()
    _L.check(L.pg_set_stream(eng.handle, stream.cuda_stream))
    flags = (_L.EVAL_RATE_GRAD if inst.clock else _L.EVAL_GRAD) | _L.EVAL_FORCE
    out = torch.zeros(1 + B, dtype=torch.float64, device="cuda")

    def step_device():
        _L.check(L.pg_evaluate_device(eng.handle, flags, out.data_ptr()))
        if world > 1:
            torch.distributed.all_reduce(out)

    for _ in range(args.warmup):
        step_device()
    _L.check(L.pg_check_errors(eng.handle))

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timed region (value)
    import ctypes as C

    _L.check(L.pg_timing(eng.handle, 1, None, None, None))
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local, args.clock_ms) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step_device()
        ev1.record(stream)
        barrier()
    _L.check(L.pg_check_errors(eng.handle))
    ms = ev0.elapsed_time(ev1) / args.steps
    n_ev, walk_tot, eval_tot = C.c_int(), C.c_double(), C.c_double()
    _L.check(L.pg_timing(eng.handle, 0, C.byref(n_ev), C.byref(walk_tot), C.byref(eval_tot)))
    walk_ms = walk_tot.value / max(n_ev.value, 1)
    t = torch.tensor([ms, walk_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms, walk_ms_max = float(t[0]), float(t[1])
    logl = float(out[0])

    # ---- end-to-end through the public API with host buffers (e2e)
    b_host = [torch.from_numpy(inst.branch_rates if inst.clock else inst.branch_lengths).double().pin_memory()]
    b_host.append((b_host[0] * (1.0 + 1e-12)).pin_memory())
    res_host = torch.empty(1 + B, dtype=torch.float64).pin_memory()
    b_dev = torch.empty(B, dtype=torch.float64, device="cuda")
    dt_dev = torch.from_numpy(inst.durations).cuda() if inst.clock else None

    b_np = [inst.branch_rates if inst.clock else inst.branch_lengths]
    b_np.append(b_np[0] * (1.0 + 1e-12))

    def step_e2e(i):
        if world == 1:
            # the user-facing call: host vector in, GradientReport (host) out
            b = b_np[i % 2] * inst.durations if inst.clock else b_np[i % 2]   # b_i = r_i dt_i (clock.hpp:42-55)
            eng.set_branch_lengths(b)
            rep = eng.rate_gradient() if inst.clock else eng.branch_gradient()
            return rep.log_likelihood
        b_dev.copy_(b_host[i % 2], non_blocking=True)  # H2D of this step's rates / lengths
        bl = b_dev * dt_dev if inst.clock else b_dev
        _L.check(L.pg_set_branch_lengths_device(eng.handle, bl.data_ptr()))
        _L.check(L.pg_evaluate_device(eng.handle, flags, out.data_ptr()))
        torch.distributed.all_reduce(out)
        res_host.copy_(out, non_blocking=True)             # D2H of [logL, grad]
        torch.cuda.current_stream().synchronize()
        _L.check(L.pg_check_errors(eng.handle))
        return float(res_host[0])

    # consecutive steps alternate between two distinct vectors so no step can
    # hit the engine's "bit-identical lengths" cache (engine.hpp:121)
    nw = max(1, args.warmup)
    for i in range(nw):
        step_e2e(i)
    barrier()
    t0 = time.perf_counter()
    e2e_walk = []
    for i in range(nw, nw + args.steps):
        step_e2e(i)
        if world == 1:
            e2e_walk.append(round(eng.last_times_ms()[0], 2))
    barrier()
    e2e_s = (time.perf_counter() - t0) / args.steps
    print(f"e2e walk ms per step: {e2e_walk}", file=sys.stderr)
    te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
    e2e_s = float(te[0])

    if rank == 0:
        prof = profiled_traffic(args.config)
        if inst.states > 32:
            # codon path: fp64 tensor-core bound (AI = 9.2 flop/B)
            peak, peak_kind = fp64_tensor_peak()
            falg = flops_alg(inst, p1 - p0)
            achieved = falg / (walk_ms_max * 1e-3) / 1e12
            roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                    "peak_source": peak_kind, "algorithmic_flops_per_launch": falg}
        else:
            peak, peak_kind = measured_peaks()
            balg = bytes_alg(inst, p1 - p0)
            achieved = balg / (walk_ms_max * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "peak_source": peak_kind, "algorithmic_bytes_per_launch": balg}
        roof.update({"kernel": eng.info()["kernel"] + " (post + pre + fused gradient)", "walk_ms": walk_ms_max,
                     "traffic": prof["dram_bytes_per_launch"] if prof else None,
                     "traffic_source": prof.get("source") if prof else None})
        if prof:
            # pipe utilisation of the same ncu capture (DMMA sub-pipe for the
            # tensor-bound kernels, fp64 FMA pipe and DRAM throughput otherwise)
            for k in ("dmma_pipe_active_pct", "fp64_pipe_active_pct", "dram_throughput_pct_of_peak"):
                if k in prof:
                    roof["ncu_" + k] = prof[k]
        value = P_total * B / (ms * 1e-3)
        info = eng.info()
        line = {
            "metric": "pattern x branch gradient updates/s (full logL + grad eval)",
            "value": value, "unit": "pattern-branch/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded; BASELINE.json config shapes)",
            "config": {"workload": args.config, "description": synth.DESCRIPTIONS[args.config],
                       "patterns": P_total, "branches": B, "tips": inst.tip_count, "states": inst.states,
                       "categories": len(inst.cat_rates),
                       "gradient": "branch rates (dt*g)" if inst.clock else "branch lengths",
                       "parallelism": f"pattern-shard dp{world}",
                       "l2": "inputs larger than L2 (edge scratch + tip codes >> 126 MB); no flush",
                       "setup_s": round(t_gen, 2), "geometry": info},
            "roofline": roof,
            "e2e": {"value": P_total * B / e2e_s, "unit": "pattern-branch/s", "ms_per_step": e2e_s * 1e3,
                    "h2d_bytes_per_step": 8 * B, "d2h_bytes_per_step": 8 * (1 + B)},
            "gpu_launches": info["launches"] * args.steps,
            "clocks": clocks.summary(),
            "logL": logl,
        }
        if not args.no_cpu_baseline and world == 1:
            threads = os.cpu_count() or 1
            sample = args.cpu_sample or default_sample(inst)
            cpu_value, how = cpu_baseline(inst, sample, threads, args.cpu_seconds)
            line["cpu_baseline"] = {"value": cpu_value, "unit": "pattern-branch/s", "cores": threads, "kind": "port",
                                    "sample": f"full tree, invalidate+gradient: {how}; {cpu_model()}"}
            if threads > 1:
                # SURVEY.md §8d variant (i): one thread, like the reference engine
                # (engine.hpp:13-17), on a quarter of the sample
                v1, how1 = cpu_baseline(inst, max(8, sample // 4), 1, min(args.cpu_seconds, 4.0))
                line["cpu_baseline"]["single_thread"] = {"value": v1, "cores": 1, "sample": how1}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
