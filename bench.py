#!/usr/bin/env python
"""phylograd-b200 benchmark: pattern x branch gradient updates per second of a
full logL + branch(-rate) gradient evaluation (BASELINE.json metric).

One step = one full evaluation of the hot path over the whole synthetic
workload: P(t) build (K1), post-order + pre-order walk with the fused gradient
(K2), fixed-order reduction with the clock chain rule (K3), and for N > 1 the
NCCL all-reduce of [logL, grad].  The job (all patterns of the config) is
fixed; N ranks each own a contiguous block of it (scaling "strong").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl reference]

--gpus N > 1 outside torchrun re-launches itself under
torch.distributed.run with N processes (one per GPU, 127.0.0.1 rendezvous).

Default workload: C3 (BASELINE.json configs[2]): 2048-taxon Yule tree,
general non-reversible 4-state Q + Gamma4, 1,000,000 simulated columns,
gradient w.r.t. 4,094 branch-specific clock rates — the largest config and the
one BASELINE.json quotes "1/2/4/8 GPUs" on.  --impl reference times the CPU
restatement of the reference engine (oracle/, "port": the reference itself needs
Eigen + Boost, absent here) on the host cores on a bounded pattern sample; its
inputs come from workloads/ (a host library separate from the product), so the
reference arm never maps libphylograd_b200.so.

At full size the device arm checks its result against the committed
full-size oracle fixture (tests/golden/full_<config>.npz, made by
tests/golden/make_fullsize.py) and reports it as "parity".
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 12146
METRIC = "pattern x branch gradient updates/s (full logL + grad eval)"
UNIT = "pattern-branch/s"
L2_NOTE = "inputs larger than L2 (edge scratch + tip codes >> 126 MB); no flush"
PARALLELISM = "contiguous pattern blocks (GPU: one rank per GPU + NCCL all-reduce; CPU: std::thread blocks)"


def parse_args(argv=None):
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
    ap.add_argument("--no-parity", action="store_true", help="skip the full-size fixture check")
    ap.add_argument("--clock-ms", type=int, default=100, help="nvidia-smi sampling period in the timed region (0: off)")
    ap.add_argument("--also", default=None,
                    help="comma-separated extra workloads summarised under other_workloads after the main line is "
                         "measured (default: C2,C4,C5 for the plain one-GPU C3 run; '' turns it off)")
    return ap.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_command(args, argv):
    """--gpus N > 1 outside torchrun: the same command under
    torch.distributed.run, one process per GPU (None: run in this process)."""
    if "WORLD_SIZE" in os.environ or args.gpus <= 1 or args.impl == "reference":
        return None
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + list(argv)


# ------------------------------------------------------------ work models
def bytes_alg(inst, patterns):
    """Algorithmic DRAM bytes of one evaluation: every
    internal non-root node's edge message e = P p (L m doubles per pattern) is
    written once by the post-order pass and read once by the pre-order pass —
    the pre-order step of a node needs both children's e, and no e survives on
    chip across the whole post pass — plus the uint8 tip codes read once per
    pass: 16 L m (N-2) P + 2 N P.  (The pre-partial of the child visited next
    stays on chip; the deferred one is re-read from L2.)"""
    L = len(inst.cat_rates)
    return 16.0 * L * inst.states * (inst.tip_count - 2) * patterns + 2.0 * inst.tip_count * patterns


def bytes_survey(inst, patterns):
    """SURVEY.md §8d canonical B_alg = 40 L m (N-2) P + 2 N P (5 materialised
    m-vectors per internal node-category): kept for comparison only."""
    L = len(inst.cat_rates)
    return 40.0 * L * inst.states * (inst.tip_count - 2) * patterns + 2.0 * inst.tip_count * patterns


def flops_alg(inst, patterns):
    """SURVEY.md §8d F_alg = 6 m^2 (N-2) L P: three dense m x m mat-vecs per
    internal non-root node per pattern-category."""
    L = len(inst.cat_rates)
    return 6.0 * inst.states ** 2 * (inst.tip_count - 2) * L * patterns


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
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
                    return float(d["tflops"]), "measured (scripts/fp64_peak.cu, profiles/fp64_peak_b200.json)"
    except Exception:
        pass
    return 37.0, "fallback (datasheet)"


def profiled_traffic(config, patterns, world):
    """DRAM bytes per walk launch from the committed full-size ncu capture of
    this config — only when this run is that workload (same pattern count,
    one GPU); otherwise None."""
    if world != 1:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_walk_summary.json")) as f:
            rec = json.load(f).get(config)
        if rec and int(rec.get("patterns", -1)) == int(patterns):
            return rec
    except Exception:
        pass
    return None


def roofline_block(inst, patterns, walk_ms, kernel, world, config):
    """Roofline of the dominant kernel (the walk), bound as BASELINE.json's
    north star frames it: HBM bandwidth for the 4- and 20-state models, the
    fp64 tensor (DMMA) peak for codons.  The arithmetic intensity F_alg /
    B_alg and the ridge of the measured peaks are reported beside it (the
    20-state model sits above the ridge at its design-floor traffic, so its
    HBM fraction is bounded well below one)."""
    hbm, hbm_src = measured_peaks()
    tf, tf_src = fp64_tensor_peak()
    balg, falg = bytes_alg(inst, patterns), flops_alg(inst, patterns)
    t = walk_ms * 1e-3
    ridge = tf * 1e12 / (hbm * 1e9)
    prof = profiled_traffic(config, inst.patterns, world)
    if inst.states > 32:
        achieved = falg / t / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tf, "unit": "TFLOP/s", "frac": achieved / tf,
                "peak_source": tf_src}
    else:
        achieved = balg / t / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "peak_source": hbm_src}
    roof.update({
        "traffic": prof["dram_bytes_per_launch"] if prof else None,
        "kernel": kernel + " (post + pre + fused gradient)", "walk_ms": walk_ms,
        "algorithmic_bytes_per_launch": balg, "algorithmic_flops_per_launch": falg,
        "bytes_model": "16 L m (N-2) P + 2 N P (edge message of each internal non-root node written once, read once)",
        "arithmetic_intensity": falg / balg, "ridge_flop_per_byte": ridge,
        "survey_b_alg_bytes": bytes_survey(inst, patterns),
        "survey_b_alg_frac_of_hbm": bytes_survey(inst, patterns) / t / 1e9 / hbm,
    })
    if prof:
        dram = prof["dram_bytes_per_launch"] / t / 1e9
        roof.update({"traffic_source": prof.get("source"), "dram_achieved_gbps": dram, "dram_frac_of_hbm": dram / hbm,
                     "traffic_over_algorithmic": prof["dram_bytes_per_launch"] / balg})
        if prof["dram_bytes_per_launch"] < balg:
            roof["traffic_note"] = ("below the algorithmic bytes: the walk never materialises the edge messages of "
                                    "cherries (tabulated per tip-code pair, DESIGN.md section 2.1)")
        for k in ("dmma_pipe_active_pct", "fp64_pipe_active_pct", "dram_throughput_pct_of_peak"):
            if k in prof:
                roof["ncu_" + k] = prof[k]
    return roof


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


def bench_config(args, inst):
    """The workload description, identical in both arms (same keys, same
    values), so the driver's same-config check compares like with like."""
    from workloads import synth

    return {"workload": args.config, "description": synth.DESCRIPTIONS[args.config], "seed": SEED,
            "sites": int(inst.weights.sum()), "patterns": inst.patterns, "branches": inst.branches,
            "tips": inst.tip_count, "states": inst.states, "categories": len(inst.cat_rates),
            "gradient": "branch rates (dt*g)" if inst.clock else "branch lengths", "parallelism": PARALLELISM,
            "l2": L2_NOTE}


def parity_block(args, inst, logl, grad):
    """The device result against the full-size oracle fixture of this exact
    workload (tests/golden/full_<config>.npz; instance digest must match)."""
    from workloads import synth

    path = os.path.join(ROOT, "tests", "golden", f"full_{args.config}.npz")
    rel = os.path.relpath(path, ROOT)
    if args.sites is not None or not os.path.exists(path):
        return {"fixture": None, "note": "no full-size fixture for this workload"}
    fx = np.load(path)
    if synth.instance_digest(inst) != str(fx["digest"]):
        return {"fixture": rel, "match": False, "note": "instance digest differs from the fixture's"}
    want = fx["rate_gradient"] if inst.clock else fx["gradient"]
    ckey = "rate_gradient_condition" if inst.clock else "gradient_condition"
    cond = fx[ckey] if ckey in fx.files else None
    g = np.asarray(grad)
    err = np.abs(g - want)
    scale = float(np.max(np.abs(want)))
    tol = 1e-9 * np.abs(want) + 1e-12 * scale
    if cond is not None:
        # SURVEY.md §8d condition-aware variant for cancelling components (the
        # reference's own eigen-vs-Pade P(t) spread is ~7e-11 of the condition)
        tol = np.maximum(tol, 1e-10 * cond)
    ok = bool(np.all(np.isfinite(g)) and np.all(err <= tol))
    ll_rel = abs(logl - float(fx["logL"])) / abs(float(fx["logL"]))
    out = {"fixture": rel, "match": True, "logL_rel": ll_rel,
           "grad_max_rel": float(np.max(err / np.maximum(np.abs(want), 1e-300))),
           "grad_max_rel_to_scale": float(np.max(err) / scale),
           "components_over_1e-9_rel": int(np.sum(err > 1e-9 * np.abs(want))),
           "within_1e-9": bool(ok and ll_rel <= 1e-9), "oracle_threads": int(fx["oracle_threads"])}
    if cond is not None:
        out["grad_max_rel_to_condition"] = float(np.max(err / np.maximum(cond, 1e-300)))
    return out


def other_workloads(args):
    """BASELINE.json's other single-GPU configs, each measured by its own
    `bench.py --config Cx` process after this run's engine was released (same
    steps / warm-up, full-size parity fixture, no CPU leg), summarised so that
    the driver's one line carries a measured number for every kernel family."""
    out = []
    for cfg in [c for c in args.also.split(",") if c]:
        cmd = [sys.executable, os.path.abspath(__file__), "--config", cfg, "--steps", str(args.steps), "--warmup",
               str(args.warmup), "--no-cpu-baseline", "--also", "", "--clock-ms", str(args.clock_ms)]
        t0 = time.perf_counter()
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
            d = json.loads(r.stdout.strip().splitlines()[-1])
            rf, par = d["roofline"], d.get("parity") or {}
            out.append({
                "workload": cfg, "patterns": d["config"]["patterns"], "branches": d["config"]["branches"],
                "states": d["config"]["states"], "kernel": d["geometry"]["kernel"], "ms_per_step": d["ms_per_step"],
                "value": d["value"], "e2e_value": d["e2e"]["value"], "unit": d["unit"], "steps": d["steps"],
                "roofline": {k: rf.get(k) for k in ("bound", "achieved", "peak", "unit", "frac", "walk_ms",
                                                      "dram_frac_of_hbm")},
                "parity": {k: par.get(k) for k in ("fixture", "logL_rel", "grad_max_rel", "grad_max_rel_to_condition",
                                                    "components_over_1e-9_rel", "within_1e-9")},
                "gpu_launches": d["gpu_launches"], "sm_mhz": (d.get("clocks") or {}).get("sm_mhz"),
                "wall_s": round(time.perf_counter() - t0, 1)})
        except Exception as e:  # the main line must not depend on the extras
            out.append({"workload": cfg, "error": f"{type(e).__name__}: {e}"[:300]})
    return out


def run_reference(args, inst):
    threads = os.cpu_count() or 1
    sample = args.cpu_sample or default_sample(inst)
    B = inst.branches
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
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": UNIT, "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded; BASELINE.json config shapes)",
        "config": bench_config(args, inst),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{how}, full tree, {threads} pattern blocks on std::threads; {cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_device(args):
    import torch

    from workloads import synth

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    t_gen = time.perf_counter()
    # columns simulated and compressed on this rank's GPU (counter-stream
    # configs; the reference arm builds the identical instance on the host)
    inst = synth.generate_shared(args.config, rank, world, (lambda: torch.distributed.barrier()) if world > 1 else None,
                                 tag=str(os.getppid()), seed=SEED, sites=args.sites, device=local)
    t_gen = time.perf_counter() - t_gen
    P_total = inst.patterns
    from paper_1905_12146_b200 import _lib as _L
    from paper_1905_12146_b200.api import EngineOptions

    opts = EngineOptions(device=local)
    if world > 1:
        # the product's ShardedEngine: this rank's contiguous block + one
        # NCCL all-reduce of [logL, g] per evaluation on the engine stream
        from paper_1905_12146_b200.sharding import ShardedEngine

        sh = ShardedEngine(*synth.api_objects(inst), opts)
        if inst.clock:
            sh.set_clock_durations(inst.durations)
        eng, p0, p1 = sh.local, sh.p0, sh.p1
    else:
        sh, eng, p0, p1 = None, synth.engine_for(inst, opts), 0, P_total
    L = _L.lib()
    B = inst.branches
    stream = torch.cuda.current_stream()
    _L.check(L.pg_set_stream(eng.handle, stream.cuda_stream))
    flags = (_L.EVAL_RATE_GRAD if inst.clock else _L.EVAL_GRAD) | _L.EVAL_FORCE
    out = torch.zeros(1 + B, dtype=torch.float64, device="cuda")

    def step_device():
        if sh is not None:
            sh.enqueue_device(flags, out)
        else:
            _L.check(L.pg_evaluate_device(eng.handle, flags, out.data_ptr()))

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
    # the device error flags are sticky until read: this reports a non-finite
    # or underflowed site in ANY of the timed evaluations
    _L.check(L.pg_check_errors(eng.handle))
    ms = ev0.elapsed_time(ev1) / args.steps
    n_ev, walk_tot, eval_tot = C.c_int(), C.c_double(), C.c_double()
    _L.check(L.pg_timing(eng.handle, 0, C.byref(n_ev), C.byref(walk_tot), C.byref(eval_tot)))
    walk_ms = walk_tot.value / max(n_ev.value, 1)
    t = torch.tensor([ms, walk_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms, walk_ms_max = float(t[0]), float(t[1])
    res = out.cpu().numpy()
    logl = float(res[0])

    # ---- end-to-end through the public API with host buffers (e2e)
    b_np = [inst.branch_rates if inst.clock else inst.branch_lengths]
    b_np.append(b_np[0] * (1.0 + 1e-12))

    def step_e2e(i):
        # the user-facing call: host vector in (H2D inside set_branch_lengths),
        # GradientReport on the host out (D2H of [logL, g])
        b = b_np[i % 2] * inst.durations if inst.clock else b_np[i % 2]   # b_i = r_i dt_i (clock.hpp:42-55)
        target = sh if sh is not None else eng
        target.set_branch_lengths(b)
        rep = target.rate_gradient() if inst.clock else target.branch_gradient()
        return rep.log_likelihood

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
        e2e_walk.append(round(eng.last_times_ms()[0], 2))
    barrier()
    e2e_s = (time.perf_counter() - t0) / args.steps
    print(f"e2e walk ms per step: {e2e_walk}", file=sys.stderr)
    te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
    e2e_s = float(te[0])

    if rank == 0:
        info = eng.info()
        nccl = {"world_size": world, "comm_size": world, "version": None}
        if world > 1:
            nccl["comm_size"] = torch.distributed.get_world_size()
            nccl["version"] = ".".join(str(v) for v in torch.cuda.nccl.version())
        line = {
            "metric": METRIC, "value": P_total * B / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "world_size": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded; BASELINE.json config shapes)",
            "config": bench_config(args, inst),
            "roofline": roofline_block(inst, p1 - p0, walk_ms_max, info["kernel"], world, args.config),
            "e2e": {"value": P_total * B / e2e_s, "unit": UNIT, "ms_per_step": e2e_s * 1e3,
                    "h2d_bytes_per_step": 8 * B, "d2h_bytes_per_step": 8 * (1 + B)},
            "gpu_launches": info["launches"] * args.steps,
            "clocks": clocks.summary(),
            "logL": logl,
            "parity": None if args.no_parity else parity_block(args, inst, logl, res[1:1 + B]),
            "nccl": nccl,
            "geometry": info, "setup_s": round(t_gen, 2), "shard_patterns": p1 - p0,
            "errors_checked": "every timed step (sticky device error flags read after the region)",
        }
        if not args.no_cpu_baseline and world == 1:
            threads = os.cpu_count() or 1
            sample = args.cpu_sample or default_sample(inst)
            cpu_value, how = cpu_baseline(inst, sample, threads, args.cpu_seconds)
            line["cpu_baseline"] = {"value": cpu_value, "unit": UNIT, "cores": threads, "kind": "port",
                                    "sample": f"full tree, invalidate+gradient: {how}; {cpu_model()}"}
            if threads > 1:
                # SURVEY.md §8d variant (i): one thread, like the reference engine
                # (engine.hpp:13-17), on a quarter of the sample
                v1, how1 = cpu_baseline(inst, max(8, sample // 4), 1, min(args.cpu_seconds, 4.0))
                line["cpu_baseline"]["single_thread"] = {"value": v1, "cores": 1, "sample": how1}
        also = args.also
        if also is None:
            also = "C2,C4,C5" if (args.config == "C3" and world == 1 and args.sites is None) else ""
        if also and world == 1:
            # release this run's engine (its scratch is a fixed share of the
            # device memory) before the other workloads' processes start
            import gc

            args.also = also
            del eng, sh, out, step_device, step_e2e
            gc.collect()
            torch.cuda.empty_cache()
            line["other_workloads"] = other_workloads(args)
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse_args(argv)
    cmd = relaunch_command(args, argv)
    if cmd is not None:
        return subprocess.call(cmd)
    rank, world, local = dist_env()
    if args.impl == "reference":
        # rank 0 alone times the CPU reference; other torchrun ranks exit
        if rank != 0:
            return 0
        from workloads import synth

        run_reference(args, synth.generate(args.config, seed=SEED, sites=args.sites))
        return 0
    if world != args.gpus:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    return run_device(args)


if __name__ == "__main__":
    sys.exit(main())
