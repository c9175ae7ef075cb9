"""bench.py contract checks that need no GPU: the reference arm (`--impl
reference`, the CPU oracle port timed on the host) prints one JSON line with
the keys the driver reads, on the same metric/unit as the device arm."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "C1", "--steps", "1",
                          "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == "pattern x branch gradient updates/s (full logL + grad eval)"
    assert d["unit"] == "pattern-branch/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 1
    assert d["config"]["workload"] == "C1"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


import pytest  # noqa: E402


@pytest.mark.gpu
def test_device_arm_json_line():
    """The device arm on a small C2 sample: one JSON line with the keys the
    driver reads (value, e2e with copied bytes, roofline with the kernel's
    algorithmic bytes, cpu_baseline with its one-thread variant, launches,
    clocks)."""
    out = subprocess.run([sys.executable, "bench.py", "--config", "C2", "--sites", "3000", "--steps", "3",
                          "--warmup", "3", "--cpu-seconds", "1"], cwd=ROOT, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["metric"] == "pattern x branch gradient updates/s (full logL + grad eval)"
    assert d["unit"] == "pattern-branch/s" and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["dtype"] == "f64"
    assert d["config"]["workload"] == "C2"
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12 and r["algorithmic_bytes_per_launch"] > 0
    assert d["gpu_launches"] == 3 * 3  # K1, walk, K3 per evaluation
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["value"] > 0 and cb["single_thread"]["cores"] == 1
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
def test_other_workloads_block():
    """`--also` measures further configs in their own processes after the main
    line (the default C3 run carries C2 / C4 / C5): here C2 next to a C1 line,
    with its full-size parity fixture."""
    out = subprocess.run([sys.executable, "bench.py", "--config", "C1", "--steps", "3", "--warmup", "3",
                          "--no-cpu-baseline", "--also", "C2"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["config"]["workload"] == "C1"
    (o,) = d["other_workloads"]
    assert "error" not in o, o
    assert o["workload"] == "C2" and o["patterns"] == 20000 and o["steps"] == 3
    assert o["ms_per_step"] > 0 and o["value"] > 0 and o["e2e_value"] > 0 and o["gpu_launches"] == 9
    assert o["roofline"]["bound"] == "hbm" and 0 < o["roofline"]["frac"] < 1.2
    assert o["parity"]["fixture"] == "tests/golden/full_C2.npz" and o["parity"]["within_1e-9"] is True


def test_both_arms_share_config_and_parity_block(tmp_path, monkeypatch):
    """Identical `config` in both arms; the parity block compares against a
    full-size fixture only when the instance digest matches."""
    import numpy as np

    import bench
    from workloads import synth

    args = bench.parse_args(["--config", "C1"])
    inst = synth.generate("C1", seed=bench.SEED)
    cfg = bench.bench_config(args, inst)
    assert cfg["workload"] == "C1" and cfg["patterns"] == inst.patterns and cfg["sites"] == 1000
    # parity: fixture with this instance's digest
    g = np.linspace(-1.0, 1.0, inst.branches)
    fx = tmp_path / "tests" / "golden"
    fx.mkdir(parents=True)
    np.savez(fx / "full_C1.npz", digest=synth.instance_digest(inst), logL=-1234.5, gradient=g,
             rate_gradient=np.zeros(0), oracle_threads=8)
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    ok = bench.parity_block(args, inst, -1234.5 * (1 + 1e-12), g * (1 + 1e-11))
    assert ok["match"] and ok["within_1e-9"] and ok["logL_rel"] < 1e-11
    bad = bench.parity_block(args, inst, -1234.5, g + 1e-3)
    assert bad["match"] and not bad["within_1e-9"]
    other = synth.generate("C1", seed=bench.SEED + 1)
    assert bench.parity_block(args, other, -1.0, g)["match"] is False
