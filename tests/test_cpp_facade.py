"""The C++ drop-in facade (include/phylograd_b200/engine.hpp): compiles against
the C-ABI library on CPU; runs the reference call pattern on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_facade_test(tmpdir):
    exe = os.path.join(str(tmpdir), "facade_test")
    libdir = os.path.join(ROOT, "paper_1905_12146_b200", "_build")
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "facade_test.cpp"), "-L", libdir, "-lphylograd_b200",
                           f"-Wl,-rpath,{libdir}", "-o", exe])
    return exe


def test_facade_compiles(tmp_path):
    assert os.path.exists(build_facade_test(tmp_path))


@pytest.mark.gpu
def test_facade_runs_reference_call_pattern(tmp_path):
    exe = build_facade_test(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout


def build_config_exe(tmpdir):
    exe = os.path.join(str(tmpdir), "facade_config")
    libdir = os.path.join(ROOT, "paper_1905_12146_b200", "_build")
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "facade_config.cpp"), "-L", libdir, "-lphylograd_b200",
                           f"-Wl,-rpath,{libdir}", "-o", exe])
    return exe


def write_instance(path, inst):
    import numpy as np

    N, m, L, P = inst.tip_count, inst.states, len(inst.cat_rates), inst.patterns
    with open(path, "wb") as f:
        np.array([N, m, L, P, int(inst.reversible), int(inst.clock)], np.int32).tofile(f)
        np.ascontiguousarray(inst.parent, np.int32).tofile(f)
        np.ascontiguousarray(inst.children, np.int32).reshape(-1).tofile(f)
        np.ascontiguousarray(inst.post_order, np.int32).tofile(f)
        for a in (inst.branch_lengths, inst.q.reshape(-1), inst.pi, inst.cat_rates, inst.cat_probs):
            np.ascontiguousarray(a, np.float64).tofile(f)
        np.ascontiguousarray(inst.codes, np.int8).tofile(f)
        np.ascontiguousarray(inst.weights, np.int64).tofile(f)
        if inst.clock:
            np.ascontiguousarray(inst.durations, np.float64).tofile(f)


def read_result(path, inst):
    import numpy as np

    B, N = inst.branches, inst.tip_count
    d = np.fromfile(path, np.float64, count=1 + B + ((1 + B + N - 1) if inst.clock else 0))
    shards = int(np.fromfile(path, np.int32, offset=8 * d.size)[0])
    out = {"logL": d[0], "g": d[1:1 + B], "shards": shards}
    if inst.clock:
        out.update(dlog_mu=d[1 + B], dlog_eps=d[2 + B:2 + 2 * B], node_time=d[2 + 2 * B:])
    return out


def test_facade_config_compiles(tmp_path):
    assert os.path.exists(build_config_exe(tmp_path))


@pytest.mark.gpu
@pytest.mark.parametrize("name,sites,devargs,shards", [
    ("C2", None, [], 1),                       # full C2 (512 taxa, 2 % gaps), one device
    ("C2", None, ["--devices", "0"], 1),       # NCCL group of one device (ncclCommInitAll)
    ("C2", None, ["--devices", "0,0", "--fixed"], 2),  # two shards, fixed rank-order reduction
    ("C3", 20000, [], 1),                      # 2,048 taxa, non-reversible, clock chain rule
    ("C3", 20000, ["--devices", "0,0,0", "--fixed"], 3),
])
def test_facade_config_scale_matches_oracle(tmp_path, name, sites, devargs, shards):
    """The reference call pattern at config scale through the C++ drop-in
    (no Python on the evaluation path), single device and sharded, against
    the CPU oracle within the north star's 1e-9."""
    import numpy as np

    from tests.helpers import assert_logl, assert_vec, oracle_for
    from workloads import synth

    exe = build_config_exe(tmp_path)
    inst = synth.generate(name, seed=12146, sites=sites)
    inp, out = os.path.join(str(tmp_path), "in.bin"), os.path.join(str(tmp_path), "out.bin")
    write_instance(inp, inst)
    r = subprocess.run([exe, inp, out] + devargs, capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    res = read_result(out, inst)
    assert res["shards"] == shards
    ref = oracle_for(inst, blocks=os.cpu_count() or 1)
    ll, g, _ = ref.branch_gradient(False)
    assert_logl(res["logL"], ll)
    assert_vec(res["g"], g)
    if inst.clock:
        b = inst.branch_lengths
        assert_vec(res["dlog_eps"], b * g, what="d logL / d log eps")
        assert res["dlog_mu"] == pytest.approx(float(np.sum(b * g)), rel=1e-9, abs=1e-12 * np.abs(b * g).sum())
        r_ = inst.branch_rates
        want = np.zeros(inst.tip_count - 1)
        for k in range(inst.tip_count - 1):
            node = inst.tip_count + 1 + k
            v = r_[node - 1] * g[node - 1] if node != 2 * inst.tip_count - 1 else 0.0
            for c in inst.children[node]:
                v -= r_[c - 1] * g[c - 1]
            want[k] = v
        assert_vec(res["node_time"], want, what="node-time gradient")


def build_adapter_exe(tmpdir):
    exe = os.path.join(str(tmpdir), "adapter_test")
    libdir = os.path.join(ROOT, "paper_1905_12146_b200", "_build")
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "adapter_test.cpp"), "-L", libdir, "-lphylograd_b200",
                           f"-Wl,-rpath,{libdir}", "-o", exe])
    return exe


def test_reference_adapter_compiles(tmp_path):
    """include/phylograd_b200/reference_adapter.hpp against stand-ins with the
    reference types' member names (no Eigen in this image)."""
    assert os.path.exists(build_adapter_exe(tmp_path))


@pytest.mark.gpu
def test_reference_adapter_runs_full_c2(tmp_path):
    """make_engine(tree, alignment, model, categories) over reference-shaped
    objects (dense tip partials, taxa in a different order than the tips) at
    full C2 size equals the oracle."""
    from tests.helpers import assert_logl, assert_vec, oracle_for
    from workloads import synth

    exe = build_adapter_exe(tmp_path)
    inst = synth.generate("C2", seed=12146)
    inp, out = os.path.join(str(tmp_path), "in.bin"), os.path.join(str(tmp_path), "out.bin")
    write_instance(inp, inst)
    r = subprocess.run([exe, inp, out], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    import numpy as np

    d = np.fromfile(out, np.float64, count=1 + inst.branches)
    ll, g, _ = oracle_for(inst, blocks=os.cpu_count() or 1).branch_gradient(False)
    assert_logl(d[0], ll)
    assert_vec(d[1:], g)
