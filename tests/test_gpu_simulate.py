"""The setup path at scale on the GPU: forward
simulation (pg_simulate_states_gpu, alignment.hpp:243-286 semantics with the
counter-based per-site stream) bit-identical with its host twin
(workloads/, PGW_SIM_COUNTER), and the whole generate-on-GPU path (simulate +
pg_compress_codes_gpu) giving the identical Instance."""
import time

import numpy as np
import pytest

from workloads import synth

pytestmark = pytest.mark.gpu


def _gpu_columns(inst, sites, seed, gap=0.0):
    import ctypes as C

    from paper_1905_12146_b200 import _lib as PL

    out = np.zeros((inst.tip_count, sites), np.int8)
    ms = C.c_float()
    f = lambda a, t=np.float64: np.ascontiguousarray(a, t)  # noqa: E731
    PL.check(PL.lib().pg_simulate_states_gpu(
        inst.tip_count, PL.ptr(f(inst.parent, np.int32), C.c_int32), PL.ptr(f(inst.post_order, np.int32), C.c_int32),
        inst.states, PL.ptr(f(inst.q), C.c_double), PL.ptr(f(inst.pi), C.c_double), int(inst.reversible),
        len(inst.cat_rates), PL.ptr(f(inst.cat_rates), C.c_double), PL.ptr(f(inst.cat_probs), C.c_double),
        PL.ptr(f(inst.branch_lengths), C.c_double), sites, seed, gap, 0, out.ctypes.data_as(C.c_void_p), 0,
        C.byref(ms)))
    return out, ms.value


@pytest.mark.parametrize("name,tips,sites,gap", [("C2", 64, 5000, 0.02), ("C3", 100, 4000, 0.0),
                                                 ("C4", 50, 3000, 0.01), ("C5", 24, 2000, 0.0)])
def test_gpu_simulation_matches_host_twin(name, tips, sites, gap):
    inst = synth.generate(name, seed=5, sites=50, tips=tips)
    gpu, _ = _gpu_columns(inst, sites, 77, gap)
    host = synth.simulate_states_counter(inst.tip_count, inst.parent, inst.post_order, inst.q, inst.pi,
                                         inst.reversible, inst.cat_rates, inst.cat_probs, inst.branch_lengths, sites,
                                         77, gap=gap)
    assert np.array_equal(gpu, host)


@pytest.mark.parametrize("name,sites", [("C3", 60000), ("C5", 8000)])
def test_generate_on_gpu_is_the_same_instance(name, sites):
    a = synth.generate(name, seed=12146, sites=sites)
    b = synth.generate(name, seed=12146, sites=sites, device=0)
    assert synth.instance_digest(a) == synth.instance_digest(b)


def test_full_c3_columns_on_gpu_timed():
    """The C3 bench shape (2,048 taxa x 10^6 columns) simulated and compressed
    on the device: identical to the host path (digest), and timed."""
    t0 = time.perf_counter()
    gpu = synth.generate("C3", seed=12146, device=0)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    host = synth.generate("C3", seed=12146)
    t_host = time.perf_counter() - t0
    inst = gpu
    _, ms = _gpu_columns(inst, 200000, 12146)
    print(f"C3 generate: GPU path {t_gpu:.2f} s, host path {t_host:.2f} s; simulation kernel "
          f"{ms * 5:.1f} ms per 10^6 columns (from 2e5)")
    assert synth.instance_digest(gpu) == synth.instance_digest(host)
