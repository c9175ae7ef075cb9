"""Seeded synthetic workloads for the BASELINE.json configs.

The paper's WNV/LASV/DENV alignments are not available; these generators
produce inputs with the configs' shapes and value distributions: Yule trees
numbered like parse_newick, model parameters drawn as the config states,
forward simulation down the tree (alignment.hpp:243-286), optional gaps, then
first-occurrence pattern compression.  C1 and C2 are simulated in the
reference's own draw order (one mt19937_64 stream, so the reference's
simulate_states regenerates their columns); C3-C5 (10^5..10^6 columns) use a
counter-based per-site stream (pg_simulate.hpp) so they simulate in parallel:
on every host core here, or on the GPU with the product's
pg_simulate_states_gpu (`generate(..., device=d)`), with identical columns.

Input generation only — never inside a timed region.  The native code is
workloads/_build/libpg_workloads.so, a host library separate from the product
(libphylograd_b200.so), so the CPU reference arm of bench.py builds the same
inputs without mapping any product code.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

import os

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "_build", "libpg_workloads.so")
SIM_BLOCKED, SIM_REFERENCE, SIM_COUNTER, SIM_NONE = 0, 1, 2, 3


class Spec(C.Structure):
    _fields_ = [
        ("tips", C.c_int),
        ("model_kind", C.c_int),
        ("categories", C.c_int),
        ("gamma_alpha", C.c_double),
        ("sites", C.c_int64),
        ("branch_mean", C.c_double),
        ("clock", C.c_int),
        ("dt_mean", C.c_double),
        ("rate_scale", C.c_double),
        ("rate_sd", C.c_double),
        ("gap_fraction", C.c_double),
        ("seed", C.c_uint64),
        ("threads", C.c_int),
        ("sim", C.c_int),
    ]


_lib = None
_P, _I, _D = C.c_void_p, C.c_int, C.c_double
_PD, _PI32, _PI64, _PI8 = C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_int8)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(f"workloads: {SO_PATH} is not built; run __graft_entry__.build()")
        L = C.CDLL(SO_PATH)
        for name, (res, args) in {
            "pgw_last_error": (C.c_char_p, []),
            "pgw_create": (_I, [C.POINTER(Spec), C.POINTER(_P), C.POINTER(_I), C.POINTER(_I)]),
            "pgw_tree": (_I, [_P, _PI32, _PI32, _PI32, _PD, _PD, _PD]),
            "pgw_model": (_I, [_P, _PD, _PD, C.POINTER(_I), _PD, _PD]),
            "pgw_patterns": (_I, [_P, _PI8, _PI64]),
            "pgw_free": (None, [_P]),
            "pgw_simulate_states": (_I, [_I, _PI32, _PI32, _I, _PD, _PD, _I, _I, _PD, _PD, _PD, C.c_int64,
                                         C.c_uint64, _PI8]),
            "pgw_simulate_states_counter": (_I, [_I, _PI32, _PI32, _I, _PD, _PD, _I, _I, _PD, _PD, _PD, C.c_int64,
                                                 C.c_uint64, _D, _I, _PI8]),
        }.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    if rc != 0:
        raise ValueError(lib().pgw_last_error().decode(errors="replace"))


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))

# name -> (tips, model_kind, categories, alpha, sites, branch_mean, clock, dt_mean, rate_scale, rate_sd, gaps)
CONFIGS = {
    "C1": dict(tips=64, model_kind=0, categories=1, gamma_alpha=1.0, sites=1000, branch_mean=0.02,
               sim=SIM_REFERENCE),
    "C2": dict(tips=512, model_kind=1, categories=4, gamma_alpha=0.5, sites=20000, branch_mean=0.01,
               gap_fraction=0.02, sim=SIM_REFERENCE),
    "C3": dict(tips=2048, model_kind=2, categories=4, gamma_alpha=0.5, sites=1000000, clock=1, dt_mean=5.0,
               rate_scale=1e-3, rate_sd=0.3, sim=SIM_COUNTER),
    "C4": dict(tips=1000, model_kind=3, categories=4, gamma_alpha=0.5, sites=200000, branch_mean=0.05,
               sim=SIM_COUNTER),
    "C5": dict(tips=256, model_kind=4, categories=4, gamma_alpha=0.5, sites=400000, branch_mean=0.1,
               sim=SIM_COUNTER),
}
DESCRIPTIONS = {
    "C1": "HKY85 k=2 pi=(.3,.2,.2,.3), L=1, Yule-64, b~Exp(0.02), 1000 columns",
    "C2": "GTR+G4(0.5), Yule-512, b~Exp(0.01), 20000 columns, 2% gaps",
    "C3": "non-reversible 4-state+G4(0.5), Yule-2048, clock rates 1e-3*exp(N(0,.3^2)) x dt~Exp(5), 1e6 columns",
    "C4": "AA-20 reversible+G4(0.5), Yule-1000, b~Exp(0.05), 2e5 columns",
    "C5": "GY94 codon (w=.3,k=2)+G4(0.5), Yule-256, b~Exp(0.1), 4e5 columns",
}


@dataclass
class Instance:
    name: str
    tip_count: int
    parent: np.ndarray       # [2N]
    children: np.ndarray     # [2N, 2]
    post_order: np.ndarray   # [2N-1]
    branch_lengths: np.ndarray  # [2N-2]
    durations: np.ndarray    # [2N-2] (zeros unless clock)
    branch_rates: np.ndarray  # [2N-2] (zeros unless clock)
    q: np.ndarray
    pi: np.ndarray
    reversible: bool
    cat_rates: np.ndarray
    cat_probs: np.ndarray
    codes: np.ndarray        # [N, P] int8, -1 missing
    weights: np.ndarray      # [P] int64
    clock: bool = False

    @property
    def states(self):
        return int(self.q.shape[0])

    @property
    def patterns(self):
        return int(self.weights.shape[0])

    @property
    def branches(self):
        return 2 * self.tip_count - 2

    def labels(self):
        return [""] + [f"t{i}" for i in range(1, self.tip_count + 1)] + [""] * (self.tip_count - 1)

    def save(self, path):
        """Uncompressed .npz (fast to share between the ranks of one node)."""
        import dataclasses
        np.savez(path, **{k: np.asarray(v) for k, v in dataclasses.asdict(self).items()})

    @staticmethod
    def load(path) -> "Instance":
        z = np.load(path, allow_pickle=False)
        return Instance(str(z["name"]), int(z["tip_count"]), z["parent"], z["children"], z["post_order"],
                        z["branch_lengths"], z["durations"], z["branch_rates"], z["q"], z["pi"],
                        bool(z["reversible"]), z["cat_rates"], z["cat_probs"], z["codes"], z["weights"],
                        bool(z["clock"]))

    def slice_patterns(self, p0, p1) -> "Instance":
        import dataclasses
        return dataclasses.replace(self, codes=np.ascontiguousarray(self.codes[:, p0:p1]),
                                   weights=np.ascontiguousarray(self.weights[p0:p1]))


def generate(name: str, seed: int = 12146, sites: int | None = None, tips: int | None = None,
             threads: int = 0, sim: int | None = None, device: int | None = None) -> Instance:
    """A seeded BASELINE.json workload.  device: simulate and compress the
    columns on that GPU (counter-stream configs only; loads the product
    library) -- the same Instance as the host path."""
    cfg = dict(CONFIGS[name])
    spec = Spec()
    spec.tips = tips or cfg["tips"]
    spec.model_kind = cfg["model_kind"]
    spec.categories = cfg["categories"]
    spec.gamma_alpha = cfg.get("gamma_alpha", 1.0)
    spec.sites = sites or cfg["sites"]
    spec.branch_mean = cfg.get("branch_mean", 0.01)
    spec.clock = cfg.get("clock", 0)
    spec.dt_mean = cfg.get("dt_mean", 1.0)
    spec.rate_scale = cfg.get("rate_scale", 1.0)
    spec.rate_sd = cfg.get("rate_sd", 0.0)
    spec.gap_fraction = cfg.get("gap_fraction", 0.0)
    spec.seed = seed
    spec.threads = threads
    spec.sim = cfg.get("sim", SIM_BLOCKED) if sim is None else sim
    on_gpu = device is not None and spec.sim == SIM_COUNTER
    if on_gpu:
        spec.sim = SIM_NONE
    L = lib()
    h = C.c_void_p()
    P = C.c_int()
    m = C.c_int()
    check(L.pgw_create(C.byref(spec), C.byref(h), C.byref(P), C.byref(m)))
    try:
        N = spec.tips
        n = 2 * N - 1
        parent = np.zeros(n + 1, np.int32)
        children = np.zeros(2 * (n + 1), np.int32)
        post = np.zeros(n, np.int32)
        blen = np.zeros(n - 1)
        dt = np.zeros(n - 1)
        rr = np.zeros(n - 1)
        check(L.pgw_tree(h, ptr(parent, C.c_int32), ptr(children, C.c_int32), ptr(post, C.c_int32),
                              ptr(blen, C.c_double), ptr(dt, C.c_double), ptr(rr, C.c_double)))
        mm = m.value
        q = np.zeros(mm * mm)
        pi = np.zeros(mm)
        rev = C.c_int()
        cr = np.zeros(spec.categories)
        cp = np.zeros(spec.categories)
        check(L.pgw_model(h, ptr(q, C.c_double), ptr(pi, C.c_double), C.byref(rev), ptr(cr, C.c_double),
                               ptr(cp, C.c_double)))
        if on_gpu:
            codes, w = _columns_on_gpu(N, parent, post, q.reshape(mm, mm), pi, rev.value, cr, cp, blen, spec.sites,
                                       seed, spec.gap_fraction, device)
        else:
            codes = np.zeros((N, P.value), np.int8)
            w = np.zeros(P.value, np.int64)
            check(L.pgw_patterns(h, ptr(codes, C.c_int8), ptr(w, C.c_int64)))
    finally:
        L.pgw_free(h)
    return Instance(name, N, parent, children.reshape(n + 1, 2), post, blen, dt, rr, q.reshape(mm, mm), pi,
                    bool(rev.value), cr, cp, codes, w, bool(spec.clock))


def instance_digest(inst: Instance) -> str:
    """sha256 over every input array of an evaluation (tree, patterns, model,
    categories, lengths, durations): equal digests mean identical inputs.
    Full-size parity fixtures (tests/golden/full_*.npz) record it."""
    import hashlib

    h = hashlib.sha256()
    for a in (inst.parent, inst.children, inst.post_order, inst.branch_lengths, inst.durations, inst.q, inst.pi,
              inst.cat_rates, inst.cat_probs, inst.codes, inst.weights):
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def tips_of(cfg) -> int:
    return int(cfg["tips"])


def generate_shared(name: str, rank: int, world: int, barrier, tag: str, seed: int = 12146,
                    sites: int | None = None, device: int | None = None) -> Instance:
    """One rank of a node simulates the workload with every host core and
    shares it through node-local shared memory; the other ranks load it
    (identical input everywhere; each rank then keeps its pattern shard).
    `barrier` is a callable synchronising all ranks (e.g. dist.barrier)."""
    import os

    if world <= 1:
        return generate(name, seed=seed, sites=sites, threads=os.cpu_count() or 1, device=device)
    # node-local shared memory when it has room for the codes (N x sites
    # bytes plus the small arrays), else /tmp
    cfg = CONFIGS[name]
    need = 2 * (tips_of(cfg) * (sites or cfg["sites"])) + (64 << 20)
    shm = "/tmp"
    if os.path.isdir("/dev/shm"):
        st = os.statvfs("/dev/shm")
        if st.f_bavail * st.f_frsize > need:
            shm = "/dev/shm"
    path = os.path.join(shm, f"pg_synth_{name}_{seed}_{sites or 0}_{tag}.npz")
    if rank == 0:
        generate(name, seed=seed, sites=sites, threads=os.cpu_count() or 1, device=device).save(path)
    barrier()
    inst = Instance.load(path)
    barrier()
    if rank == 0:
        os.remove(path)
    return inst


def _columns_on_gpu(N, parent, post, q, pi, reversible, cat_rates, cat_probs, blen, sites, seed, gap, device):
    """pg_simulate_states_gpu into device memory, then pg_compress_codes_gpu
    on the device-resident columns: (pattern codes [N][P] int8, weights)."""
    import torch

    from paper_1905_12146_b200 import _lib as PL

    L = PL.lib()
    m = int(q.shape[0])
    cols = torch.empty((N, sites), dtype=torch.int8, device=f"cuda:{device}")
    f = C.c_float()
    qq = np.ascontiguousarray(q, np.float64)
    PL.check(L.pg_simulate_states_gpu(N, ptr(np.ascontiguousarray(parent, np.int32), C.c_int32),
                                      ptr(np.ascontiguousarray(post, np.int32), C.c_int32), m, ptr(qq, C.c_double),
                                      ptr(np.ascontiguousarray(pi, np.float64), C.c_double), int(reversible),
                                      len(cat_rates), ptr(np.ascontiguousarray(cat_rates, np.float64), C.c_double),
                                      ptr(np.ascontiguousarray(cat_probs, np.float64), C.c_double),
                                      ptr(np.ascontiguousarray(blen, np.float64), C.c_double), sites, seed, gap, device,
                                      cols.data_ptr(), 1, C.byref(f)))
    h = C.c_void_p()
    P = C.c_int()
    PL.check(L.pg_compress_codes_gpu(N, sites, cols.data_ptr(), 1, m, device, C.byref(h), C.byref(P)))
    try:
        codes = np.zeros((N, P.value), np.int8)
        w = np.zeros(P.value, np.int64)
        PL.check(L.pg_compress_result_gpu(h, codes.ctypes.data_as(C.c_void_p), ptr(w, C.c_int64), None, None))
    finally:
        L.pg_compress_free_gpu(h)
    del cols
    return codes, w


def simulate_states_counter(tip_count, parent, post_order, q, pi, reversible, cat_rates, cat_probs, branch_lengths,
                            sites, seed, gap=0.0, threads=0):
    """The counter-based per-site simulation (host twin of
    pg_simulate_states_gpu): tip states [tip_count][sites] int8, -1 gap."""
    m = int(np.asarray(q).shape[0])
    out = np.zeros((tip_count, sites), np.int8)
    q = np.ascontiguousarray(q, np.float64)
    pi = np.ascontiguousarray(pi, np.float64)
    cr = np.ascontiguousarray(cat_rates, np.float64)
    cp = np.ascontiguousarray(cat_probs, np.float64)
    b = np.ascontiguousarray(branch_lengths, np.float64)
    par = np.ascontiguousarray(parent, np.int32)
    post = np.ascontiguousarray(post_order, np.int32)
    check(lib().pgw_simulate_states_counter(tip_count, ptr(par, C.c_int32), ptr(post, C.c_int32), m,
                                            ptr(q, C.c_double), ptr(pi, C.c_double), int(bool(reversible)), len(cr),
                                            ptr(cr, C.c_double), ptr(cp, C.c_double), ptr(b, C.c_double), sites, seed,
                                            float(gap), threads, ptr(out, C.c_int8)))
    return out


def simulate_states(tip_count, parent, post_order, q, pi, reversible, cat_rates, cat_probs, branch_lengths,
                    sites, seed):
    """alignment.hpp:243-286 in the reference's draw order (one
    mt19937_64(seed) stream): tip states [tip_count][sites] int8."""
    m = int(np.asarray(q).shape[0])
    out = np.zeros((tip_count, sites), np.int8)
    q = np.ascontiguousarray(q, np.float64)
    pi = np.ascontiguousarray(pi, np.float64)
    cr = np.ascontiguousarray(cat_rates, np.float64)
    cp = np.ascontiguousarray(cat_probs, np.float64)
    b = np.ascontiguousarray(branch_lengths, np.float64)
    par = np.ascontiguousarray(parent, np.int32)
    post = np.ascontiguousarray(post_order, np.int32)
    check(lib().pgw_simulate_states(tip_count, ptr(par, C.c_int32), ptr(post, C.c_int32), m, ptr(q, C.c_double),
                                    ptr(pi, C.c_double), int(bool(reversible)), len(cr), ptr(cr, C.c_double),
                                    ptr(cp, C.c_double), ptr(b, C.c_double), sites, seed, ptr(out, C.c_int8)))
    return out


def api_objects(inst: Instance):
    """The product API's setup objects (Tree, SitePatternAlignment,
    SubstitutionModel, RateCategories) for an Instance (tips bound in order)."""
    from paper_1905_12146_b200.api import RateCategories, SitePatternAlignment, SubstitutionModel, Tree

    labels = inst.labels()
    tree = Tree(inst.tip_count, inst.parent, inst.children,
                np.concatenate([[0.0], inst.branch_lengths, [0.0]]), labels, inst.post_order)
    aln = SitePatternAlignment(labels[1:inst.tip_count + 1], inst.states, inst.codes, inst.weights)
    model = SubstitutionModel(inst.q, inst.pi, inst.reversible)
    cats = RateCategories(inst.cat_rates, inst.cat_probs)
    return tree, aln, model, cats


def engine_for(inst: Instance, options=None):
    """Builds a LikelihoodEngine over an Instance (tips bound in order)."""
    from paper_1905_12146_b200.api import LikelihoodEngine

    eng = LikelihoodEngine(*api_objects(inst), options)
    if inst.clock:
        eng.set_clock_durations(inst.durations)
    return eng
