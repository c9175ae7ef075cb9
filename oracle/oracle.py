"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU parity oracle (oracle.cpp).

The oracle is a std-only C++ restatement of the reference's hot path
(/root/reference/proj/include/phylograd/{engine,substitution,tree,alignment,
validation}.hpp).  Only tests/, __graft_entry__.smoke() and bench.py's CPU
legs may import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liborc.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(os.path.join(_HERE, "oracle.cpp")):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _SO


class OracleError(Exception):
    pass


class OracleInvalidArgument(OracleError, ValueError):
    pass


class OracleLogicError(OracleError):
    pass


class OracleNewickError(OracleError):
    pass


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        _lib = C.CDLL(_SO)
        _declare(_lib)
    return _lib


P = C.c_void_p
I = C.c_int
D = C.c_double
U64 = C.c_uint64
PD = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
PI = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
PI64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def _declare(L):
    sig = {
        "orc_last_error": (C.c_char_p, []),
        "orc_rng_new": (P, [U64]),
        "orc_rng_free": (None, [P]),
        "orc_rng_next": (U64, [P]),
        "orc_rng_uniform": (D, [P, D, D]),
        "orc_tree_parse": (I, [C.c_char_p, C.POINTER(P)]),
        "orc_newick_error_position": (I, [C.c_char_p]),
        "orc_tree_from_arrays": (I, [I, PI, PI, PD, C.c_void_p, C.POINTER(P)]),
        "orc_tree_random": (I, [P, I, D, D, I, C.POINTER(P)]),
        "orc_tree_caterpillar": (I, [I, D, C.POINTER(P)]),
        "orc_tree_random_post_order": (I, [P, P, PI]),
        "orc_tree_free": (None, [P]),
        "orc_tree_tips": (I, [P]),
        "orc_tree_get": (I, [P, PI, PI, PD, PI, PI, PD]),
        "orc_tree_label": (I, [P, I, C.c_char_p, I]),
        "orc_tree_serialize": (I, [P, C.c_char_p, I]),
        "orc_tree_validate": (I, [I, PI, PI, PD, PI, C.c_void_p]),
        "orc_tree_assign_times": (I, [P, PD]),
        "orc_discrete_gamma": (I, [D, I, PD, PD]),
        "orc_gamma_quantile": (D, [D, D, D]),
        "orc_categories_check": (I, [I, PD, PD]),
        "orc_gtr": (I, [PD, PD, PD]),
        "orc_finish_generator": (None, [I, PD, PD]),
        "orc_model_new": (I, [I, PD, PD, I, C.POINTER(P)]),
        "orc_model_set_branch_generator": (I, [P, I, PD]),
        "orc_model_free": (None, [P]),
        "orc_model_has_eigen": (I, [P]),
        "orc_transition_matrix": (I, [P, I, D, D, PD]),
        "orc_expm": (I, [I, PD, PD]),
        "orc_aln_from_codes": (I, [I, C.c_long, PI, I, C.c_void_p, C.POINTER(P)]),
        "orc_aln_from_fasta": (I, [C.c_char_p, C.POINTER(P)]),
        "orc_aln_from_patterns": (I, [I, I, I, PI, I, C.c_void_p, PI64, C.c_void_p, C.POINTER(P)]),
        "orc_aln_free": (None, [P]),
        "orc_aln_patterns": (I, [P]),
        "orc_aln_taxa": (I, [P]),
        "orc_aln_states": (I, [P]),
        "orc_aln_weights": (None, [P, PI64]),
        "orc_aln_pattern_codes": (None, [P, PI]),
        "orc_aln_tip_partials": (None, [P, I, PD]),
        "orc_aln_pattern_column": (I, [P, I, C.c_char_p, I]),
        "orc_aln_taxon_name": (I, [P, I, C.c_char_p, I]),
        "orc_simulate_states": (I, [P, P, I, PD, PD, PD, C.c_long, U64, PI]),
        "orc_engine_new": (I, [P, P, P, I, PD, PD, D, I, I, I, C.POINTER(P)]),
        "orc_engine_free": (None, [P]),
        "orc_engine_set_branch_lengths": (I, [P, PD]),
        "orc_engine_invalidate": (None, [P]),
        "orc_engine_node_visits": (U64, [P]),
        "orc_engine_reset_node_visits": (None, [P]),
        "orc_engine_log_likelihood": (I, [P, C.POINTER(D)]),
        "orc_engine_post_order_pass": (I, [P]),
        "orc_engine_pre_order_pass": (I, [P, I]),
        "orc_engine_branch_gradient": (I, [P, I, C.POINTER(D), PD, PD]),
        "orc_engine_log_likelihood_at_node": (I, [P, I, C.POINTER(D)]),
        "orc_engine_gradient_abs": (I, [P, PD]),
        "orc_engine_post_partial": (I, [P, I, I, PD]),
        "orc_engine_pre_partial": (I, [P, I, I, PD]),
        "orc_engine_scalers": (I, [P, I, PD, PD]),
        "orc_engine_site_log_likelihoods": (I, [P, PD]),
        "orc_brute_force": (I, [P, P, P, I, PD, PD, PD, C.POINTER(D)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def _check(rc):
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == 1:
        raise OracleInvalidArgument(msg)
    if rc == 3:
        raise OracleLogicError(msg)
    if rc == 4:
        raise OracleNewickError(msg)
    raise OracleError(msg)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class Rng:
    """std::mt19937_64 shared with the oracle's random generators."""

    def __init__(self, seed: int):
        self.h = lib().orc_rng_new(seed)

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().orc_rng_free(self.h)
            except Exception:  # interpreter shutdown
                pass

    def next(self) -> int:
        return int(lib().orc_rng_next(self.h))

    def uniform(self, lo, hi) -> float:
        return float(lib().orc_rng_uniform(self.h, lo, hi))


class Tree:
    """Restated phylograd::Tree (tree.hpp:27-50)."""

    def __init__(self, handle):
        self.h = handle
        n = 2 * lib().orc_tree_tips(handle) - 1
        self.tip_count = n // 2 + 1
        self.parent = np.zeros(n + 1, np.int32)
        self.children = np.zeros((n + 1, 2), np.int32)
        self.branch_lengths = np.zeros(n - 1, np.float64)
        self.post_order = np.zeros(n, np.int32)
        self.pre_order = np.zeros(n, np.int32)
        times = np.zeros(n + 1, np.float64)
        has_t = lib().orc_tree_get(handle, self.parent, self.children, self.branch_lengths,
                                   self.post_order, self.pre_order, times)
        self.node_time = times if has_t else None
        buf = C.create_string_buffer(4096)
        self.labels = [""] * (n + 1)
        for i in range(1, n + 1):
            lib().orc_tree_label(handle, i, buf, 4096)
            self.labels[i] = buf.value.decode()

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().orc_tree_free(self.h)
            except Exception:  # interpreter shutdown
                pass

    @property
    def node_count(self):
        return 2 * self.tip_count - 1

    @property
    def root(self):
        return self.node_count

    @property
    def branch_count(self):
        return self.node_count - 1

    def is_tip(self, node):
        return 1 <= node <= self.tip_count

    def sibling(self, node):
        p = self.parent[node]
        c = self.children[p]
        return int(c[1] if c[0] == node else c[0])

    @staticmethod
    def parse(text: str) -> "Tree":
        h = P()
        _check(lib().orc_tree_parse(text.encode(), C.byref(h)))
        return Tree(h)

    @staticmethod
    def newick_error_position(text: str) -> int:
        return int(lib().orc_newick_error_position(text.encode()))

    @staticmethod
    def from_arrays(tip_count, parent, children, branch_lengths, post_order=None) -> "Tree":
        h = P()
        post = None if post_order is None else _i32(post_order)
        _check(lib().orc_tree_from_arrays(tip_count, _i32(parent), _i32(children).reshape(-1),
                                          _f64(branch_lengths),
                                          None if post is None else post.ctypes.data_as(C.c_void_p),
                                          C.byref(h)))
        t = Tree(h)
        t._post_keep = post
        return t

    @staticmethod
    def random(rng: Rng, tips, lo, hi) -> "Tree":
        """testutil.hpp:20-27 random_tree (coalescent topology, U(lo,hi) lengths)."""
        h = P()
        _check(lib().orc_tree_random(rng.h, tips, lo, hi, 0, C.byref(h)))
        return Tree(h)

    @staticmethod
    def coalescent(rng: Rng, tips, height_scale=0.5) -> "Tree":
        h = P()
        _check(lib().orc_tree_random(rng.h, tips, 0.0, height_scale, 1, C.byref(h)))
        return Tree(h)

    @staticmethod
    def caterpillar(tips, branch) -> "Tree":
        h = P()
        _check(lib().orc_tree_caterpillar(tips, branch, C.byref(h)))
        return Tree(h)

    def random_post_order(self, rng: Rng):
        out = np.zeros(self.node_count, np.int32)
        _check(lib().orc_tree_random_post_order(self.h, rng.h, out))
        return out

    def serialize(self) -> str:
        buf = C.create_string_buffer(1 << 20)
        lib().orc_tree_serialize(self.h, buf, 1 << 20)
        return buf.value.decode()

    def assign_times(self):
        times = np.zeros(self.node_count + 1)
        _check(lib().orc_tree_assign_times(self.h, times))
        self.node_time = times
        return times

    @staticmethod
    def validate(tip_count, parent, children, branch_lengths, post_order, node_time=None):
        t = None if node_time is None else _f64(node_time)
        _check(lib().orc_tree_validate(tip_count, _i32(parent), _i32(children).reshape(-1),
                                       _f64(branch_lengths), _i32(post_order),
                                       None if t is None else t.ctypes.data_as(C.c_void_p)))


def discrete_gamma(alpha, count):
    r = np.zeros(count)
    p = np.zeros(count)
    _check(lib().orc_discrete_gamma(alpha, count, r, p))
    return r, p


def gamma_quantile(shape, rate, p):
    return float(lib().orc_gamma_quantile(shape, rate, p))


def check_categories(rates, probs):
    _check(lib().orc_categories_check(len(rates), _f64(rates), _f64(probs)))


def gtr_generator(exch, freqs):
    q = np.zeros(16)
    _check(lib().orc_gtr(_f64(exch), _f64(freqs), q))
    return q.reshape(4, 4)


def finish_generator(q, pi):
    q = _f64(q).copy()
    m = q.shape[0]
    flat = q.reshape(-1).copy()
    lib().orc_finish_generator(m, flat, _f64(pi))
    return flat.reshape(m, m)


def expm(a):
    a = _f64(a)
    out = np.zeros(a.size)
    _check(lib().orc_expm(a.shape[0], a.reshape(-1), out))
    return out.reshape(a.shape)


class Model:
    """Restated phylograd::SubstitutionModel (substitution.hpp:77-219)."""

    def __init__(self, q, pi, reversible):
        q = _f64(q)
        self.m = q.shape[0]
        self.q = q.copy()
        self.pi = _f64(pi).copy()
        self.reversible = bool(reversible)
        self.branch_q = {}
        h = P()
        _check(lib().orc_model_new(self.m, q.reshape(-1), self.pi, int(reversible), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().orc_model_free(self.h)
            except Exception:  # interpreter shutdown
                pass

    @staticmethod
    def gtr(exch, freqs):
        return Model(gtr_generator(exch, freqs), freqs, True)

    @staticmethod
    def hky85(kappa, freqs):
        if not kappa > 0:
            raise OracleInvalidArgument("hky85: kappa must be positive")
        return Model.gtr([1.0, kappa, 1.0, 1.0, kappa, 1.0], freqs)

    @staticmethod
    def jc69():
        return Model.hky85(1.0, [0.25] * 4)

    def set_branch_generator(self, branch, q):
        q = _f64(q)
        _check(lib().orc_model_set_branch_generator(self.h, branch, q.reshape(-1)))
        self.branch_q[branch] = q.copy()

    def has_eigen(self):
        return bool(lib().orc_model_has_eigen(self.h))

    def transition_matrix(self, branch, b, c=1.0):
        out = np.zeros(self.m * self.m)
        _check(lib().orc_transition_matrix(self.h, branch, b, c, out))
        return out.reshape(self.m, self.m)


class Alignment:
    """Restated phylograd::SitePatternAlignment (alignment.hpp:129-238)."""

    def __init__(self, handle):
        self.h = handle
        self.pattern_count = lib().orc_aln_patterns(handle)
        self.taxon_count = lib().orc_aln_taxa(handle)
        self.state_count = lib().orc_aln_states(handle)
        self.weights = np.zeros(self.pattern_count, np.int64)
        lib().orc_aln_weights(handle, self.weights)
        buf = C.create_string_buffer(4096)
        self.taxa = []
        for r in range(self.taxon_count):
            lib().orc_aln_taxon_name(handle, r, buf, 4096)
            self.taxa.append(buf.value.decode())

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().orc_aln_free(self.h)
            except Exception:  # interpreter shutdown
                pass

    @staticmethod
    def from_codes(codes, m, labels=None) -> "Alignment":
        codes = _i32(codes)
        h = P()
        arr = None
        if labels is not None:
            arr = (C.c_char_p * len(labels))(*[s.encode() for s in labels])
        _check(lib().orc_aln_from_codes(codes.shape[0], codes.shape[1], codes.reshape(-1), m,
                                        None if arr is None else C.cast(arr, C.c_void_p), C.byref(h)))
        return Alignment(h)

    @staticmethod
    def from_fasta(text) -> "Alignment":
        h = P()
        _check(lib().orc_aln_from_fasta(text.encode(), C.byref(h)))
        return Alignment(h)

    @staticmethod
    def from_patterns(codes, m, weights, ambiguity=None, labels=None) -> "Alignment":
        """codes: ntax x P int (state, -1 missing, >= m ambiguity class)."""
        codes = _i32(codes)
        amb = np.zeros((0, m)) if ambiguity is None else _f64(ambiguity)
        h = P()
        arr = None
        if labels is not None:
            arr = (C.c_char_p * len(labels))(*[s.encode() for s in labels])
        _check(lib().orc_aln_from_patterns(codes.shape[0], codes.shape[1], m, codes.reshape(-1), amb.shape[0],
                                           amb.reshape(-1).ctypes.data_as(C.c_void_p),
                                           np.ascontiguousarray(weights, np.int64),
                                           None if arr is None else C.cast(arr, C.c_void_p), C.byref(h)))
        a = Alignment(h)
        a._keep = amb
        return a

    def pattern_codes(self):
        out = np.zeros(self.taxon_count * self.pattern_count, np.int32)
        lib().orc_aln_pattern_codes(self.h, out)
        return out.reshape(self.taxon_count, self.pattern_count)

    def tip_partials(self, taxon):
        out = np.zeros(self.state_count * self.pattern_count)
        lib().orc_aln_tip_partials(self.h, taxon, out)
        return out.reshape(self.pattern_count, self.state_count).T

    def pattern_column(self, p):
        buf = C.create_string_buffer(1 << 16)
        lib().orc_aln_pattern_column(self.h, p, buf, 1 << 16)
        return buf.value.decode()

    def taxon_index(self, name):
        return self.taxa.index(name) if name in self.taxa else -1


def simulate_states(tree: Tree, model: Model, rates, probs, branch_lengths, sites, seed):
    """alignment.hpp:243-286, draw-for-draw (std::mt19937_64, libstdc++)."""
    out = np.zeros(tree.tip_count * sites, np.int32)
    _check(lib().orc_simulate_states(tree.h, model.h, len(rates), _f64(rates), _f64(probs),
                                     _f64(branch_lengths), sites, seed, out))
    return out.reshape(tree.tip_count, sites)


class Engine:
    """Restated phylograd::LikelihoodEngine (engine.hpp:47-438).

    ``blocks`` > 1 splits the patterns into contiguous blocks evaluated on
    std::threads with a fixed-order reduction."""

    def __init__(self, tree: Tree, aln: Alignment, model: Model, rates=(1.0,), probs=(1.0,),
                 threshold=1e-150, force_rescaling=False, disable_rescaling=False, blocks=1):
        self.tree, self.aln, self.model = tree, aln, model
        self.rates, self.probs = _f64(rates), _f64(probs)
        h = P()
        _check(lib().orc_engine_new(tree.h, aln.h, model.h, len(self.rates), self.rates, self.probs, threshold,
                                    int(force_rescaling), int(disable_rescaling), blocks, C.byref(h)))
        self.h = h
        self.B = tree.branch_count
        self._blen = tree.branch_lengths.copy()

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().orc_engine_free(self.h)
            except Exception:  # interpreter shutdown
                pass

    @property
    def branch_lengths(self):
        return self._blen.copy()

    def set_branch_lengths(self, b):
        b = _f64(b)
        _check(lib().orc_engine_set_branch_lengths(self.h, b))
        self._blen = b.copy()

    def invalidate_caches(self):
        lib().orc_engine_invalidate(self.h)

    def node_visits(self):
        return int(lib().orc_engine_node_visits(self.h))

    def reset_node_visits(self):
        lib().orc_engine_reset_node_visits(self.h)

    def log_likelihood(self):
        v = D()
        _check(lib().orc_engine_log_likelihood(self.h, C.byref(v)))
        return v.value

    def post_order_pass(self):
        _check(lib().orc_engine_post_order_pass(self.h))

    def pre_order_pass(self, hess=False):
        _check(lib().orc_engine_pre_order_pass(self.h, int(hess)))

    def branch_gradient(self, with_hessian=False):
        ll = D()
        g = np.zeros(self.B)
        h = np.zeros(self.B)
        _check(lib().orc_engine_branch_gradient(self.h, int(with_hessian), C.byref(ll), g, h))
        return ll.value, g, (h if with_hessian else None)

    def gradient_condition(self):
        """Per branch of the last gradient pass, the gradient sum with every
        product of each per-pattern term taken in absolute value (sum_s w_s
        sum_l c_l w_l sum_i |q_i| sum_j |Q_ij e_j| / L_s): the scale against
        which a component whose terms cancel -- inside Q e or across
        patterns -- is judged (SURVEY.md §8d condition-aware parity)."""
        out = np.zeros(self.B)
        _check(lib().orc_engine_gradient_abs(self.h, out))
        return out

    def log_likelihood_at_node(self, node):
        v = D()
        _check(lib().orc_engine_log_likelihood_at_node(self.h, node, C.byref(v)))
        return v.value

    def post_partial(self, node, l):
        out = np.zeros(self.model.m * self.aln.pattern_count)
        _check(lib().orc_engine_post_partial(self.h, node, l, out))
        return out.reshape(self.aln.pattern_count, self.model.m).T

    def pre_partial(self, node, l):
        out = np.zeros(self.model.m * self.aln.pattern_count)
        _check(lib().orc_engine_pre_partial(self.h, node, l, out))
        return out.reshape(self.aln.pattern_count, self.model.m).T

    def scalers(self, node):
        a = np.zeros(self.aln.pattern_count)
        b = np.zeros(self.aln.pattern_count)
        _check(lib().orc_engine_scalers(self.h, node, a, b))
        return a, b

    def site_log_likelihoods(self):
        out = np.zeros(self.aln.pattern_count)
        _check(lib().orc_engine_site_log_likelihoods(self.h, out))
        return out


def brute_force_log_likelihood(tree, aln, model, rates, probs, branch_lengths):
    v = D()
    _check(lib().orc_brute_force(tree.h, aln.h, model.h, len(rates), _f64(rates), _f64(probs),
                                 _f64(branch_lengths), C.byref(v)))
    return v.value


def fd_branch_gradient(engine: Engine, h=1e-5):
    """validation.hpp:124-137: central differences in log space, divided back."""
    saved = engine.branch_lengths
    if np.any(saved <= 0):
        raise OracleInvalidArgument("fd gradient: log-space differencing needs positive lengths")
    x = np.log(saved)
    g = np.zeros_like(x)
    for i in range(len(x)):
        xp = x.copy(); xp[i] += h
        xm = x.copy(); xm[i] -= h
        engine.set_branch_lengths(np.exp(xp)); up = engine.log_likelihood()
        engine.set_branch_lengths(np.exp(xm)); dn = engine.log_likelihood()
        g[i] = (up - dn) / (2 * h)
    engine.set_branch_lengths(saved)
    return g / saved


def fd_branch_hessian_diagonal(engine: Engine, h=1e-4):
    """validation.hpp:139-148."""
    saved = engine.branch_lengths
    c = engine.log_likelihood()
    d = np.zeros_like(saved)
    for i in range(len(saved)):
        xp = saved.copy(); xp[i] += h
        xm = saved.copy(); xm[i] -= h
        engine.set_branch_lengths(xp); up = engine.log_likelihood()
        engine.set_branch_lengths(xm); dn = engine.log_likelihood()
        d[i] = (up - 2 * c + dn) / (h * h)
    engine.set_branch_lengths(saved)
    return d
