"""Python mirror of the reference's C++ API for the logL + gradient path.

Names, argument meaning and error behaviour follow phylograd
(/root/reference/proj/include/phylograd): ``Tree``/``parse_newick``
(tree.hpp:27-289), ``SitePatternAlignment`` (alignment.hpp:129-238),
``SubstitutionModel`` (substitution.hpp:77-219), ``RateCategories`` /
``discrete_gamma_categories`` (substitution.hpp:23-68), ``EngineOptions`` /
``GradientReport`` / ``LikelihoodEngine`` (engine.hpp:33-438) and the clock
chain rule (clock.hpp:42-55, :140-213).  All arithmetic on the hot path runs in
the sm_100a kernels behind the C-ABI (``_lib``); nothing here computes a
likelihood on the CPU.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _lib as _L
from ._lib import InvalidArgument, LogicError, NewickError, PgError, RuntimeFailure, check, f64, i32, lib, ptr


# ----------------------------------------------------------------------- tree
class Tree:
    """Rooted binary tree with the reference's numbering (tree.hpp:27-50):
    tips 1..N, internal nodes N+1..2N-1, root 2N-1; per-node arrays have
    node_count()+1 entries (slot 0 unused)."""

    def __init__(self, tip_count: int, parent, children, branch_length, labels=None, post_order=None,
                 node_time=None):
        self.tip_count = int(tip_count)
        n = self.node_count()
        self.parent = np.asarray(parent, dtype=np.int32).copy()
        self.children = np.asarray(children, dtype=np.int32).reshape(n + 1, 2).copy()
        self.branch_length = np.asarray(branch_length, dtype=np.float64).copy()
        if self.branch_length.shape[0] != n + 1:
            raise InvalidArgument("tree vectors not sized node_count()+1")
        self.labels = list(labels) if labels is not None else [""] + [f"t{i}" for i in range(1, self.tip_count + 1)] + [
            ""] * (n - self.tip_count)
        self.node_time = None if node_time is None else np.asarray(node_time, dtype=np.float64).copy()
        if post_order is None:
            self.rebuild_traversals()
        else:
            self.post_order = np.asarray(post_order, dtype=np.int32).copy()
            self.pre_order = self.post_order[::-1].copy()

    def node_count(self) -> int:
        return 2 * self.tip_count - 1

    def root(self) -> int:
        return self.node_count()

    def branch_count(self) -> int:
        return self.node_count() - 1

    def is_tip(self, node: int) -> bool:
        return 1 <= node <= self.tip_count

    def has_times(self) -> bool:
        return self.node_time is not None

    def sibling(self, node: int) -> int:
        p = self.parent[node]
        c = self.children[p]
        return int(c[1] if c[0] == node else c[0])

    def rebuild_traversals(self):
        """tree.hpp:60-77: iterative left-child-first post order; pre = reverse."""
        order: List[int] = []
        stack = [(self.root(), False)]
        while stack:
            node, expanded = stack.pop()
            if expanded or self.is_tip(node):
                order.append(node)
            else:
                stack.append((node, True))
                stack.append((int(self.children[node][1]), False))
                stack.append((int(self.children[node][0]), False))
        self.post_order = np.asarray(order, dtype=np.int32)
        self.pre_order = self.post_order[::-1].copy()

    def branch_lengths(self) -> np.ndarray:
        """Vector of the 2N-2 branch lengths, entry node-1 (engine.hpp:106-107)."""
        return self.branch_length[1:self.node_count()].copy()

    def assign_times_from_branch_lengths(self):
        """tree.hpp:131-140."""
        t = np.zeros(self.node_count() + 1)
        for node in self.pre_order:
            if node == self.root():
                continue
            if self.branch_length[node] <= 0.0:
                raise InvalidArgument("durations must be positive to assign node times")
            t[node] = t[self.parent[node]] + self.branch_length[node]
        self.node_time = t
        return t


def parse_newick(text: str) -> Tree:
    """tree.hpp:284-289, same numbering contract, errors as NewickError."""
    L = lib()
    nt = C.c_int(0)
    b = text.encode()
    check(L.pg_newick_parse(b, C.byref(nt), None, None, None, None, None, 0))
    N = nt.value
    n = 2 * N - 1
    parent = np.zeros(n + 1, np.int32)
    children = np.zeros(2 * (n + 1), np.int32)
    blen = np.zeros(n + 1, np.float64)
    post = np.zeros(n, np.int32)
    cap = len(b) + N + 16
    buf = C.create_string_buffer(cap)
    check(L.pg_newick_parse(b, C.byref(nt), ptr(parent, C.c_int32), ptr(children, C.c_int32),
                            ptr(blen, C.c_double), ptr(post, C.c_int32), buf, cap))
    names = buf.raw[:cap].split(b"\0")[:N]
    labels = [""] + [x.decode() for x in names] + [""] * (n - N)
    return Tree(N, parent, children, blen, labels, post)


# ------------------------------------------------------------------ alignment
_NUC = {"A": 1, "C": 2, "G": 4, "T": 8, "R": 5, "Y": 10, "S": 6, "W": 9, "K": 12, "M": 3, "B": 14, "D": 13,
        "H": 11, "V": 7, "N": 15, "-": 15, "?": 15}


@dataclass
class RawAlignment:
    taxa: List[str]
    sequences: List[str]

    def taxon_count(self):
        return len(self.taxa)

    def site_count(self):
        return len(self.sequences[0]) if self.taxa else 0


def _check_raw(raw: RawAlignment):
    """alignment.hpp:55-72."""
    if not raw.taxa:
        raise InvalidArgument("alignment: no records")
    seen = set()
    for r, name in enumerate(raw.taxa):
        if name in seen:
            raise InvalidArgument(f"alignment: duplicate taxon name '{name}'")
        seen.add(name)
        seq = raw.sequences[r].upper()
        if len(seq) != len(raw.sequences[0]):
            raise InvalidArgument(f"alignment: ragged record '{name}'")
        for ch in seq:
            if ch not in _NUC:
                raise InvalidArgument(f"alignment: unknown character '{ch}' in record '{name}'")
        raw.sequences[r] = seq
    if not raw.sequences[0]:
        raise InvalidArgument("alignment: zero-length sequences")


def parse_fasta(text: str) -> RawAlignment:
    """alignment.hpp:76-100."""
    taxa, seqs = [], []
    for line in text.split("\n"):
        if line.endswith("\r"):
            line = line[:-1]
        if not line or line[0] == ";":
            continue
        if line[0] == ">":
            name = line[1:].strip(" \t").split()[0] if line[1:].strip(" \t") else ""
            if not name:
                raise InvalidArgument("fasta: empty record name")
            taxa.append(name)
            seqs.append("")
        else:
            if not taxa:
                raise InvalidArgument("fasta: sequence before first header")
            seqs[-1] += "".join(line.split())
    raw = RawAlignment(taxa, seqs)
    _check_raw(raw)
    return raw


class SitePatternAlignment:
    """alignment.hpp:129-238: weighted unique site patterns in first-occurrence
    order.  Tip data are stored as compact int8 codes (state index, -1 missing,
    or m+a for ambiguity class a) instead of dense m x P partials."""

    def __init__(self, taxa, state_count, codes, weights, ambiguity=None, columns=None, site_count=None):
        self._taxa = list(taxa)
        self._m = int(state_count)
        self.codes = np.ascontiguousarray(codes, dtype=np.int8)
        self._weights = np.ascontiguousarray(weights, dtype=np.int64)
        self.ambiguity = np.zeros((0, self._m)) if ambiguity is None else f64(ambiguity).reshape(-1, self._m)
        self._columns = columns
        self._site_count = int(self._weights.sum()) if site_count is None else int(site_count)

    def state_count(self):
        return self._m

    def pattern_count(self):
        return int(self._weights.shape[0])

    def site_count(self):
        return self._site_count

    def taxa(self):
        return list(self._taxa)

    def weights(self):
        return self._weights.copy()

    def taxon_index(self, name):
        try:
            return self._taxa.index(name)
        except ValueError:
            return -1

    def pattern_column(self, p):
        return "" if self._columns is None else self._columns[p]

    def tip_partials(self, taxon_index):
        """Dense m x P partial of one taxon (alignment.hpp:138), for inspection."""
        c = self.codes[taxon_index].astype(np.int64)
        out = np.zeros((self._m, c.shape[0]))
        for s, code in enumerate(c):
            if code < 0:
                out[:, s] = 1.0
            elif code < self._m:
                out[code, s] = 1.0
            else:
                out[:, s] = self.ambiguity[code - self._m]
        return out

    @staticmethod
    def compress(raw: RawAlignment) -> "SitePatternAlignment":
        """alignment.hpp:153-182: key = literal character column."""
        _check_raw(raw)
        nt = raw.taxon_count()
        seen: Dict[str, int] = {}
        columns, weights = [], []
        for s in range(raw.site_count()):
            col = "".join(raw.sequences[r][s] for r in range(nt))
            idx = seen.get(col)
            if idx is None:
                seen[col] = len(columns)
                columns.append(col)
                weights.append(1)
            else:
                weights[idx] += 1
        masks = sorted({_NUC[ch] for col in columns for ch in col if bin(_NUC[ch]).count("1") > 1})
        cls = {mk: i for i, mk in enumerate(masks)}
        amb = np.array([[(mk >> j) & 1 for j in range(4)] for mk in masks], dtype=np.float64).reshape(-1, 4)
        codes = np.zeros((nt, len(columns)), np.int8)
        for p, col in enumerate(columns):
            for r, ch in enumerate(col):
                mk = _NUC[ch]
                codes[r, p] = (mk.bit_length() - 1) if bin(mk).count("1") == 1 else 4 + cls[mk]
        return SitePatternAlignment(raw.taxa, 4, codes, weights, amb, columns, raw.site_count())

    @staticmethod
    def from_codes(taxa: Sequence[str], codes, state_count: int, device=None) -> "SitePatternAlignment":
        """alignment.hpp:186-229 (first-occurrence order, bit-exact), compressed
        by the multithreaded hash compressor in the C-ABI, or on GPU `device`
        (pg_compress_codes_gpu) when given."""
        if device is not None:
            aln, _ = compress_codes_gpu(taxa, codes, state_count, device)
            return aln
        if state_count < 2:
            raise InvalidArgument("alignment: state count must be >= 2")
        codes = i32(codes)
        if codes.ndim != 2 or codes.shape[0] != len(taxa):
            raise InvalidArgument("alignment: taxa/codes mismatch")
        L = lib()
        h = C.c_void_p()
        npat = C.c_int(0)
        check(L.pg_compress_codes(codes.shape[0], codes.shape[1], ptr(codes, C.c_int32), state_count, C.byref(h),
                                  C.byref(npat)))
        try:
            P = npat.value
            pc = np.zeros((codes.shape[0], P), np.int32)
            w = np.zeros(P, np.int64)
            check(L.pg_compress_result(h, ptr(pc, C.c_int32), ptr(w, C.c_int64), None))
        finally:
            L.pg_compress_free(h)
        return SitePatternAlignment(taxa, state_count, pc.astype(np.int8), w, None, None, codes.shape[1])


def compress_codes_gpu(taxa: Sequence[str], codes, state_count: int, device: int = 0, with_site_map=False):
    """GPU first-occurrence compression (pg_compress_codes_gpu, SURVEY.md §8f
    row 3), bit-exact with from_codes.  `codes` is int8-convertible [ntax][sites]
    (values -1..m-1).  Returns (SitePatternAlignment, info) where info holds
    the device time of the compression kernels and, if requested, the
    site -> pattern map."""
    if state_count < 2:
        raise InvalidArgument("alignment: state count must be >= 2")
    codes = np.asarray(codes)
    if codes.ndim != 2 or codes.shape[0] != len(taxa):
        raise InvalidArgument("alignment: taxa/codes mismatch")
    if codes.size and (codes.min() < -1 or codes.max() >= state_count):
        raise InvalidArgument("alignment: state code out of range")
    c8 = np.ascontiguousarray(codes, dtype=np.int8)
    L = lib()
    h = C.c_void_p()
    npat = C.c_int(0)
    check(L.pg_compress_codes_gpu(c8.shape[0], c8.shape[1], c8.ctypes.data_as(C.c_void_p), 0, state_count, device,
                                  C.byref(h), C.byref(npat)))
    try:
        P = npat.value
        pc = np.zeros((c8.shape[0], P), np.int8)
        w = np.zeros(P, np.int64)
        site = np.zeros(c8.shape[1], np.int32) if with_site_map else None
        ms = C.c_float(0.0)
        check(L.pg_compress_result_gpu(h, pc.ctypes.data_as(C.c_void_p), ptr(w, C.c_int64),
                                       ptr(site, C.c_int32) if site is not None else None, C.byref(ms)))
    finally:
        L.pg_compress_free_gpu(h)
    info = {"device_ms": float(ms.value), "site_to_pattern": site}
    return SitePatternAlignment(taxa, state_count, pc, w, None, None, c8.shape[1]), info


# -------------------------------------------------------------------- models
@dataclass
class RateCategories:
    rates: np.ndarray
    probs: np.ndarray

    def count(self):
        return int(len(self.rates))

    @staticmethod
    def single():
        return RateCategories(np.ones(1), np.ones(1))

    @staticmethod
    def make(rates, probs):
        """substitution.hpp:36-50."""
        rates, probs = f64(rates), f64(probs)
        if rates.size < 1 or rates.size != probs.size:
            raise InvalidArgument("rate categories: need L >= 1 matched rates/probs")
        if np.any(rates <= 0):
            raise InvalidArgument("rate categories: rates must be positive")
        if abs(probs.sum() - 1.0) > 1e-12:
            raise InvalidArgument("rate categories: probabilities must sum to 1")
        if abs(rates @ probs - 1.0) > 1e-10:
            raise InvalidArgument("rate categories: mixture mean must be 1")
        return RateCategories(rates.copy(), probs.copy())


def discrete_gamma_categories(alpha: float, count: int) -> RateCategories:
    """substitution.hpp:55-68 (bin medians rescaled to mean one)."""
    r = np.zeros(max(count, 1))
    p = np.zeros(max(count, 1))
    check(lib().pg_discrete_gamma(float(alpha), int(count), ptr(r, C.c_double), ptr(p, C.c_double)))
    return RateCategories(r, p)


def _finish_generator(q, pi):
    """substitution.hpp:183-191."""
    q = q.copy()
    np.fill_diagonal(q, 0.0)
    np.fill_diagonal(q, -q.sum(axis=1))
    rate = -float(np.sum(pi * np.diag(q)))
    return q / rate


def _check_generator(q):
    """substitution.hpp:168-180."""
    if not np.all(np.isfinite(q)):
        raise InvalidArgument("generator: non-finite entries")
    off = q - np.diag(np.diag(q))
    if np.any(off < 0):
        raise InvalidArgument("generator: negative off-diagonal entry")
    if np.any(np.abs(q.sum(axis=1)) > 1e-12):
        raise InvalidArgument("generator: rows must sum to zero")


class SubstitutionModel:
    """substitution.hpp:77-219 (generators and root distribution; P(t) itself is
    formed on the GPU by the engine)."""

    def __init__(self, q, pi, reversible: bool):
        q = f64(q)
        _check_generator(q)
        pi = f64(pi)
        if pi.size != q.shape[0]:
            raise InvalidArgument("model: pi length must match state count")
        if np.any(pi < -1e-12) or abs(pi.sum() - 1.0) > 1e-12:
            raise InvalidArgument("model: pi must be a probability vector")
        self._q = q.copy()
        self._pi = pi.copy()
        self._reversible = bool(reversible)
        self._branch_q: Dict[int, np.ndarray] = {}

    @staticmethod
    def jc69():
        return SubstitutionModel.hky85(1.0, [0.25] * 4)

    @staticmethod
    def hky85(kappa, freqs):
        if not kappa > 0:
            raise InvalidArgument("hky85: kappa must be positive")
        return SubstitutionModel.gtr([1.0, kappa, 1.0, 1.0, kappa, 1.0], freqs)

    @staticmethod
    def gtr(exchangeabilities, freqs):
        e = f64(exchangeabilities)
        f = f64(freqs)
        if np.any(e <= 0):
            raise InvalidArgument("gtr: exchangeabilities must be positive")
        if np.any(f <= 0) or abs(f.sum() - 1.0) > 1e-12:
            raise InvalidArgument("frequencies must be positive and sum to 1")
        q = np.zeros((4, 4))
        k = 0
        for i in range(4):
            for j in range(i + 1, 4):
                q[i, j] = e[k] * f[j]
                q[j, i] = e[k] * f[i]
                k += 1
        return SubstitutionModel(_finish_generator(q, f), f, True)

    def state_count(self):
        return int(self._q.shape[0])

    def root_distribution(self):
        return self._pi.copy()

    def reversible(self):
        return self._reversible

    def homogeneous(self):
        return not self._branch_q

    def generator(self, branch: int = 0):
        return self._branch_q.get(branch, self._q).copy()

    def set_branch_generator(self, branch: int, q):
        q = f64(q)
        if q.shape != self._q.shape:
            raise InvalidArgument("branch generator: wrong dimensions")
        _check_generator(q)
        self._branch_q[int(branch)] = q.copy()


# -------------------------------------------------------------------- engine
@dataclass
class EngineOptions:
    """engine.hpp:33-37, plus device placement and debug capture."""
    rescaling_threshold: float = 1e-150
    force_rescaling: bool = False
    disable_rescaling: bool = False
    device: int = 0
    capture_partials: bool = False
    # multi-GPU from one process (pg_create_multi): shard the patterns over
    # these devices; reduce "nccl" (ncclAllReduce) or "fixed" (rank-order sum
    # on the first device, bit-reproducible; repeated devices allowed)
    devices: Optional[Sequence[int]] = None
    reduce: str = "nccl"


@dataclass
class ClockGradient:
    """Likelihood part of RelaxedClockPosterior::gradient (clock.hpp:140-152)
    and node_time_gradient (clock.hpp:199-213)."""
    log_likelihood: float = 0.0
    dlog_mu: float = 0.0                                                 # sum_i b_i g_i
    dlog_epsilon: np.ndarray = field(default_factory=lambda: np.zeros(0))  # b_i g_i
    node_time: np.ndarray = field(default_factory=lambda: np.zeros(0))     # [N-1], nodes N+1..2N-1


@dataclass
class GradientReport:
    """engine.hpp:39-45."""
    log_likelihood: float = 0.0
    branch_gradient: np.ndarray = field(default_factory=lambda: np.zeros(0))
    hessian_diagonal: np.ndarray = field(default_factory=lambda: np.zeros(0))
    pattern_count: int = 0
    category_count: int = 0


class LikelihoodEngine:
    """engine.hpp:47-438 on the GPU.

    Unlike the reference (which keeps const references, engine.hpp:416-418),
    the engine copies tree, patterns, model and categories to device memory at
    construction; later mutation of the host objects has no effect.
    """

    def __init__(self, tree: Tree, alignment: SitePatternAlignment, model: SubstitutionModel,
                 categories: RateCategories, options: Optional[EngineOptions] = None):
        opts = options or EngineOptions()
        m = model.state_count()
        if alignment.state_count() != m:
            raise InvalidArgument("engine: alignment/model state counts differ")
        if len(alignment.taxa()) != tree.tip_count:
            raise InvalidArgument("engine: alignment must carry exactly one record per tree tip")
        rows = []
        for t in range(1, tree.tip_count + 1):
            r = alignment.taxon_index(tree.labels[t])
            if r < 0:
                raise InvalidArgument(f"engine: tree tip '{tree.labels[t]}' not found in alignment")
            rows.append(r)
        self._tree, self._aln, self._model = tree, alignment, model
        self._cats = RateCategories(f64(categories.rates).copy(), f64(categories.probs).copy())
        self._opts = opts
        L = lib()
        o = _L.Options()
        L.pg_default_options(C.byref(o))
        o.rescaling_threshold = opts.rescaling_threshold
        o.force_rescaling = int(opts.force_rescaling)
        o.disable_rescaling = int(opts.disable_rescaling)
        o.device = int(opts.device)
        o.capture_partials = int(opts.capture_partials)
        h = C.c_void_p()
        if opts.devices:
            if opts.reduce not in ("nccl", "fixed"):
                raise InvalidArgument("engine: reduce must be 'nccl' or 'fixed'")
            devs = (C.c_int * len(opts.devices))(*[int(d) for d in opts.devices])
            check(L.pg_create_multi(C.byref(o), len(opts.devices), devs,
                                    _L.REDUCE_NCCL if opts.reduce == "nccl" else _L.REDUCE_FIXED_ORDER, C.byref(h)))
        else:
            check(L.pg_create(C.byref(o), C.byref(h)))
        self._h = h
        children = np.ascontiguousarray(tree.children.reshape(-1), np.int32)
        check(L.pg_set_topology(h, tree.tip_count, ptr(i32(tree.parent), C.c_int32), ptr(children, C.c_int32),
                                ptr(i32(tree.post_order), C.c_int32)))
        codes = np.ascontiguousarray(alignment.codes[rows], np.int8)
        self._codes = codes
        amb = f64(alignment.ambiguity).reshape(-1)
        w = np.ascontiguousarray(alignment.weights(), np.int64)
        check(L.pg_set_patterns(h, m, alignment.pattern_count(), ptr(codes, C.c_int8), alignment.ambiguity.shape[0],
                                ptr(amb, C.c_double) if amb.size else None, ptr(w, C.c_int64)))
        q = f64(model.generator(0))
        check(L.pg_set_model(h, m, ptr(q, C.c_double), ptr(f64(model.root_distribution()), C.c_double),
                             int(model.reversible())))
        for br, qb in model._branch_q.items():
            qb = f64(qb)
            check(L.pg_set_branch_generator(h, br, ptr(qb, C.c_double)))
        check(L.pg_set_categories(h, self._cats.count(), ptr(self._cats.rates, C.c_double),
                                  ptr(self._cats.probs, C.c_double)))
        self._B = tree.branch_count()
        self.set_branch_lengths(tree.branch_lengths())

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().pg_destroy(h)
            except Exception:  # interpreter shutdown: module globals already gone
                pass
            self._h = None

    # --- accessors (engine.hpp:112-114)
    def tree(self):
        return self._tree

    def categories(self):
        return self._cats

    def branch_lengths(self):
        b = np.zeros(self._B)
        check(lib().pg_get_branch_lengths(self._h, ptr(b, C.c_double)))
        return b

    def set_branch_lengths(self, lengths):
        """engine.hpp:116-124."""
        b = f64(lengths)
        if b.shape != (self._B,):
            raise InvalidArgument("engine: branch length vector has wrong size")
        check(lib().pg_set_branch_lengths(self._h, ptr(b, C.c_double)))

    def set_clock_durations(self, durations):
        d = f64(durations)
        if d.shape != (self._B,):
            raise InvalidArgument("clock: need one duration per branch")
        check(lib().pg_set_clock_durations(self._h, ptr(d, C.c_double)))

    def node_visits(self):
        return int(lib().pg_node_visits(self._h))

    def reset_node_visits(self):
        lib().pg_reset_node_visits(self._h)

    def invalidate_caches(self):
        lib().pg_invalidate_caches(self._h)

    # --- evaluation (engine.hpp:146-164)
    def _eval(self, flags):
        ll = C.c_double(0.0)
        g = np.zeros(self._B)
        h = np.zeros(self._B)
        check(lib().pg_evaluate(self._h, flags, C.byref(ll), ptr(g, C.c_double), ptr(h, C.c_double)))
        return ll.value, g, h

    def log_likelihood(self) -> float:
        return self._eval(_L.EVAL_LOGL)[0]

    def post_order_pass(self):
        self._eval(_L.EVAL_LOGL | _L.EVAL_POST_PASS)

    def pre_order_pass(self, with_hessian_diagonal=False):
        self._eval(_L.EVAL_GRAD | _L.EVAL_REQUIRE_POST | (_L.EVAL_HESS if with_hessian_diagonal else 0))

    def branch_gradient(self, with_hessian_diagonal=False) -> GradientReport:
        flags = _L.EVAL_GRAD | (_L.EVAL_HESS if with_hessian_diagonal else 0)
        ll, g, h = self._eval(flags)
        return GradientReport(ll, g, h if with_hessian_diagonal else np.zeros(0), self._aln.pattern_count(),
                              self._cats.count())

    def hessian_diagonal(self):
        return self.branch_gradient(True).hessian_diagonal

    def rate_gradient(self, with_hessian_diagonal=False) -> GradientReport:
        """d logL / d r_i = dt_i g_i for b_i = r_i dt_i (clock.hpp:146-152,
        cli.hpp:437-438), chain rule applied on the GPU."""
        flags = _L.EVAL_RATE_GRAD | (_L.EVAL_HESS if with_hessian_diagonal else 0)
        ll, g, h = self._eval(flags)
        return GradientReport(ll, g, h if with_hessian_diagonal else np.zeros(0), self._aln.pattern_count(),
                              self._cats.count())

    def clock_gradient(self, rates=None) -> ClockGradient:
        """clock.hpp:140-152 / :199-213 on the GPU at the current lengths
        b_i = r_i dt_i: d logL/d log eps_i = b_i g_i, d logL/d log mu =
        sum_i b_i g_i (fixed order), d logL/d t_k (internal nodes).  `rates`
        r_i = mu eps_i; None derives them as b_i / dt_i from the durations."""
        r = None if rates is None else f64(rates)
        if r is not None and r.shape != (self._B,):
            raise InvalidArgument("clock: need one rate per branch")
        ll, mu = C.c_double(), C.c_double()
        eps = np.zeros(self._B)
        node = np.zeros(self._tree.tip_count - 1)
        check(lib().pg_clock_gradient(self._h, None if r is None else ptr(r, C.c_double), C.byref(ll), C.byref(mu),
                                      ptr(eps, C.c_double), ptr(node, C.c_double)))
        return ClockGradient(ll.value, mu.value, eps, node)

    def group_info(self):
        n, v, r = C.c_int(), C.c_int(), C.c_int()
        check(lib().pg_group_info(self._h, C.byref(n), C.byref(v), C.byref(r)))
        return {"shards": n.value, "nccl_version": v.value, "reduce": ["nccl", "fixed"][r.value]}

    def site_log_likelihoods(self):
        out = np.zeros(self._aln.pattern_count())
        check(lib().pg_get_site_log_likelihoods(self._h, ptr(out, C.c_double)))
        return out

    # --- debug accessors (engine.hpp:134-141), need capture_partials
    def _partials(self, node, category):
        m, P = self._model.state_count(), self._aln.pattern_count()
        a = np.zeros(m * P)
        b = np.zeros(m * P)
        sa = np.zeros(P)
        sb = np.zeros(P)
        check(lib().pg_get_partials(self._h, node, category, ptr(a, C.c_double), ptr(b, C.c_double),
                                    ptr(sa, C.c_double), ptr(sb, C.c_double)))
        return a.reshape(P, m).T, b.reshape(P, m).T, sa, sb

    def post_partial(self, node, category):
        if self._tree.is_tip(node):
            return self._aln.tip_partials(self._aln.taxon_index(self._tree.labels[node]))
        return self._partials(node, category)[0]

    def pre_partial(self, node, category):
        return self._partials(node, category)[1]

    def post_scaler(self, node):
        if self._tree.is_tip(node):
            return np.zeros(self._aln.pattern_count())
        return self._partials(node, 0)[2]

    def pre_scaler(self, node):
        return self._partials(node, 0)[3]

    def log_likelihood_at_node(self, node):
        """engine.hpp:168-180 from the captured partials."""
        self.branch_gradient()
        w = self._aln.weights().astype(np.float64)
        mix = np.zeros(self._aln.pattern_count())
        for l in range(self._cats.count()):
            mix += self._cats.probs[l] * np.sum(self.post_partial(node, l) * self.pre_partial(node, l), axis=0)
        return float(np.sum(w * (np.log(mix) + self.post_scaler(node) + self.pre_scaler(node))))

    def info(self):
        a, b, c, d = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        check(lib().pg_engine_info(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        return {"launches": a.value, "total_warps": b.value, "lanes_per_pattern": c.value, "padded_states": d.value,
                "kernel": ["walk_kernel", "walk4_kernel", "walkm_kernel",
                           "walkl_kernel", "walk4s_kernel", "walk4t_kernel"][lib().pg_engine_variant(self._h)]}

    def last_times_ms(self):
        w, t = C.c_float(), C.c_float()
        check(lib().pg_last_walk_ms(self._h, C.byref(w), C.byref(t)))
        return w.value, t.value

    @property
    def handle(self):
        return self._h


# --------------------------------------------------------------------- clock
def branch_lengths_from_clock(tree: Tree, mu: float, epsilon) -> np.ndarray:
    """clock.hpp:42-55: b_i = mu eps_i (t_i - t_pa(i))."""
    if not tree.has_times():
        raise InvalidArgument("clock: tree has no node times attached")
    eps = f64(epsilon)
    if eps.size != tree.branch_count():
        raise InvalidArgument("clock: need one epsilon per branch")
    if not mu > 0 or np.any(eps <= 0):
        raise InvalidArgument("clock: rates must be positive")
    i = np.arange(1, tree.node_count())
    return mu * eps * (tree.node_time[i] - tree.node_time[tree.parent[i]])


def node_time_gradient(engine: "LikelihoodEngine", tree: Tree, mu: float, epsilon) -> np.ndarray:
    """RelaxedClockPosterior::node_time_gradient (clock.hpp:199-213): sets the
    engine's lengths from the clock (b_i = mu eps_i dt_i), evaluates the
    branch gradient and returns d logL / d t_k = r_k g_k [k non-root] -
    sum_children r_c g_c for the internal nodes N+1..2N-1 (computed on the GPU)."""
    eps = f64(epsilon)
    engine.set_branch_lengths(branch_lengths_from_clock(tree, mu, eps))
    return engine.clock_gradient(mu * eps).node_time


def clock_likelihood_gradient(engine: "LikelihoodEngine", tree: Tree, mu: float, epsilon):
    """Likelihood part of RelaxedClockPosterior::gradient in the unconstrained
    space (clock.hpp:140-152): returns (d logL/d log mu, d logL/d log eps)."""
    eps = f64(epsilon)
    engine.set_branch_lengths(branch_lengths_from_clock(tree, mu, eps))
    cg = engine.clock_gradient(mu * eps)
    return cg.dlog_mu, cg.dlog_epsilon
