"""GPU site-pattern compression (pg_compress_codes_gpu)
against the oracle's restatement of alignment.hpp:186-229 and the host
compressor: pattern order, codes, weights and the site map must be bit-exact."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _gpu(codes, m, with_map=True):
    import paper_1905_12146_b200 as pg

    labels = [f"t{i}" for i in range(codes.shape[0])]
    return pg.compress_codes_gpu(labels, codes, m, 0, with_site_map=with_map)


def _host_site_map(codes, m):
    from paper_1905_12146_b200._lib import check, lib, ptr

    c32 = np.ascontiguousarray(codes, dtype=np.int32)
    L = lib()
    h = C.c_void_p()
    n = C.c_int(0)
    check(L.pg_compress_codes(c32.shape[0], c32.shape[1], ptr(c32, C.c_int32), m, C.byref(h), C.byref(n)))
    try:
        site = np.zeros(c32.shape[1], np.int32)
        w = np.zeros(n.value, np.int64)
        pc = np.zeros((c32.shape[0], n.value), np.int32)
        check(L.pg_compress_result(h, ptr(pc, C.c_int32), ptr(w, C.c_int64), ptr(site, C.c_int32)))
    finally:
        L.pg_compress_free(h)
    return pc, w, site


def _check_against_oracle(codes, m):
    aln, info = _gpu(codes, m)
    ref = O.Alignment.from_codes(codes.astype(np.int32), m, [f"t{i}" for i in range(codes.shape[0])])
    assert aln.pattern_count() == ref.pattern_count
    assert np.array_equal(aln.weights(), ref.weights)
    assert np.array_equal(aln.codes.astype(np.int32), ref.pattern_codes())
    pc, w, site = _host_site_map(codes, m)
    assert np.array_equal(info["site_to_pattern"], site)
    # the map reproduces every column
    assert np.array_equal(aln.codes[:, info["site_to_pattern"]].astype(np.int32), codes.astype(np.int32))
    return aln, info


@pytest.mark.parametrize("seed,m", [(1, 4), (2, 20), (3, 61)])
def test_random_with_duplicates(seed, m):
    rng = np.random.default_rng(seed)
    ntax, sites = 9, 5000
    codes = rng.integers(-1, m, size=(ntax, sites))
    codes[:, ::3] = codes[:, 7:8]
    codes[:, 1::11] = codes[:, 4:5]
    codes[:, 2::5] = codes[:, 2::5][:, ::-1]
    _check_against_oracle(codes, m)


def test_low_entropy_columns():  # many repeats, few distinct columns, gaps
    rng = np.random.default_rng(7)
    codes = rng.choice([-1, 0, 1], size=(30, 20000), p=[0.05, 0.9, 0.05])
    aln, _ = _check_against_oracle(codes, 4)
    assert aln.weights().sum() == 20000


def test_edge_cases():
    # one taxon
    _check_against_oracle(np.array([[0, 1, 0, 2, 2, -1]]), 4)
    # all columns identical
    aln, info = _check_against_oracle(np.tile(np.array([[1], [2], [-1]]), (1, 777)), 4)
    assert aln.pattern_count() == 1 and aln.weights()[0] == 777
    assert not info["site_to_pattern"].any()
    # every column distinct
    codes = np.array([[i % 4, (i // 4) % 4, (i // 16) % 4] for i in range(64)]).T
    aln, _ = _check_against_oracle(codes, 4)
    assert aln.pattern_count() == 64
    # all missing
    aln, _ = _check_against_oracle(-np.ones((5, 100), np.int64), 4)
    assert aln.pattern_count() == 1
    # one column
    _check_against_oracle(np.array([[3], [0]]), 4)


def test_empty_alignment():
    aln, info = _gpu(np.zeros((4, 0), np.int8), 4)
    assert aln.pattern_count() == 0 and aln.weights().size == 0


def test_rejects_out_of_range_in_kernel():
    """The device kernel validates codes itself (called below the Python check)."""
    import paper_1905_12146_b200 as pg
    from paper_1905_12146_b200._lib import check, lib

    c8 = np.zeros((3, 4000), np.int8)
    c8[2, 3999] = 4
    h = C.c_void_p()
    n = C.c_int(0)
    with pytest.raises(pg.InvalidArgument, match="out of range"):
        check(lib().pg_compress_codes_gpu(3, 4000, c8.ctypes.data_as(C.c_void_p), 0, 4, 0, C.byref(h), C.byref(n)))
    c8[2, 3999] = -2
    with pytest.raises(pg.InvalidArgument, match="out of range"):
        check(lib().pg_compress_codes_gpu(3, 4000, c8.ctypes.data_as(C.c_void_p), 0, 4, 0, C.byref(h), C.byref(n)))


def test_large_matches_host():
    """10^6 columns x 128 taxa (C3-scale column count), ~40 % duplicates."""
    rng = np.random.default_rng(11)
    ntax, sites = 128, 1_000_000
    codes = rng.integers(0, 4, size=(ntax, sites), dtype=np.int8)
    dup = rng.random(sites) < 0.4
    src = rng.integers(0, sites, size=sites)
    src = np.where(dup, np.minimum(src, np.arange(sites)), np.arange(sites))
    codes = codes[:, src]
    aln, info = _gpu(codes, 4)
    pc, w, site = _host_site_map(codes, 4)
    assert aln.pattern_count() == w.size
    assert np.array_equal(aln.weights(), w)
    assert np.array_equal(info["site_to_pattern"], site)
    assert np.array_equal(aln.codes.astype(np.int32), pc)
    assert info["device_ms"] > 0.0
