"""Throughput of the GPU site-pattern compressor (pg_compress_codes_gpu) vs the
multithreaded host compressor, C3-shaped columns (2048 taxa, 4 states)."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12146_b200 as pg  # noqa: E402
from paper_1905_12146_b200._lib import check, lib, ptr  # noqa: E402

ntax = 2048
rng = np.random.default_rng(5)
out = []
SIZES = [(int(a), b == "1") for a, b in (x.split(":") for x in os.environ.get("SIZES", "250000:1,1000000:0").split(","))]
for sites, host in SIZES:
    codes = rng.integers(0, 4, size=(ntax, sites), dtype=np.int8)
    src = np.where(rng.random(sites) < 0.1, rng.integers(0, sites, size=sites), np.arange(sites))
    src = np.minimum(src, np.arange(sites))
    codes = np.ascontiguousarray(codes[:, src])
    labels = [f"t{i}" for i in range(ntax)]
    pg.compress_codes_gpu(labels, codes[:, :1000], 4, 0)  # warm up the context
    t = time.perf_counter()
    aln, info = pg.compress_codes_gpu(labels, codes, 4, 0, with_site_map=True)
    wall = time.perf_counter() - t
    rec = {"taxa": ntax, "sites": sites, "patterns": aln.pattern_count(), "gpu_kernels_ms": info["device_ms"],
           "gpu_wall_s_incl_h2d_d2h": wall, "input_GB": ntax * sites / 1e9,
           "gpu_GBps": ntax * sites / 1e9 / (info["device_ms"] * 1e-3)}
    if host:
        c32 = codes.astype(np.int32)
        h = C.c_void_p()
        n = C.c_int(0)
        t = time.perf_counter()
        check(lib().pg_compress_codes(ntax, sites, ptr(c32, C.c_int32), 4, C.byref(h), C.byref(n)))
        rec["host_s"] = time.perf_counter() - t
        rec["host_threads"] = os.cpu_count()
        site = np.zeros(sites, np.int32)
        w = np.zeros(n.value, np.int64)
        check(lib().pg_compress_result(h, None, ptr(w, C.c_int64), ptr(site, C.c_int32)))
        lib().pg_compress_free(h)
        rec["bit_exact_vs_host"] = bool(np.array_equal(site, info["site_to_pattern"]) and
                                        np.array_equal(w, aln.weights()))
    out.append(rec)
    print(json.dumps(rec), flush=True)
