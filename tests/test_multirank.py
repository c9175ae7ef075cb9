"""World-size-2 gloo test of the multi-GPU path's host logic (CPU): contiguous
pattern shards, one all-reduce of [logL, g, H], result equal to the unsharded
evaluation.  The local engine is the CPU oracle here (no GPU in CI); on the
B200 the same ShardedEngine drives the CUDA engine over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O


class OracleLocal:
    """Adapter: product API setup types -> CPU oracle engine."""

    def __init__(self, tree, aln, model, cats, options=None):
        self.t = O.Tree.from_arrays(tree.tip_count, tree.parent, tree.children, tree.branch_lengths(), tree.post_order)
        self.a = O.Alignment.from_patterns(aln.codes.astype(np.int32), aln.state_count(), aln.weights())
        self.m = O.Model(model.generator(0), model.root_distribution(), model.reversible())
        self.e = O.Engine(self.t, self.a, self.m, cats.rates, cats.probs)

    def branch_gradient(self, hess=False):
        return self.e.branch_gradient(hess)

    def log_likelihood(self):
        return self.e.log_likelihood()

    def set_branch_lengths(self, b):
        self.e.set_branch_lengths(b)

    def invalidate_caches(self):
        self.e.invalidate_caches()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from workloads import synth
        from paper_1905_12146_b200.api import RateCategories, SitePatternAlignment, SubstitutionModel, Tree
        from paper_1905_12146_b200.sharding import ShardedEngine, shard_range

        inst = synth.generate("C2", seed=5, sites=1500, tips=40)
        labels = inst.labels()
        tree = Tree(inst.tip_count, inst.parent, inst.children, np.concatenate([[0.0], inst.branch_lengths, [0.0]]),
                    labels, inst.post_order)
        aln = SitePatternAlignment(labels[1:inst.tip_count + 1], inst.states, inst.codes, inst.weights)
        model = SubstitutionModel(inst.q, inst.pi, inst.reversible)
        cats = RateCategories(inst.cat_rates, inst.cat_probs)
        sh = ShardedEngine(tree, aln, model, cats, engine_factory=OracleLocal)
        assert (sh.p0, sh.p1) == shard_range(inst.patterns, rank, world)
        rep = sh.branch_gradient(True)
        ll = sh.log_likelihood()
        result_q.put((rank, rep.log_likelihood, rep.branch_gradient, rep.hessian_diagonal, ll, sh.p1 - sh.p0))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharded_gradient():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from workloads import synth
    from tests.helpers import oracle_for

    inst = synth.generate("C2", seed=5, sites=1500, tips=40)
    ll, g, h = oracle_for(inst).branch_gradient(True)
    assert sum(r[5] for r in results) == inst.patterns
    for _, rll, rg, rh, rll2, _ in results:
        assert rll == pytest.approx(ll, rel=1e-12)
        assert rll2 == pytest.approx(ll, rel=1e-12)
        np.testing.assert_allclose(rg, g, rtol=1e-10, atol=1e-12 * np.abs(g).max())
        np.testing.assert_allclose(rh, h, rtol=1e-10, atol=1e-12 * np.abs(h).max())
    # every rank holds the identical reduced vector
    np.testing.assert_array_equal(results[0][2], results[1][2])


def test_shard_ranges_partition():
    from paper_1905_12146_b200.sharding import shard_range

    for P in (0, 1, 7, 1000, 906112):
        for G in (1, 2, 3, 4, 8):
            blocks = [shard_range(P, r, G) for r in range(G)]
            assert blocks[0][0] == 0 and blocks[-1][1] == P
            for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
                assert a1 == b0 and a0 <= a1


@pytest.mark.gpu
def test_single_rank_nccl_device_path():
    """The NCCL device path of ShardedEngine (pg_evaluate_device into a CUDA
    buffer + all-reduce on the engine's stream) against the oracle, with a
    one-rank NCCL group (a multi-rank NCCL group needs one GPU per rank)."""
    import torch
    import torch.distributed as dist

    from workloads import synth
    from paper_1905_12146_b200.api import RateCategories, SitePatternAlignment, SubstitutionModel, Tree
    from paper_1905_12146_b200.sharding import ShardedEngine
    from tests.helpers import assert_logl, assert_vec, oracle_for

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        inst = synth.generate("C4", seed=9, sites=400, tips=60)
        labels = inst.labels()
        tree = Tree(inst.tip_count, inst.parent, inst.children,
                    np.concatenate([[0.0], inst.branch_lengths, [0.0]]), labels, inst.post_order)
        aln = SitePatternAlignment(labels[1:inst.tip_count + 1], inst.states, inst.codes, inst.weights)
        sh = ShardedEngine(tree, aln, SubstitutionModel(inst.q, inst.pi, inst.reversible),
                           RateCategories(inst.cat_rates, inst.cat_probs))
        assert sh._device_path
        rep = sh.branch_gradient(True)
        ll, g, h = oracle_for(inst, blocks=4).branch_gradient(True)
        assert_logl(rep.log_likelihood, ll)
        assert_vec(rep.branch_gradient, g)
        assert_vec(rep.hessian_diagonal, h, rtol=1e-8, what="hessian")
    finally:
        dist.destroy_process_group()


def _share_worker(rank, world, port, q):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from workloads import synth

        inst = synth.generate_shared("C2", rank, world, dist.barrier, tag=f"test{port}", seed=3, sites=700)
        q.put((rank, inst.patterns, int(inst.codes.astype(np.int64).sum()), int(inst.weights.sum()),
               float(inst.branch_lengths.sum())))
    finally:
        dist.destroy_process_group()


def test_shared_workload_generation():
    """bench.py's multi-rank setup: rank 0 simulates, the others load the
    identical instance from node-local shared memory."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_share_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from workloads import synth

    ref = synth.generate("C2", seed=3, sites=700)
    want = (ref.patterns, int(ref.codes.astype(np.int64).sum()), int(ref.weights.sum()), float(ref.branch_lengths.sum()))
    for r in res:
        assert r[1:] == want


def _bench_worker(rank, world, port, q):
    """bench.py's multi-rank e2e step on CPU: shared workload generation,
    the product ShardedEngine over this rank's block (oracle as the local
    engine), the clock chain rule (set_clock_durations + rate_gradient)."""
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1905_12146_b200.sharding import ShardedEngine
        from workloads import synth

        inst = synth.generate_shared("C3", rank, world, dist.barrier, tag=f"bench{port}", seed=11, sites=900)
        sh = ShardedEngine(*synth.api_objects(inst), engine_factory=OracleLocal)
        sh.set_clock_durations(inst.durations)
        b = inst.branch_rates * inst.durations
        sh.set_branch_lengths(b)
        rep = sh.rate_gradient()
        q.put((rank, rep.log_likelihood, rep.branch_gradient, sh.p1 - sh.p0))
    finally:
        dist.destroy_process_group()


def test_bench_multirank_step_gloo():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from tests.helpers import oracle_for
    from workloads import synth

    inst = synth.generate("C3", seed=11, sites=900)
    ll, g, _ = oracle_for(inst, blocks=4).branch_gradient(False)
    assert sum(r[3] for r in results) == inst.patterns
    for _, rll, rg, _ in results:
        assert rll == pytest.approx(ll, rel=1e-12)
        np.testing.assert_allclose(rg, inst.durations * g, rtol=1e-10,
                                   atol=1e-12 * np.abs(inst.durations * g).max())


def test_bench_relaunches_under_torchrun(monkeypatch):
    """`bench.py --gpus N` outside torchrun re-executes itself under
    torch.distributed.run with N processes on a 127.0.0.1 rendezvous; under
    torchrun a --gpus / WORLD_SIZE mismatch is an error."""
    import bench

    monkeypatch.delenv("WORLD_SIZE", raising=False)
    args = bench.parse_args(["--gpus", "4", "--steps", "2"])
    cmd = bench.relaunch_command(args, ["--gpus", "4", "--steps", "2"])
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "2"]
    assert bench.relaunch_command(bench.parse_args(["--gpus", "1"]), []) is None
    assert bench.relaunch_command(bench.parse_args(["--gpus", "4", "--impl", "reference"]), []) is None
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert bench.relaunch_command(args, []) is None
    assert bench.main(["--gpus", "4"]) == 2


def _product_worker(rank, world, port, q):
    """One rank of the sharded product on the GPU: the CUDA LikelihoodEngine
    over this rank's pattern block, the [logL, g, H] all-reduce over gloo
    (host tensors -- no rank's kernel waits on another's)."""
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_1905_12146_b200.sharding import ShardedEngine
        from workloads import synth

        inst = synth.generate("C3", seed=13, sites=20000, tips=128)
        sh = ShardedEngine(*synth.api_objects(inst))
        assert not sh._device_path and hasattr(sh.local, "handle")  # the CUDA engine, host reduction
        sh.set_clock_durations(inst.durations)
        rep = sh.branch_gradient(True)
        rrep = sh.rate_gradient()
        q.put((rank, rep.log_likelihood, rep.branch_gradient, rep.hessian_diagonal, rrep.branch_gradient,
               sh.p1 - sh.p0, sh.local.info()["kernel"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_product_on_gpu(world):
    """The multi-GPU path with the product as the local engine: `world`
    processes each evaluate their contiguous pattern block with the CUDA
    engine; the reduced logL, gradient, Hessian and rate gradient equal the
    unsharded product evaluation (summation order only) and the oracle."""
    from tests.helpers import assert_logl, assert_vec, oracle_for
    from workloads import synth

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_product_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted((q.get(timeout=600) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0

    inst = synth.generate("C3", seed=13, sites=20000, tips=128)
    assert sum(r[5] for r in results) == inst.patterns
    eng = synth.engine_for(inst)
    whole = eng.branch_gradient(True)
    ll, g, h = oracle_for(inst, blocks=8).branch_gradient(True)
    for _, rll, rg, rh, rr, _, kernel in results:
        # every rank holds the same reduced result
        assert rll == results[0][1] and np.array_equal(rg, results[0][2])
        assert rll == pytest.approx(whole.log_likelihood, rel=1e-13)
        np.testing.assert_allclose(rg, whole.branch_gradient, rtol=1e-11,
                                   atol=1e-13 * np.abs(whole.branch_gradient).max())
        assert_logl(rll, ll)
        assert_vec(rg, g)
        assert_vec(rh, h, rtol=1e-8, what="hessian")
        assert_vec(rr, inst.durations * g, what="rate gradient")
