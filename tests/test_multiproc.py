"""World-size-2 gloo tests of the multi-rank host path (CPU tier).

The path is embarrassingly parallel: rank r owns the contiguous orbit shard
shard_bounds(M, W, r) with its GLOBAL orbit ids, there is no data-path
collective, and the host-assembled store must be bit-identical to a single
process run.  On CPU the device integration of each shard is stood in by the
oracle (test-only monkeypatch) so the sharding, orbit-id offsets, failure
renumbering, gather/assembly and the max-over-ranks timing reduction of
bench.py are exercised end to end.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_run_batch(model, config, batch, *, orbit_offset=0):
    """Test stand-in for the device run: the oracle on global ids."""
    from oracle import sdeb_oracle as O
    from paper_1908_03869_b200.engine import (OrbitFailure, TrajectoryStore,
                                              iteration_count)
    chunks = iteration_count(config.tspan, config.dt, config.ksteps)
    times, values, fails = O.integrate(
        batch.init, batch.params, dt=config.dt, ksteps=config.ksteps, chunks=chunks,
        seed=config.seed, stream=config.stream,
        orbit_ids=np.arange(orbit_offset, orbit_offset + batch.orbits))
    failures = [OrbitFailure(*f) for f in fails]
    return TrajectoryStore(times=times, values=values, model_name=model.name, config=config,
                           failures=failures)


def _worker(rank, world, port, init, params, out_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1908_03869_b200 as sdb
        from paper_1908_03869_b200 import engine
        import bench
        engine.run_batch = _oracle_run_batch  # test-only device stand-in
        model = sdb.kuramoto_model(init.shape[1])
        cfg = sdb.EngineConfig(dt=0.5, tspan=4.0, ksteps=2, orbits=init.shape[0], seed=3,
                               stream="sfc64")

        def gather(obj):
            parts = [None] * world
            dist.all_gather_object(parts, obj)
            return parts

        store = engine.run_batch_sharded(model, cfg, sdb.OrbitBatch(init=init, params=params),
                                         world=world, rank=rank, gather=gather)
        tmax = bench.reduce_max_cpu(dist, float(rank + 1))
        out_q.put((rank, store.values, [(f.orbit, f.chunk, f.step) for f in store.failures],
                   tmax))
    finally:
        dist.destroy_process_group()


def test_two_rank_shards_assemble_bitwise():
    from oracle import sdeb_oracle as O
    n, m = 6, 37
    init, params = O.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.03), 0.3, seed=4)
    params[5, 1 + 2] = 1e308  # orbit 5 overflows -> failure record, renumbered globally
    params[30, 1 + 4] = 1e308  # orbit 30 lands on rank 1
    params[[5, 30], 0] = 0.0
    params[[5, 30], n + 1:] = 0.0
    _, full, fails = O.integrate(init, params, dt=0.5, ksteps=2, chunks=4, seed=3,
                                 stream="sfc64")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, init, params, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, values, flist, tmax in results:
        assert np.array_equal(values, full, equal_nan=True)
        assert flist == [(f[0], f[1], f[2]) for f in fails]
        assert [f[0] for f in fails] == [5, 30]
        assert tmax == 2.0


def test_shard_bounds_cover_exactly_once():
    from paper_1908_03869_b200.engine import shard_bounds
    for m in (1, 7, 64, 65536, 1 << 20):
        for w in (1, 2, 3, 4, 8):
            spans = [shard_bounds(m, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
