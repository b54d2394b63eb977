"""Expert-sharded serving host logic: placement e mod G, dispatch of
requests to owner ranks and collection of results, over a world_size-2 gloo group on CPU.
The per-rank "engine" here is the CPU oracle (test infrastructure); on the GPU box it is
the fused multi-expert decode."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2406_09041_b200.shard import Placement, ShardedService, partition

M, N, E = 64, 48, 5


def _experts():
    from oracle import mesw as om
    rng = np.random.default_rng(0)
    W = rng.normal(0, 0.02, size=(M, N)).astype(np.float32)
    layers = [om.random_layer(np.random.default_rng(10 + e), M, N, 2, 4) for e in range(E)]
    return W, layers


def _serve_oracle(W, layers):
    from oracle import mesw as om

    def serve(reqs):
        out = {}
        for rid, e, x in reqs:
            x = np.asarray(x, np.float32)[None, :]
            out[rid] = (x @ W + om.delta_matvec_batch(x, layers[e]))[0]
        return out
    return serve


def _requests():
    rng = np.random.default_rng(3)
    return [(i, int(rng.integers(0, E)), rng.normal(0, 1, M).astype(np.float32).tolist()) for i in range(23)]


def _worker(rank, ws, port, q):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
    try:
        W, layers = _experts()
        pl = Placement(E, ws)
        local = {e: layers[e] for e in pl.local_experts(rank)}
        served = []

        def serve(reqs):
            served.extend(r[0] for r in reqs)
            assert all(r[1] in local for r in reqs)  # only owned experts reach this rank
            return _serve_oracle(W, layers)(reqs)

        svc = ShardedService(pl, rank, serve)
        res = svc.step(_requests() if rank == 0 else None)
        if rank == 0:
            q.put(("results", {k: v.tolist() for k, v in res.items()}))
        q.put(("served", rank, served))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_placement_and_partition():
    pl = Placement(64, 8)
    assert [pl.owner(e) for e in (0, 7, 8, 63)] == [0, 7, 0, 7]
    assert pl.local_experts(3) == list(range(3, 64, 8))
    parts = partition([(i, i % 64, None) for i in range(200)], pl)
    assert sum(len(p) for p in parts) == 200
    assert all(pl.owner(r[1]) == k for k, p in enumerate(parts) for r in p)
    with pytest.raises(ValueError):
        pl.owner(64)


def test_sharded_service_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=120) for _ in range(3)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results = next(m[1] for m in msgs if m[0] == "results")
    served = {m[1]: m[2] for m in msgs if m[0] == "served"}
    reqs = _requests()
    pl = Placement(E, 2)
    # every request served exactly once, by its expert's owner
    assert sorted(served[0] + served[1]) == [r[0] for r in reqs]
    for rank, ids in served.items():
        assert all(pl.owner(reqs[i][1]) == rank for i in ids)
    # results equal a single-process run
    W, layers = _experts()
    ref = _serve_oracle(W, layers)(reqs)
    for rid, v in results.items():
        assert np.array_equal(np.asarray(v), np.asarray(ref[rid]))
