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


class _FakeEngine:
    """CPU stand-in with the serving engine's batch contract (MistralMultiExpert.set_batch:
    requests regrouped by expert on 16-row boundaries, rows[r] = request index or -1;
    decode(host_in, host_out) -> next ids).  Next id = f(expert, current id): a pure
    function, so the collected token streams are checkable per request."""

    def __init__(self, experts):
        self.slot = {e: i for i, e in enumerate(experts)}

    def set_batch(self, expert_ids, prompt_lens=None):
        rows = []
        for e in sorted(set(expert_ids), key=lambda e: self.slot[e]):
            while len(rows) % 16:
                rows.append(-1)
            rows.extend(i for i, x in enumerate(expert_ids) if x == e)
        self.rows = np.asarray(rows)
        self.B = len(rows)
        self.exp = [expert_ids[q] if q >= 0 else None for q in rows]
        return self.rows

    def decode(self, host_in, host_out):
        for r in range(self.B):
            e = self.exp[r]
            host_out[r] = 0 if e is None else (int(host_in[r]) * 7 + 13 * e + 1) % 1000
        return host_out


def _expected_stream(e, tok0, steps):
    out, t = [], tok0
    for _ in range(steps):
        t = (t * 7 + 13 * e + 1) % 1000
        out.append(t)
    return out


def _engine_worker(rank, ws, port, q):
    import torch
    import torch.distributed as dist
    import bench_mistral as bm
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
    try:
        n_exp, steps = 6, 4
        pl = Placement(n_exp, ws)
        reqs = [(100 + i, (3 * i + 1) % n_exp, None) for i in range(19)] if rank == 0 else None
        mine = []
        ShardedService(pl, rank, lambda lr: (mine.extend(lr), {})[1]).step(reqs)
        eng = _FakeEngine(pl.local_experts(rank))
        eng.set_batch([r[1] for r in mine])
        host_in = torch.zeros(max(eng.B, 1), dtype=torch.int32)
        for r, qi in enumerate(eng.rows):
            host_in[r] = 0 if qi < 0 else mine[qi][0]  # first token = request id
        host_out = torch.zeros_like(host_in)
        res = ShardedService(pl, rank, bm.make_serve(eng, steps, host_in, host_out)).step(reqs)
        if rank == 0:
            q.put(("res", res))
        q.put(("mine", rank, [r[0] for r in mine]))
    finally:
        dist.destroy_process_group()


def test_engine_serve_path_world_size_2():
    """bench_mistral.make_serve (the per-rank serve the benchmark's e2e runs) behind
    ShardedService over gloo: every request decoded on its owner rank, token streams
    returned to rank 0 in request order, none lost or duplicated."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_engine_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(3)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res = next(g[1] for g in got if g[0] == "res")
    mine = {g[1]: g[2] for g in got if g[0] == "mine"}
    assert sorted(mine[0] + mine[1]) == [100 + i for i in range(19)]
    for i in range(19):
        e = (3 * i + 1) % 6
        assert (100 + i) in mine[e % 2]
        assert res[100 + i] == _expected_stream(e, 100 + i, 4)
