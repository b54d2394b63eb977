"""Expert registry host logic vs the sequential LRU trace oracle.
The loader here is a stub (no GPU); the GPU load path is tests/test_gpu_registry.py."""
import json
import os
import random
import threading

import numpy as np
import pytest

from oracle.registry import replay
from paper_2406_09041_b200 import compress, synth
from paper_2406_09041_b200.errors import (BaseDigestMismatchError, BudgetExceededError, DuplicateExpertError,
                                          UnknownExpertError)
from paper_2406_09041_b200.registry import ExpertRegistry


def _blob(seed, n=64, domain="code"):
    return synth.synthetic_expert_artifact(seed, [(64, n)], domain)


def _size(blob):
    return compress.compressed_size_bytes(compress.deserialize_artifact(blob)).total


class Stub:
    def __init__(self):
        self.loaded, self.unloaded = [], []

    def load(self, eid, art):
        self.loaded.append(eid)
        return ("handle", eid)

    def unload(self, eid, handle):
        self.unloaded.append(eid)


def test_spec_examples():
    blobs = {e: _blob(i) for i, e in enumerate("ABCD")}
    sz = _size(blobs["A"])
    st = Stub()
    reg = ExpertRegistry(2 * sz, "synthetic", loader=st.load, unloader=st.unload)
    for e, b in blobs.items():
        ent = reg.register(e, b)
        assert ent.size_bytes == sz  # size metadata = compressed_size_bytes
    assert reg.stats().current_bytes == 0  # registered, nothing resident
    for e in "AB":
        reg.acquire(e)
        reg.release(e)
    reg.acquire("C")  # budget = 2 artifacts: C evicts A (LRU)
    assert st.unloaded == ["A"] and sorted(reg.stats().resident) == ["B", "C"]
    n = reg.stats().load_count
    reg.acquire("B")  # resident: no load
    assert reg.stats().load_count == n
    with pytest.raises(BudgetExceededError):  # B, C pinned: nothing evictable
        reg.acquire("D")
    s = reg.stats()
    assert s.peak_bytes == 2 * sz and s.current_bytes == 2 * sz
    with pytest.raises(DuplicateExpertError):
        reg.register("A", blobs["A"])
    with pytest.raises(UnknownExpertError):
        reg.acquire("Z")
    with pytest.raises(BaseDigestMismatchError):
        ExpertRegistry(2 * sz, "other-base").register("A", blobs["A"])


def test_lru_matches_trace_oracle():
    rng = random.Random(0)
    ids = [f"e{i}" for i in range(8)]
    blobs = {e: _blob(i, n=64 * (1 + i % 3)) for i, e in enumerate(ids)}
    sizes = {e: _size(b) for e, b in blobs.items()}
    budget = 3 * max(sizes.values())
    ops = [("register", e, sizes[e]) for e in ids]
    held = []
    for _ in range(400):
        if held and rng.random() < 0.45:
            e = held.pop(rng.randrange(len(held)))
            ops.append(("release", e))
        else:
            e = rng.choice(ids)
            ops.append(("acquire", e))
            held.append(e)
    want, orc = replay(budget, ops)
    st = Stub()
    reg = ExpertRegistry(budget, "synthetic", loader=st.load, unloader=st.unload)
    for op, w in zip(ops, want):
        if op[0] == "register":
            reg.register(op[1], blobs[op[1]])
        elif op[0] == "acquire":
            before = list(st.unloaded)
            if w[0] == "error":
                with pytest.raises(BudgetExceededError):
                    reg.acquire(op[1])
            else:
                reg.acquire(op[1])
                if w[0] == "load":
                    assert tuple(st.unloaded[len(before):]) == w[1]  # same LRU victims, same order
                else:
                    assert st.unloaded == before
        else:
            if w[0] == "ok":
                reg.release(op[1])
            else:
                with pytest.raises(UnknownExpertError):
                    reg.release(op[1])
        assert reg.stats().current_bytes <= budget
    s = reg.stats()
    assert (s.current_bytes, s.peak_bytes, s.load_count, s.evict_count) == (orc.current, orc.peak, orc.loads, orc.evicts)


def test_concurrent_stress_budget_safety():
    ids = [f"e{i}" for i in range(12)]
    blobs = {e: _blob(i) for i, e in enumerate(ids)}
    budget = 4 * _size(blobs[ids[0]])
    reg = ExpertRegistry(budget, "synthetic", loader=lambda e, a: e)
    for e in ids:
        reg.register(e, blobs[e])
    errors = []

    def worker(seed):
        r = random.Random(seed)
        for _ in range(1250):
            e = r.choice(ids)
            try:
                reg.acquire(e)
            except BudgetExceededError:
                continue
            assert reg.stats().current_bytes <= budget
            reg.release(e)

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    s = reg.stats()
    assert s.current_bytes <= budget and all(p == 0 for _, _, p in s.resident.values())


def test_from_root(tmp_path):
    blobs = {e: _blob(i) for i, e in enumerate(["math", "code"])}
    for e, b in blobs.items():
        (tmp_path / f"{e}.mesw").write_bytes(b)
    man = {"base_digest": "synthetic", "experts": [{"id": e, "domain": "d", "size_bytes": _size(b)}
                                                   for e, b in blobs.items()]}
    (tmp_path / "registry.json").write_text(json.dumps(man))
    reg = ExpertRegistry.from_root(str(tmp_path), 10 * _size(blobs["math"]), loader=lambda e, a: e)
    assert reg.acquire("code") == "code"


def test_eviction_waits_for_release_fence_and_size_fn():
    """release(eid, stream) records the consumer fence on the handle; eviction calls
    wait_idle() on the victim BEFORE the unloader frees it; size_fn sets the budget unit."""
    events = []

    class H:
        def __init__(self, eid):
            self.eid = eid

        def fence(self, stream=None):
            events.append(("fence", self.eid, stream))

        def wait_idle(self):
            events.append(("wait", self.eid))

    blobs = {e: _blob(i) for i, e in enumerate("ABC")}
    reg = ExpertRegistry(2000, "synthetic", loader=lambda e, a: H(e),
                         unloader=lambda e, h: events.append(("unload", e)), size_fn=lambda art: 1000)
    for e, b in blobs.items():
        assert reg.register(e, b).size_bytes == 1000
    reg.acquire("A")
    reg.release("A", "decode-stream")
    reg.acquire("B")
    reg.release("B", "decode-stream")
    reg.acquire("C")  # evicts A (LRU)
    assert events[:2] == [("fence", "A", "decode-stream"), ("fence", "B", "decode-stream")]
    assert events[2:] == [("wait", "A"), ("unload", "A")]
    assert reg.stats().current_bytes == 2000


def test_salient_index_out_of_range_rejected():
    """An artifact whose salient index is >= rows loads nowhere (the reference's reconstruct()
    raises IndexError, compress.py:119-120): the C ABI table builder rejects it."""
    import ctypes as C
    from paper_2406_09041_b200 import _lib
    from paper_2406_09041_b200.device import LinearGeometry, build_salient_tables
    from oracle import mesw as om
    rng = np.random.default_rng(0)
    ol = om.random_layer(rng, 64, 128, 2, 3)
    ol.salient_idx = np.array([5, 9, 64])  # 64 == rows: out of range
    art = compress.deserialize_artifact(om.serialize_artifact(
        {"model_id": "x", "domain": "d", "base_digest": "0", "layer_count": 1}, [ol]))
    with pytest.raises(IndexError):
        build_salient_tables(art.layers, LinearGeometry(64, (128,)))
