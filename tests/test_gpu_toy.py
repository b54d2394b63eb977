"""Drop-in acceptance on the reference toy model: GPU providers plugged into the
reference's provider protocol (restated in oracle/toylm.py, since /root/reference
is absent on the GPU box) reproduce the reference's own forward / greedy decode
outputs stored in tests/golden (made from the real reference)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import toylm as ot

pytestmark = pytest.mark.gpu


def _base():
    zb = np.load(os.path.join(GOLDEN, "toy_base.npz"))
    return ot.ToyWeights(zb["embedding"], [zb[f"layer{i}"] for i in range(4)], zb["head"])


def test_gpu_providers_in_reference_forward_with_delta():
    from paper_2406_09041_b200 import compress
    from paper_2406_09041_b200.infer import GpuCompressedProvider
    base = _base()
    ze = np.load(os.path.join(GOLDEN, "toy_expected.npz"))
    for e in range(3):
        art = compress.load_artifact(os.path.join(GOLDEN, f"toy_expert_{e}.mesw"))
        provs = [GpuCompressedProvider(l) for l in art.layers]
        assert not isinstance(getattr(provs[0], "rows"), int)  # protocol trap (toylm.py:175)
        logits = ot.forward_with_delta(base, provs, ze["tokens"])
        ref = ze[f"fwd_delta_{e}"]
        assert np.max(np.abs(logits - ref)) <= 1e-4 * np.max(np.abs(ref))  # SPEC.md:373 (1e-4)
        assert ot.greedy_decode(base, ze["prompt"], 12, provs) == ze[f"greedy_{e}"].tolist()


def test_batched_multi_model_forward_gpu():
    from paper_2406_09041_b200 import compress
    from paper_2406_09041_b200.infer import BatchPlan, ExpertSet, ToyBase, batched_multi_model_forward
    base = _base()
    gbase = ToyBase(base.embedding, base.layers, base.head)
    experts = ExpertSet(gbase)
    arts = {}
    for e, name in enumerate(["instruct", "math", "code"]):
        arts[name] = compress.load_artifact(os.path.join(GOLDEN, f"toy_expert_{e}.mesw"))
        experts.add(name, arts[name])
    rng = np.random.default_rng(0)
    items = []
    for q in range(10):
        eid = ["instruct", "math", "code", "nope"][q % 4] if q != 9 else "math"
        items.append((f"q{q}", eid, rng.integers(0, 256, size=int(rng.integers(1, 9))).tolist()))
    out = batched_multi_model_forward(gbase, experts, BatchPlan.of(items))
    assert [o[0] for o in out] == [i[0] for i in items]
    ze = np.load(os.path.join(GOLDEN, "toy_expected.npz"))
    bf = lambda a: np.asarray(a, np.float32).astype(np.float32)  # noqa: E731
    for (qid, eid, toks), (rq, logits, err) in zip(items, out):
        if eid == "nope":
            assert logits is None and "unknown expert" in err
            continue
        assert err is None
        from oracle import mesw as om
        provs = [ot.DenseProvider(om.parse_artifact(compress.serialize_artifact(arts[eid]))[1][i].reconstruct())
                 for i in range(6)]
        ref = ot.forward_with_delta(base, provs, toks)
        # f32-accurate mode (bf16 hi/lo pairs): SPEC.md:438 tolerance 1e-4 vs per-query forward_with_delta
        assert np.max(np.abs(logits - ref)) <= 1e-4 * np.max(np.abs(ref)), qid
    # a batch of one equals the same query inside the batch (same math, regrouped f32 sums)
    single = batched_multi_model_forward(gbase, experts, BatchPlan.of([items[1]]))[0][1]
    assert np.max(np.abs(single - out[1][1])) <= 1e-6 * np.max(np.abs(single))
    # group order does not change any bit: the same batch with the expert groups permuted
    out2 = batched_multi_model_forward(gbase, experts, BatchPlan.of(items[::-1]))
    for a, b in zip(out, out2[::-1]):
        if a[1] is not None:
            assert np.array_equal(a[1], b[1])


def _reference_toylm():
    """The unmodified reference package installed by tools/install_reference.sh into
    baseline/_ref (git-ignored; it travels to the GPU box with the repo), or None."""
    import sys
    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "meswitch")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    from meswitch import toylm
    return toylm


def test_gpu_providers_in_the_reference_packages_own_forward():
    """The drop-in proper: the reference package's OWN toylm.forward_with_delta and
    greedy_decode (toylm.py:189-248) call the GPU providers through their protocol
    (matvec_batch / rows) and reproduce the reference-made golden outputs."""
    toylm = _reference_toylm()
    if toylm is None:
        pytest.skip("reference package not installed (tools/install_reference.sh)")
    from paper_2406_09041_b200 import compress
    from paper_2406_09041_b200.infer import GpuCompressedProvider
    zb = np.load(os.path.join(GOLDEN, "toy_base.npz"))
    layers = tuple(zb[f"layer{i}"] for i in range(4))
    model = toylm.ToyLM(vocab=zb["embedding"].shape[0], width=zb["embedding"].shape[1], depth=len(layers),
                        embedding=zb["embedding"], layers=layers, head=zb["head"])
    ze = np.load(os.path.join(GOLDEN, "toy_expected.npz"))
    for e in range(3):
        art = compress.load_artifact(os.path.join(GOLDEN, f"toy_expert_{e}.mesw"))
        provs = [GpuCompressedProvider(l) for l in art.layers]
        logits = toylm.forward_with_delta(model, provs, ze["tokens"])
        ref = ze[f"fwd_delta_{e}"]
        assert np.max(np.abs(logits - ref)) <= 1e-4 * np.max(np.abs(ref))  # SPEC.md:373 (1e-4)
        assert toylm.greedy_decode(model, ze["prompt"], 12, provs) == ze[f"greedy_{e}"].tolist()
