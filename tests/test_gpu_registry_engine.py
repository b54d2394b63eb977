"""Registry in the serving loop: a 16-expert engine whose HBM
budget holds only 4 experts serves a router-assigned request stream.  Each batch acquires
(loads on demand, pins) its experts through ExpertRegistry and releases the previous
batch's; eviction is strict LRU over unpinned experts and waits for the decode stream's
fence.  Outputs must be bit-identical to an engine with all 16 experts resident (the
fused kernel's per-row results depend only on the padded row count, not on slots)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mini():
    from paper_2406_09041_b200.synth import MistralShape
    return MistralShape(hidden=256, intermediate=384, n_layers=2, n_heads=2, n_kv_heads=1, head_dim=128,
                        vocab=1000, rope_theta=10000.0)


def _engine(shape, seed=0):
    import torch
    from paper_2406_09041_b200.mistral import MistralMultiExpert
    eng = MistralMultiExpert(shape, max_batch=256, ctx_max=32, tune=False)
    eng.load_synthetic_base(seed=seed, std=0.06)
    return eng


def _route(domains, pick, n, rng):
    from paper_2406_09041_b200 import router as pr
    pools = {d: [f"{d}k{j}" for j in range(8)] for d in domains}
    r = pr.train_router([(" ".join(rng.choice(pools[d], size=6)), d) for d in domains for _ in range(10)], domains)
    truth = [pick[i % len(pick)] for i in range(n)]
    got = pr.DeviceRouter(r).classify_batch([" ".join(rng.choice(pools[d], size=5)) for d in truth])
    names = [g[0] for g in got]
    assert names == truth
    return names


def _run(eng, reqs, kv, ids):
    """One eager decode step for `reqs` (expert id per request) with per-request KV / ids."""
    import torch
    rows = eng.set_batch(reqs, [6] * len(reqs))
    R = eng.B
    idx = torch.as_tensor(np.maximum(rows, 0), device="cuda")
    real = torch.as_tensor(rows >= 0, device="cuda")
    for cache, src in ((eng.kcache, kv[0]), (eng.vcache, kv[1])):
        cache[:, :R] = torch.where(real[None, :, None, None, None], src[:, idx], torch.zeros_like(src[:, idx]))
    eng.ids[:R] = torch.where(real, ids[idx], torch.zeros_like(ids[idx]))
    eng.step()
    torch.cuda.synchronize()
    out_ids = eng.ids[:R].cpu().numpy()
    logits = eng.logits[:R, :eng.shape.vocab].float().cpu().numpy()
    order = np.argsort(np.where(rows >= 0, rows, 1 << 30))[:len(reqs)]
    return out_ids[order], logits[order]


def test_registry_budget_4_of_16_experts_bit_identical():
    import torch
    from paper_2406_09041_b200 import compress, synth
    from paper_2406_09041_b200.errors import BudgetExceededError
    shape = _mini()
    shapes = synth.mistral_expert_shapes(shape, shape.n_layers)
    names = [f"dom{i}" for i in range(16)]
    blobs = {n: synth.synthetic_expert_artifact(500 + i, shapes, n) for i, n in enumerate(names)}
    full = _engine(shape)
    for n in names:
        full.add_expert(n, compress.deserialize_artifact(blobs[n]))
    eng = _engine(shape)
    per = eng.expert_device_bytes(compress.deserialize_artifact(blobs[names[0]]))
    reg = eng.make_registry(4 * per, "synthetic")
    for n in names:
        ent = reg.register(n, blobs[n])
        assert ent.size_bytes == per  # device bytes, not artifact bytes
    assert reg.stats().current_bytes == 0

    rng = np.random.default_rng(1)
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    kv = (torch.randn((shape.n_layers, 64, 32, 1, 128), generator=g, device="cuda").to(torch.bfloat16),
          torch.randn((shape.n_layers, 64, 32, 1, 128), generator=g, device="cuda").to(torch.bfloat16))
    ids = torch.randint(0, shape.vocab, (64,), generator=g, device="cuda", dtype=torch.int32)
    peak_resident = 0
    for b in range(8):
        pick = list(rng.choice(names, size=4, replace=False))
        reqs = _route(names, pick, 12, rng)
        got_ids, got_logits = _run(eng, reqs, kv, ids)
        want_ids, want_logits = _run(full, reqs, kv, ids)
        assert np.array_equal(got_ids, want_ids), b
        assert np.array_equal(got_logits, want_logits), b
        st = reg.stats()
        assert st.current_bytes <= 4 * per
        assert set(pick) <= set(st.resident)
        assert all(st.resident[p][2] == 1 for p in pick)  # this batch's experts are pinned
        peak_resident = max(peak_resident, len(st.resident))
    st = reg.stats()
    assert st.evict_count > 0 and st.load_count > 4 and peak_resident <= 4
    assert st.peak_bytes <= 4 * per
    # a 5-expert batch cannot fit a 4-expert budget: the request fails, state unchanged
    with pytest.raises(BudgetExceededError):
        eng.set_batch(names[:5], [6] * 5)
    after = reg.stats()
    assert after.current_bytes <= 4 * per
    assert all(v[2] == 0 for v in after.resident.values())  # nothing left pinned by the failed batch


def test_decode_on_fresh_engine_equals_one_eager_step():
    """decode() (graph capture on first use) advances exactly one step (ADVICE: capture's
    warm-up step must not leak state)."""
    import torch
    from paper_2406_09041_b200 import compress, synth
    shape = _mini()
    shapes = synth.mistral_expert_shapes(shape, shape.n_layers)
    engs = []
    for _ in range(2):
        e = _engine(shape)
        for i in range(3):
            e.add_expert(f"e{i}", compress.deserialize_artifact(synth.synthetic_expert_artifact(40 + i, shapes, "d")))
        e.set_batch(["e0", "e1", "e2", "e1"], [5] * 4)
        e.fill_random_kv(5, seed=2)
        engs.append(e)
    R = engs[0].B
    start = (torch.arange(R, dtype=torch.int32) * 11 % shape.vocab)
    engs[0].ids[:R] = start.cuda()
    engs[0].step()
    torch.cuda.synchronize()
    eager = engs[0].ids[:R].cpu()
    out = engs[1].decode(start.pin_memory(), torch.zeros(R, dtype=torch.int32).pin_memory())
    assert torch.equal(out.cpu(), eager)
    assert torch.equal(engs[1].pos[:R].cpu(), engs[0].pos[:R].cpu())


def test_cache_window_error_instead_of_wrap():
    import torch
    from paper_2406_09041_b200 import compress, synth
    from paper_2406_09041_b200.mistral import CacheWindowError
    shape = _mini()
    eng = _engine(shape)
    shapes = synth.mistral_expert_shapes(shape, shape.n_layers)
    eng.add_expert("e0", compress.deserialize_artifact(synth.synthetic_expert_artifact(9, shapes, "d")))
    eng.set_batch(["e0"], [30])
    R = eng.B
    hin = torch.zeros(R, dtype=torch.int32).pin_memory()
    hout = torch.zeros(R, dtype=torch.int32).pin_memory()
    eng.decode(hin, hout)  # position 30
    eng.decode(hin, hout)  # position 31 = ctx_max - 1
    with pytest.raises(CacheWindowError):
        eng.decode(hin, hout)
