"""Parity at the BASELINE configs' real dimensions (hidden 4096, intermediate 14336, 32 q /
8 kv heads, vocab 32000): every fused linear of the sampled decoder layers and the lm_head,
checked against the f64 restatement on the identical bf16 inputs (oracle/parity.py), with
router-assigned experts and the serving engine's offset-code path.

* 3 experts (C2 shape, 2 layers): expert 0's layer-0 k projection is the block the
  REFERENCE's own compress_layer made (tests/golden/ref_kproj_4096x1024.mesw).
* 16 experts (C3 shape, 1 layer, B = 64): one fused launch per linear holds all 16 expert
  windows when the row budget allows it, else launch groups.

Tolerance (north_star): max rel err <= 1e-2 per linear; logits argmax agreement reported
and required >= 0.97 (first-maximum argmax over the engine's f32 logits vs f64 logits).
"""

import os

import numpy as np
import pytest

from oracle import mesw as om
from oracle.parity import LinearParity

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
TOL = 1e-2


def _router_batch(domains, B, seed):
    """Queries synthesised per domain (disjoint keyword pools), classified on the GPU (K4)."""
    from paper_2406_09041_b200 import router as pr
    rng = np.random.default_rng(seed)
    pools = {d: [f"{d}kw{i}" for i in range(12)] for d in domains}

    def query(d):
        return " ".join(rng.choice(pools[d], size=6))

    train = [(query(d), d) for d in domains for _ in range(20)]
    r = pr.train_router(train, domains)
    dev = pr.DeviceRouter(r)
    truth = [domains[i % len(domains)] for i in range(B)]
    rng.shuffle(truth)
    qs = [query(d) for d in truth]
    picked = [name for name, _, _ in dev.classify_batch(qs)]
    assert picked == truth  # separable pools: the router recovers every domain
    return picked


def _engine(n_layers, n_experts, B, ref_block: bool, seed=0):
    import torch
    from paper_2406_09041_b200 import compress, synth
    from paper_2406_09041_b200.mistral import MistralMultiExpert
    shape = synth.MistralShape()
    eng = MistralMultiExpert(shape, max_batch=B + 16 * n_experts, ctx_max=160, n_layers=n_layers)
    eng.load_synthetic_base(seed=seed)
    shapes = synth.mistral_expert_shapes(shape, n_layers)
    experts = {}
    names = [f"dom{e}" for e in range(n_experts)]
    for e, name in enumerate(names):
        blob = synth.synthetic_expert_artifact(1000 + e, shapes, name)
        man, layers = om.parse_artifact(blob)
        if ref_block and e == 0:  # layer-0 k_proj from the reference's own compress_layer
            with open(os.path.join(HERE, "golden", "ref_kproj_4096x1024.mesw"), "rb") as f:
                _, (ref_layer,) = om.parse_artifact(f.read())
            assert (ref_layer.m, ref_layer.n) == (layers[1].m, layers[1].n)
            layers[1] = ref_layer
            blob = om.serialize_artifact(man, layers)
        experts[name] = layers
        eng.add_expert(name, compress.deserialize_artifact(blob))
    reqs = _router_batch(names, B, seed + 11)
    eng.set_batch(reqs, [128] * B)
    eng.fill_random_kv(128, seed=seed + 7)
    g = torch.Generator(device="cuda")
    g.manual_seed(seed + 5)
    eng.ids[:eng.B] = torch.randint(0, shape.vocab, (eng.B,), generator=g, device="cuda", dtype=torch.int32)
    return eng, experts


@pytest.mark.parametrize("n_layers,n_experts,B,layers", [(2, 3, 32, (0, 1)), (1, 16, 64, (0,))])
def test_mistral_dims_per_linear_parity(n_layers, n_experts, B, layers):
    import torch
    eng, experts = _engine(n_layers, n_experts, B, ref_block=(n_experts == 3))
    chk = LinearParity(eng, experts, layers=layers, head=True)
    eng.step(trace=chk)
    torch.cuda.synchronize()
    s = chk.summary()
    kinds = {(r["kind"], r["layer"]) for r in s["per_linear"]}
    assert kinds == {(k, l) for l in layers for k in ("qkv", "o", "gu", "down")} | {("head", -1)}
    bad = [r for r in s["per_linear"] if not r["max_rel_err"] <= TOL]
    assert not bad, bad
    assert s["argmax_agree"] >= 0.97, s["argmax_agree"]
    print(f"\n{n_experts} experts, B={B}: max rel err {s['max_rel_err']:.2e} over {s['linears_checked']} "
          f"launches, argmax agreement {s['argmax_agree']:.3f}")


def test_reference_block_reconstruct_on_device():
    """The reference-made Mistral-shape block decodes bit-exactly on the device (K1/K6)
    and its fused delta product matches the reference's x @ reconstruct()."""
    import torch
    from paper_2406_09041_b200 import compress
    from paper_2406_09041_b200.device import DeviceDelta, ExpertTable, me_linear
    with open(os.path.join(HERE, "golden", "ref_kproj_4096x1024.mesw"), "rb") as f:
        art = compress.deserialize_artifact(f.read())
    _, (ol,) = om.parse_artifact(compress.serialize_artifact(art))
    d = DeviceDelta.from_blocks([art.layers[0]])
    assert np.array_equal(d.reconstruct().cpu().numpy(), ol.reconstruct())
    x = np.random.default_rng(7).normal(0, 1, size=(4, 4096)).astype(np.float32)
    want = np.load(os.path.join(HERE, "golden", "ref_kproj_y.npy"))
    t = ExpertTable("cuda")
    t.set(0, d)
    xb = torch.from_numpy(x).to(torch.bfloat16).cuda()
    y = me_linear(xb, None, t, [(0, 4, 0)], out_dtype=torch.float32, geom=d.geom).cpu().numpy()
    ref = om.delta_matvec_batch(xb.float().cpu().numpy(), ol)  # same bf16 inputs, f64
    assert np.max(np.abs(y - ref)) / np.max(np.abs(ref)) <= 1e-5
    # and the reference's own f32 product on the unrounded x, within bf16 input rounding
    assert np.max(np.abs(y - want)) / np.max(np.abs(want)) <= 1e-2
