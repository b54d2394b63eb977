"""K3 prefill kernel (mesw_me_linear_prefill) vs the f64 restatement of Eq. 4 on identical bf16
inputs: y = x.W + x.Dtilde_e per 128-token expert group (compress.py:115-121 reconstruct,
SPEC.md:424-438).  The kernel folds Dtilde into the bf16 A operand (one extra rounding of
W + Dtilde per weight), so the bound is the north-star layer tolerance, max rel err <= 1e-2."""

import os

import numpy as np
import pytest

from oracle import mesw as om

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
TOL = 1e-2


def _bf(a):
    import torch
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)


def _setup(m, n, layers, seed=0):
    import torch
    from paper_2406_09041_b200 import compress
    from paper_2406_09041_b200.device import DeviceDelta, DeviceWeight, ExpertTable
    rng = np.random.default_rng(seed)
    W = rng.normal(0, 0.02, size=(m, n)).astype(np.float32)
    dw = DeviceWeight.from_dense([W])
    table = ExpertTable("cuda")
    man = {"model_id": "p", "domain": "d", "base_digest": "0", "layer_count": 1}
    for e, ol in enumerate(layers):
        art = compress.deserialize_artifact(om.serialize_artifact(man, [ol]))
        table.set(e, DeviceDelta.from_blocks([art.layers[0]]))
    return W, dw, table


def _ref(x, W, layers, slot_of_group, rows=None):
    xb, wb = _bf(x), _bf(W)
    rows = np.arange(x.shape[0]) if rows is None else rows
    y = xb[rows] @ wb
    for i, r in enumerate(rows):
        s = slot_of_group[r // 128]
        if s >= 0:
            y[i] += om.delta_matvec_batch(xb[r:r + 1], layers[s])[0]
    return y


def _rel(y, ref):
    return float(np.max(np.abs(y - ref)) / np.max(np.abs(ref)))


def test_prefill_small_with_reference_block_and_base_only_group():
    import torch
    from paper_2406_09041_b200.device import PrefillPlan, pack_x
    rng = np.random.default_rng(1)
    with open(os.path.join(HERE, "golden", "layer_l2_256x384_k8.mesw"), "rb") as f:
        _, (ref_layer,) = om.parse_artifact(f.read())  # made by the reference's compress_layer
    layers = [ref_layer, om.random_layer(rng, 256, 384, 2, 8, step_scale=3e-3),
              om.random_layer(rng, 256, 384, 2, 0, step_scale=3e-3)]
    W, dw, table = _setup(256, 384, layers)
    T = 512
    slots = [0, 1, -1, 2]
    x = rng.normal(0, 1, size=(T, 256)).astype(np.float32)
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    y = torch.empty((T, 384), dtype=torch.float32, device="cuda")
    PrefillPlan(pack_x(xt), T, T, dw, table, slots, y)()
    got = y.cpu().numpy()
    ref = _ref(x, W, layers, slots)
    err = _rel(got, ref)
    assert err <= TOL, err
    # base-only group: A = W exactly -> the plain bf16 GEMM (f32 accumulation)
    assert _rel(got[256:384], ref[256:384]) <= 1e-4
    # the delta is really applied: without it the error would be the delta's size
    base_only = _bf(x) @ _bf(W)
    assert _rel(got[:256], base_only[:256]) > 10 * _rel(got[:256], ref[:256])


def test_prefill_residual_bf16_out_and_unaligned_segments():
    import torch
    from paper_2406_09041_b200.device import me_linear_prefill
    rng = np.random.default_rng(2)
    layers = [om.random_layer(rng, 384, 512, 2, 8, step_scale=3e-3) for _ in range(3)]
    W, dw, table = _setup(384, 512, layers, seed=3)
    segs = [(0, 100, 2), (100, 357, 0), (357, 400, 1)]  # not 128-aligned: re-laid out by the host
    B = 410  # rows 400..409: base only
    x = rng.normal(0, 1, size=(B, 384)).astype(np.float32)
    res = rng.normal(0, 1, size=(B, 512)).astype(np.float32)
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    rt = torch.from_numpy(res).to(torch.bfloat16).cuda()
    y = me_linear_prefill(xt, dw, table, segs, residual=rt).float().cpu().numpy()
    xb, wb = _bf(x), _bf(W)
    ref = xb @ wb + _bf(res)
    for b, e, sl in segs:
        ref[b:e] += om.delta_matvec_batch(xb[b:e], layers[sl])
    assert _rel(y, ref) <= TOL


def test_prefill_mistral_c4_shape_sampled_rows():
    """BASELINE config 4 shape: 2048 tokens x 16 experts through a 4096x14336 linear; rows of
    the first, a middle and the last expert group checked against the f64 restatement."""
    import torch
    from paper_2406_09041_b200 import compress, synth
    from paper_2406_09041_b200.device import (DeviceDelta, DeviceWeight, ExpertTable, LinearGeometry, PrefillPlan,
                                               pack_x)
    m, n, T, E = 4096, 14336, 2048, 16
    g = torch.Generator(device="cuda").manual_seed(0)
    wt = (torch.randn((m, n), generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    dw = DeviceWeight.empty(LinearGeometry(m, (n,)))
    dw.load_block(0, wt)
    table = ExpertTable("cuda")
    layers = []
    for e in range(E):
        blob = synth.synthetic_expert_artifact(300 + e, [(m, n)], f"e{e}")
        table.set(e, DeviceDelta.from_blocks([compress.deserialize_artifact(blob).layers[0]]))
        if e in (0, 7, 15):
            _, (ol,) = om.parse_artifact(blob)
            layers.append((e, ol))
    x = torch.randn((T, m), generator=g, device="cuda").to(torch.bfloat16)
    y = torch.empty((T, n), dtype=torch.bfloat16, device="cuda")
    PrefillPlan(pack_x(x), T, T, dw, table, list(range(E)), y)()
    torch.cuda.synchronize()
    W = wt.float().cpu().numpy().astype(np.float64)
    xs = x.float().cpu().numpy().astype(np.float64)
    yh = y.float().cpu().numpy()
    for e, ol in layers:
        rows = np.arange(128 * e, 128 * e + 128, 16)  # 8 sampled rows of the group
        ref = xs[rows] @ W + om.delta_matvec_batch(xs[rows], ol)
        assert _rel(yh[rows], ref) <= TOL, e
