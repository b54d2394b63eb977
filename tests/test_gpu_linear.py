"""GPU parity of the loader (K1), debug decoders (K6) and the fused multi-expert
linear (K2) against the oracle and the reference golden fixtures."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import mesw as om

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def _read(name):
    with open(os.path.join(GOLDEN, name), "rb") as f:
        return f.read()


def _layer_names():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        return json.load(f)["layers"]


def _art_layer(olayer):
    from paper_2406_09041_b200 import compress
    man = {"model_id": "t", "domain": "d", "base_digest": "0", "layer_count": 1}
    return compress.deserialize_artifact(om.serialize_artifact(man, [olayer])).layers[0]


def test_repack_and_unpack_bit_exact_on_reference_layers():
    from paper_2406_09041_b200 import compress
    from paper_2406_09041_b200.device import DeviceDelta
    z = np.load(os.path.join(GOLDEN, "layer_expected.npz"))
    for name in _layer_names():
        L = compress.load_artifact(os.path.join(GOLDEN, f"layer_{name}.mesw")).layers[0]
        d = DeviceDelta.from_blocks([L])
        codes = d.unpack_codes().cpu().numpy()
        ref = z[f"{name}_codes"].copy()
        ref[z[f"{name}_salient"]] = 0  # the reference writes salient codes as 0 (compress.py:205-214)
        assert np.array_equal(codes, ref), name
        # K6 dense reconstruction == reference reconstruct(), bit for bit
        rec = d.reconstruct().cpu().numpy()
        assert np.array_equal(rec, z[f"{name}_recon"]), name


@pytest.mark.parametrize("bits", [1, 2, 3, 4, 8])
def test_repack_random_codes_all_widths(bits):
    from paper_2406_09041_b200.device import DeviceDelta
    rng = np.random.default_rng(bits)
    for (m, n, k) in [(1, 1, 0), (129, 257, 3), (384, 130, 0), (256, 512, 8)]:
        k = 0 if bits == 1 else min(k, m)
        ol = om.random_layer(rng, m, n, bits, k)
        d = DeviceDelta.from_blocks([_art_layer(ol)])
        ref = ol.codes().copy()
        ref[ol.salient_idx] = 0
        assert np.array_equal(d.unpack_codes().cpu().numpy(), ref)
        assert np.array_equal(d.reconstruct().cpu().numpy(), ol.reconstruct())


def test_weight_repack_roundtrip():
    torch = _torch()
    from paper_2406_09041_b200.device import DeviceWeight
    g = torch.Generator().manual_seed(0)
    w = torch.randn(300, 200, generator=g).to(torch.bfloat16).cuda()
    dw = DeviceWeight.from_dense([w])
    assert torch.equal(dw.dense(), w)
    wt = torch.randn(130, 257, generator=g).to(torch.bfloat16).cuda()  # nn.Linear [out, in]
    dw2 = DeviceWeight.from_dense([wt], transposed=True)
    assert torch.equal(dw2.dense(), wt.t())


def test_provider_matches_reference_layers():
    """Delta-only fused kernel (hi/lo f32 split) vs reference x @ reconstruct() (1e-5)."""
    from paper_2406_09041_b200 import compress
    from paper_2406_09041_b200.infer import GpuCompressedProvider
    z = np.load(os.path.join(GOLDEN, "layer_expected.npz"))
    for name in _layer_names():
        L = compress.load_artifact(os.path.join(GOLDEN, f"layer_{name}.mesw")).layers[0]
        p = GpuCompressedProvider(L)
        y = p.matvec_batch(z[f"{name}_x"])
        ref = z[f"{name}_y"]
        err = np.max(np.abs(y - ref)) / max(np.max(np.abs(ref)), 1e-30)
        assert err <= 1e-5, (name, err)
        # rows(ids) is bit-exact with reconstruct()[ids]
        ids = np.array([0, 3, L.rows - 1])
        assert np.array_equal(p.rows(ids), z[f"{name}_recon"][ids])
        assert np.allclose(p.matvec(z[f"{name}_x"][0]), ref[0], rtol=1e-5, atol=1e-5 * np.abs(ref).max())


def _setup_linear(m, ns, n_experts, bits=2, k=8, seed=0, device="cuda"):
    torch = _torch()
    from paper_2406_09041_b200.device import DeviceDelta, DeviceWeight, ExpertTable, LinearGeometry
    rng = np.random.default_rng(seed)
    geom = LinearGeometry(m, tuple(ns))
    w_blocks = [rng.normal(0, 0.02, size=(m, n)).astype(np.float32) for n in ns]
    dw = DeviceWeight.empty(geom, device)
    for b, wb in enumerate(w_blocks):
        dw.load_block(b, torch.from_numpy(wb).to(device).to(torch.bfloat16))
    w_bf = [torch.from_numpy(wb).to(torch.bfloat16).to(torch.float32).numpy() for wb in w_blocks]
    table = ExpertTable(device)
    experts = []
    for e in range(n_experts):
        blocks = [om.random_layer(rng, m, n, bits, min(k, m) if bits != 1 else 0) for n in ns]
        experts.append(blocks)
        table.set(e, DeviceDelta.from_blocks([_art_layer(b) for b in blocks], geom, device))
    return geom, dw, w_bf, table, experts


def _oracle_linear(x_bf, w_bf, experts, segs, geom, B):
    """f64 oracle on the same bf16-rounded inputs: x.W + x.reconstruct_e."""
    n = geom.n
    y = np.zeros((B, n), np.float64)
    for b, cb in enumerate(geom.col_base):
        nb = geom.block_n[b]
        y[:, cb:cb + nb] = x_bf.astype(np.float64) @ w_bf[b].astype(np.float64)
    for (s0, s1, slot) in segs:
        for b, cb in enumerate(geom.col_base):
            nb = geom.block_n[b]
            y[s0:s1, cb:cb + nb] += om.delta_matvec_batch(x_bf[s0:s1], experts[slot][b])
    return y


def _rel(y, ref):
    return float(np.max(np.abs(y - ref)) / max(np.max(np.abs(ref)), 1e-30))


@pytest.mark.parametrize("B,segs,num_ctas", [
    (1, [(0, 1, 0)], 0),
    (5, [(0, 2, 1), (2, 5, 0)], 0),
    (8, [(0, 3, 0), (3, 6, 1), (6, 8, 2)], 0),
    (8, [(0, 3, 0), (3, 6, 1), (6, 8, 2)], 7),
    (13, [(0, 4, 2), (6, 13, 1)], 13),
    (32, [(0, 11, 0), (11, 22, 1), (22, 32, 2)], 0),
    (64, [(i * 4, i * 4 + 4, i % 3) for i in range(16)], 0),
    (20, [], 0),
])
def test_fused_linear_matches_oracle(B, segs, num_ctas):
    torch = _torch()
    from paper_2406_09041_b200.device import me_linear
    geom, dw, w_bf, table, experts = _setup_linear(384, (256, 128), 3, seed=B)
    rng = np.random.default_rng(100 + B)
    x = torch.from_numpy(rng.normal(0, 1, size=(B, geom.m_pad)).astype(np.float32)).to(torch.bfloat16).cuda()
    ref = _oracle_linear(x.float().cpu().numpy()[:, :geom.m], w_bf, experts, segs, geom, B)
    res = torch.from_numpy(rng.normal(0, 1, size=(B, geom.n)).astype(np.float32)).to(torch.bfloat16).cuda()
    ys = []
    for offset in (False, True):  # exact q expansion / offset form + bias table (mesw.h x_corr)
        y = me_linear(x, dw, table, segs, out_dtype=torch.float32, num_ctas=num_ctas,
                      offset_codes=offset).cpu().numpy()
        assert _rel(y, ref) <= 2e-3
        ys.append(y)
        # bf16 output + residual epilogue
        y2 = me_linear(x, dw, table, segs, residual=res, num_ctas=num_ctas, offset_codes=offset).float().cpu().numpy()
        assert _rel(y2, ref + res.float().cpu().numpy()) <= 1e-2
    assert _rel(ys[1], ys[0]) <= 1e-5  # the bias removal costs only f32 rounding


@pytest.mark.parametrize("bits", [1, 3, 4, 8])
def test_fused_linear_other_widths(bits):
    torch = _torch()
    from paper_2406_09041_b200.device import me_linear
    geom, dw, w_bf, table, experts = _setup_linear(256, (384,), 2, bits=bits, k=4, seed=bits)
    rng = np.random.default_rng(bits)
    B, segs = 9, [(0, 4, 1), (4, 9, 0)]
    x = torch.from_numpy(rng.normal(0, 1, size=(B, geom.m_pad)).astype(np.float32)).to(torch.bfloat16).cuda()
    y = me_linear(x, dw, table, segs, out_dtype=torch.float32).cpu().numpy()
    ref = _oracle_linear(x.float().cpu().numpy()[:, :geom.m], w_bf, experts, segs, geom, B)
    assert _rel(y, ref) <= 2e-3


def _grouped(expert_of, perm):
    order = np.concatenate([np.flatnonzero(expert_of == e) for e in perm])
    segs, cur = [], 0
    for e in perm:
        cnt = int((expert_of == e).sum())
        if cnt:
            segs.append((cur, cur + cnt, e))
        cur += cnt
    return order, segs


@pytest.mark.parametrize("B", [7, 16, 24, 64])
def test_group_order_invariance_bitwise(B):
    """per-query results do not depend on the order in which expert
    groups are laid out in the batch -- exact equality."""
    torch = _torch()
    from paper_2406_09041_b200.device import me_linear
    geom, dw, w_bf, table, experts = _setup_linear(512, (384,), 3, seed=11)
    rng = np.random.default_rng(B)
    X = torch.from_numpy(rng.normal(0, 1, size=(B, geom.m_pad)).astype(np.float32)).to(torch.bfloat16).cuda()
    expert_of = rng.integers(0, 3, size=B)
    results = []
    for perm in ([0, 1, 2], [2, 0, 1], [1, 2, 0]):
        order, segs = _grouped(expert_of, perm)
        y = me_linear(X[torch.from_numpy(order).cuda()].contiguous(), dw, table, segs,
                      out_dtype=torch.float32).cpu().numpy()
        back = np.empty_like(y)
        back[order] = y
        results.append(back)
    assert np.array_equal(results[0], results[1]) and np.array_equal(results[0], results[2])


def test_batch_of_one_and_same_expert_pairs_bitwise():
    """SPEC.md:438 examples: a batch of one equals a single call; two queries of the same
    expert equal two single calls (exact).  Across token-tile classes (B<=8, <=16, <=32,
    <=64) the k-reduction is regrouped, so results agree to f32 reassociation only."""
    torch = _torch()
    from paper_2406_09041_b200.device import me_linear
    geom, dw, w_bf, table, experts = _setup_linear(512, (384,), 3, seed=12)
    rng = np.random.default_rng(1)
    X = torch.from_numpy(rng.normal(0, 1, size=(8, geom.m_pad)).astype(np.float32)).to(torch.bfloat16).cuda()
    y_pair = me_linear(X[:2].contiguous(), dw, table, [(0, 2, 1)], out_dtype=torch.float32).cpu().numpy()
    for i in range(2):
        y1 = me_linear(X[i:i + 1].contiguous(), dw, table, [(0, 1, 1)], out_dtype=torch.float32).cpu().numpy()
        assert np.array_equal(y1[0], y_pair[i])
    y8 = me_linear(X, dw, table, [(0, 3, 0), (3, 8, 1)], out_dtype=torch.float32).cpu().numpy()
    y1 = me_linear(X[4:5].contiguous(), dw, table, [(0, 1, 1)], out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(y1[0], y8[4])
    X32 = torch.cat([X] * 4).contiguous()
    y32 = me_linear(X32, dw, table, [(0, 3, 0), (3, 32, 1)], out_dtype=torch.float32).cpu().numpy()
    assert _rel(y32[4], y8[4]) <= 1e-6


def test_c1_shape_mixed_decode():
    """BASELINE config 1 shape: 4096x14336, 3 experts (2-bit, k=8), batch-8 mixed decode."""
    torch = _torch()
    from paper_2406_09041_b200.device import me_linear
    geom, dw, w_bf, table, experts = _setup_linear(4096, (14336,), 3, seed=1)
    rng = np.random.default_rng(7)
    x = torch.from_numpy(rng.normal(0, 1, size=(8, 4096)).astype(np.float32)).to(torch.bfloat16).cuda()
    # experts t mod 3 -> grouped order
    segs = [(0, 3, 0), (3, 6, 1), (6, 8, 2)]
    ref = _oracle_linear(x.float().cpu().numpy(), w_bf, experts, segs, geom, 8)
    # exact / offset-form codes, all SMs / the widths the tuner picks for this shape
    for offset, ctas in ((False, 0), (True, 0), (True, 142), (True, 112)):
        y = me_linear(x, dw, table, segs, out_dtype=torch.float32, offset_codes=offset,
                      num_ctas=ctas).cpu().numpy()
        assert _rel(y, ref) <= 2e-3, (offset, ctas)


def test_pack_x_roundtrip_and_layout():
    torch = _torch()
    from paper_2406_09041_b200.device import canonical_rows, pack_x, unpack_x
    g = torch.Generator().manual_seed(3)
    for B, m in [(1, 5), (7, 200), (16, 128), (37, 300)]:
        x = torch.randn(B, m, generator=g).to(torch.bfloat16).cuda()
        xc = pack_x(x)
        assert torch.equal(unpack_x(xc, B, m), x)
        NP = canonical_rows(B)
        flat = xc.cpu()
        t, k = B - 1, m - 1
        idx = ((k // 128) * NP * 128 + ((t // 8) % 2) * (NP // 2) * 128 + (t // 16) * 1024
               + ((k % 128) // 8) * 64 + (t % 8) * 8 + k % 8)
        assert flat[idx] == x[t, k].cpu()


def test_me_linear_caller_row_order_on_device():
    """Public me_linear with rows in arbitrary order (experts interleaved, base-only rows,
    residual): rows are grouped on the device (mesw_pack_x_gather) and results written back
    to the caller's rows by the epilogue (y_rows) -- bitwise equal to calling the kernel on
    pre-grouped rows, and the call issues only libmesw kernels."""
    import torch
    from paper_2406_09041_b200 import compress
    from paper_2406_09041_b200.device import DeviceDelta, DeviceWeight, ExpertTable, me_linear
    rng = np.random.default_rng(21)
    m, n = 256, 384
    W = rng.normal(0, 0.02, size=(m, n)).astype(np.float32)
    dw = DeviceWeight.from_dense([W])
    table = ExpertTable("cuda")
    man = {"model_id": "x", "domain": "d", "base_digest": "0", "layer_count": 1}
    for e in range(3):
        ol = om.random_layer(rng, m, n, 2, 8)
        table.set(e, DeviceDelta.from_blocks([compress.deserialize_artifact(om.serialize_artifact(man, [ol])).layers[0]]))
    B = 23
    x = torch.from_numpy(rng.normal(0, 1, size=(B, m)).astype(np.float32)).to(torch.bfloat16).cuda()
    res = torch.from_numpy(rng.normal(0, 1, size=(B, n)).astype(np.float32)).to(torch.bfloat16).cuda()
    segs = [(0, 5, 2), (5, 6, 0), (6, 17, 1)]  # rows 17..22: base only
    y1 = me_linear(x, dw, table, segs, residual=res, out_dtype=torch.float32)
    y2 = me_linear(x, dw, table, segs, residual=res, out_dtype=torch.float32)  # cached plan
    # reference launch: the same rows pre-grouped on 16-row boundaries, one segment per window
    order = list(range(0, 5)) + [-1] * 11 + [5] + [-1] * 15 + list(range(6, 17)) + [-1] * 5 + list(range(17, 23))
    xg = torch.zeros((len(order), m), dtype=torch.bfloat16, device="cuda")
    rg = torch.zeros((len(order), n), dtype=torch.bfloat16, device="cuda")
    for i, r in enumerate(order):
        if r >= 0:
            xg[i], rg[i] = x[r], res[r]
    yg = me_linear(xg, dw, table, [(0, 5, 2), (16, 17, 0), (32, 43, 1)], residual=rg, out_dtype=torch.float32)
    want = torch.stack([yg[order.index(r)] for r in range(B)])
    assert torch.equal(y1, want) and torch.equal(y2, want)
    # the same call captured once and replayed on new inputs (device.MeLinearGraph)
    from paper_2406_09041_b200.device import MeLinearGraph
    xs, ys = torch.zeros_like(x), torch.empty((B, n), dtype=torch.float32, device="cuda")
    rs = torch.zeros_like(res)
    g = MeLinearGraph(xs, dw, table, segs, ys, residual=rs)
    xs.copy_(x)
    rs.copy_(res)
    assert torch.equal(g(), want)
    x2 = torch.flip(x, [0]).contiguous()
    xs.copy_(x2)
    assert torch.equal(g(), me_linear(x2, dw, table, segs, residual=res, out_dtype=torch.float32))


def test_swiglu_epilogue_matches_swiglu_kernel():
    """The fused gate|up launch with the SwiGLU epilogue (mesw_linear_args.swiglu_I) writes
    the same act and bias table, bit for bit, as the plain launch followed by mesw_swiglu --
    for stream-K splits (all SMs) and whole column groups (narrow grid)."""
    import ctypes as C
    import torch
    from paper_2406_09041_b200 import _lib, compress
    from paper_2406_09041_b200.device import (DeviceDelta, DeviceWeight, ExpertTable, LinearGeometry, LinearPlan,
                                               canonical_numel, canonical_rows, corr_table, pack_x)
    L = _lib.lib()
    rng = np.random.default_rng(33)
    m, I, B = 256, 512, 21
    W = rng.normal(0, 0.05, size=(m, 2 * I)).astype(np.float32)
    geom = LinearGeometry(m, (2 * I,))
    dw = DeviceWeight.from_dense([W])
    table = ExpertTable("cuda")
    man = {"model_id": "x", "domain": "d", "base_digest": "0", "layer_count": 1}
    for e in range(2):
        ol = om.random_layer(rng, m, 2 * I, 2, 8)
        table.set(e, DeviceDelta.from_blocks([compress.deserialize_artifact(om.serialize_artifact(man, [ol])).layers[0]]))
    x = torch.from_numpy(rng.normal(0, 1, size=(B, m)).astype(np.float32)).to(torch.bfloat16).cuda()
    corr = corr_table(B, m, "cuda")
    xc = pack_x(x, corr=corr)
    segs = [(0, 5, 0), (8, 21, 1)]
    s = torch.cuda.current_stream()
    for ctas in (0, 8):
        gu1 = torch.empty((B, 2 * I), dtype=torch.bfloat16, device="cuda")
        gu2 = torch.empty_like(gu1)
        act1 = torch.zeros(canonical_numel(B, I), dtype=torch.bfloat16, device="cuda")
        act2 = torch.zeros_like(act1)
        c1, c2 = corr_table(B, I, "cuda"), corr_table(B, I, "cuda")
        LinearPlan(xc, B, dw, table, segs, gu1, geom=geom, x_corr=corr, num_ctas=ctas)()
        _lib.check(L.mesw_swiglu(gu1.data_ptr(), gu1.stride(0), B, I, act1.data_ptr(), 0, canonical_rows(B),
                                 c1.data_ptr(), c1.stride(0), C.c_void_p(s.cuda_stream)))
        for _ in range(2):  # second launch: the block counters reset themselves
            LinearPlan(xc, B, dw, table, segs, gu2, geom=geom, x_corr=corr, num_ctas=ctas,
                       swiglu=(I, act2, c2))()
        torch.cuda.synchronize()
        assert torch.equal(gu1, gu2)
        assert torch.equal(act1, act2)
        assert torch.equal(c1, c2)
