"""f3 step-size distillation on the GPU: the per-layer kernels bit-exact with the oracle
(itself pinned to the reference, tests/test_distill_cpu.py), the whole loop within f32
tolerance of the reference's own run (tests/golden/distill.npz)."""

import ctypes as C
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import distill as od
from oracle.compress import quantize_codes
from oracle.mesw import pack_codes, unpack_codes

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def _s(torch):
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("bits", [1, 2, 4])
def test_ste_grad_kernel_known_answers(bits):
    torch = _torch()
    from paper_2406_09041_b200 import _lib
    z = np.load(os.path.join(GOLDEN, "distill.npz"))
    x, st, up = (torch.from_numpy(z[k]).cuda() for k in ("ste_x", "ste_steps", "ste_up"))
    g = torch.empty(x.shape[1], dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().mesw_ste_step_grad(x.data_ptr(), x.shape[0], x.shape[1], st.data_ptr(), bits, None,
                                             up.data_ptr(), g.data_ptr(), _s(torch)))
    assert np.array_equal(g.cpu().numpy(), z[f"ste_grad_b{bits}"])


def test_reconstruct_grad_adam_pack_match_oracle():
    torch = _torch()
    from paper_2406_09041_b200 import _lib
    L = _lib.lib()
    rng = np.random.default_rng(5)
    m, n, k, bits = 300, 200, 6, 2
    delta = rng.normal(0, 0.02, size=(m, n)).astype(np.float32)
    base = rng.normal(0, 0.05, size=(m, n)).astype(np.float32)
    idx = np.sort(rng.choice(m, k, replace=False))
    rows = rng.normal(0, 0.05, size=(k, n)).astype(np.float16)
    steps = (np.abs(delta).max(axis=0) / 1.0).astype(np.float32)
    st = od.LayerState(delta, idx, rows.astype(np.float32), steps.copy(), bits)
    slot = np.full(m, -1, np.int32)
    slot[idx] = np.arange(k, dtype=np.int32)
    d_delta, d_base, d_steps = (torch.from_numpy(a).cuda() for a in (delta, base, steps))
    d_slot, d_rows = torch.from_numpy(slot).cuda(), torch.from_numpy(rows.astype(np.float32)).cuda()
    out = torch.empty_like(d_delta)
    _lib.check(L.mesw_ste_reconstruct(d_delta.data_ptr(), m, n, d_steps.data_ptr(), bits, d_slot.data_ptr(),
                                      d_rows.data_ptr(), d_base.data_ptr(), out.data_ptr(), _s(torch)))
    assert np.array_equal(out.cpu().numpy(), base + st.reconstruct())
    up = rng.normal(0, 1, size=(m, n)).astype(np.float32)
    g = torch.empty(n, dtype=torch.float32, device="cuda")
    _lib.check(L.mesw_ste_step_grad(d_delta.data_ptr(), m, n, d_steps.data_ptr(), bits, d_slot.data_ptr(),
                                    torch.from_numpy(up).cuda().data_ptr(), g.data_ptr(), _s(torch)))
    g_ref = st.step_gradient(up)
    assert np.array_equal(g.cpu().numpy(), g_ref)
    # three AdamW steps (f64 moments) on the device vs the oracle
    opt = od.Adam([n], lr=1e-3)
    dm, dv = torch.zeros(n, dtype=torch.float64, device="cuda"), torch.zeros(n, dtype=torch.float64, device="cuda")
    p_ref = steps.copy()
    for t in range(1, 4):
        gr = rng.normal(0, 1, size=n).astype(np.float32)
        gr[:3] = 0.0
        p_ref = np.maximum(opt.step([p_ref], [gr])[0], od.STEP_FLOOR).astype(np.float32)
        _lib.check(L.mesw_adam_step(d_steps.data_ptr(), dm.data_ptr(), dv.data_ptr(), torch.from_numpy(gr).cuda().data_ptr(),
                                    n, 1e-3, 0.9, 0.999, 1e-8, 1 - 0.9 ** t, 1 - 0.999 ** t, C.c_float(od.STEP_FLOOR),
                                    _s(torch)))
        assert np.array_equal(d_steps.cpu().numpy(), p_ref), t
        assert np.array_equal(dm.cpu().numpy(), opt.m[0]) and np.array_equal(dv.cpu().numpy(), opt.v[0])
    # _repack: codes of the trained steps, salient rows zero, packed like the reference
    mask = np.zeros(m, np.uint8)
    mask[idx] = 1
    packed = torch.empty(int(L.mesw_packed_nbytes(m, n, bits)), dtype=torch.uint8, device="cuda")
    _lib.check(L.mesw_quantize_pack(d_delta.data_ptr(), m, n, d_steps.data_ptr(), bits,
                                    torch.from_numpy(mask).cuda().data_ptr(), packed.data_ptr(), _s(torch)))
    codes = np.zeros((m, n), np.int8)
    keep = mask == 0
    codes[keep] = quantize_codes(delta[keep], p_ref, bits)
    assert packed.cpu().numpy().tobytes() == pack_codes(codes, bits)


def test_distill_matches_reference_run():
    torch = _torch()
    from paper_2406_09041_b200 import compress, distill
    from oracle.toylm import ToyWeights
    z = np.load(os.path.join(GOLDEN, "distill.npz"))
    zb = np.load(os.path.join(GOLDEN, "toy_base.npz"))
    depth = sum(1 for k in zb.files if k.startswith("layer"))
    base = ToyWeights(zb["embedding"], [zb[f"layer{i}"] for i in range(depth)], zb["head"])
    ft = ToyWeights(z["ft_embedding"], [z[f"ft_layer{i}"] for i in range(depth)], z["ft_head"])
    arts = []
    for l in range(depth + 2):
        m, n = base.weight_matrices()[l].shape
        idx = z[f"init_idx_{l}"]
        arts.append(compress.CompressedDelta(
            salient=compress.SalientSet(indices=idx, k=idx.size), salient_rows=z[f"init_rows_{l}"],
            steps=z[f"init_steps_{l}"], packed=compress.PackedCodes(bits=2, rows=m, cols=n, data=b"")))
    seqs = [list(r) for r in z["seqs"]]
    cfg = distill.DistillConfig(epochs=int(z["epochs"]), lr=float(z["lr"]), batch_size=int(z["batch_size"]))
    res = distill.distill_step_sizes(base, ft, arts, seqs, cfg)
    rel = lambda a, b: abs(a - b) / abs(b)  # noqa: E731
    assert rel(res.initial_loss, float(z["initial_loss"])) < 1e-5
    assert rel(res.final_loss, float(z["final_loss"])) < 1e-4
    assert np.allclose(res.batch_losses, z["batch_losses"], rtol=1e-4, atol=0)
    n_updates = len(res.batch_losses)
    for l, layer in enumerate(res.layers):
        ref = z[f"steps_{l}"]
        # each AdamW update moves a step by at most ~lr: a gradient-sign flip from GEMM rounding
        # can cost at most 2 * lr per update
        assert np.max(np.abs(layer.steps - ref)) <= 2 * cfg.lr * n_updates, l
        assert np.mean(layer.steps == ref) > 0.9, l
        codes = unpack_codes(layer.packed.data, layer.rows, layer.cols, 2)
        assert np.mean(codes != z[f"codes_{l}"]) < 1e-3, l
