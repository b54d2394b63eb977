"""Decoder glue kernels (K5) vs numpy: split-context GQA decode attention."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("lens,G,ctx_max", [([1, 64, 65, 200], 4, 256), ([7, 130], 1, 192), ([256], 8, 256)])
def test_attention_decode_matches_numpy(lens, G, ctx_max):
    import torch
    from paper_2406_09041_b200 import _lib
    L = _lib.lib()
    B, n_kv, D = len(lens), 2, 128
    n_heads = G * n_kv
    rng = np.random.default_rng(sum(lens) + G)
    q = rng.normal(0, 1, size=(B, n_heads * D)).astype(np.float32)
    k = rng.normal(0, 1, size=(B, ctx_max, n_kv, D)).astype(np.float32)
    v = rng.normal(0, 1, size=(B, ctx_max, n_kv, D)).astype(np.float32)
    tq = torch.from_numpy(q).to(torch.bfloat16).cuda()
    tk = torch.from_numpy(k).to(torch.bfloat16).cuda()
    tv = torch.from_numpy(v).to(torch.bfloat16).cuda()
    tl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    out = torch.empty((B, n_heads * D), dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(int(L.mesw_attention_workspace_bytes(B, n_heads, ctx_max)), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    _lib.check(L.mesw_attention_decode(tq.data_ptr(), tq.stride(0), tk.data_ptr(), tv.data_ptr(), tl.data_ptr(), B,
                                       n_heads, n_kv, D, ctx_max, out.data_ptr(), out.stride(0), 0, ws.data_ptr(),
                                       ws.numel(), None, 0, C.c_void_p(s.cuda_stream)))
    got = out.float().cpu().numpy()
    qb, kb, vb = tq.float().cpu().numpy(), tk.float().cpu().numpy(), tv.float().cpu().numpy()
    ref = np.zeros_like(got)
    for b in range(B):
        n = lens[b]
        for h in range(n_heads):
            g = h // G
            sc = kb[b, :n, g, :] @ qb[b, h * D:(h + 1) * D] / np.sqrt(D)
            p = np.exp(sc - sc.max())
            ref[b, h * D:(h + 1) * D] = (p / p.sum()) @ vb[b, :n, g, :]
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-2
    with pytest.raises(ValueError):
        _lib.check(L.mesw_attention_decode(tq.data_ptr(), tq.stride(0), tk.data_ptr(), tv.data_ptr(), tl.data_ptr(),
                                           B, n_heads, n_kv, D, ctx_max, out.data_ptr(), out.stride(0), 0,
                                           ws.data_ptr(), 16, None, 0, C.c_void_p(s.cuda_stream)))


@pytest.mark.parametrize("lens,G,ctx_max", [([1, 64, 65, 200], 4, 256), ([7, 130, 128], 1, 192), ([256, 2], 8, 256)])
def test_attention_decode_rope_matches_two_call_form(lens, G, ctx_max):
    """The fused rope + KV append + attention launch is bit-identical to mesw_rope_append
    followed by mesw_attention_decode (output, bias table and both caches)."""
    import torch
    from paper_2406_09041_b200 import _lib
    L = _lib.lib()
    B, n_kv, D, theta = len(lens), 2, 128, 1e6
    n_heads = G * n_kv
    rng = np.random.default_rng(3 * sum(lens) + G)
    qkv = torch.from_numpy(rng.normal(0, 1, size=(B, (n_heads + 2 * n_kv) * D)).astype(np.float32)).to(
        torch.bfloat16).cuda()
    kc0 = torch.from_numpy(rng.normal(0, 1, size=(B, ctx_max, n_kv, D)).astype(np.float32)).to(torch.bfloat16).cuda()
    vc0 = torch.from_numpy(rng.normal(0, 1, size=(B, ctx_max, n_kv, D)).astype(np.float32)).to(torch.bfloat16).cuda()
    ln = torch.tensor(lens, dtype=torch.int32, device="cuda")
    pos = ln - 1
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    ws = torch.empty(int(L.mesw_attention_workspace_bytes(B, n_heads, ctx_max)), dtype=torch.uint8, device="cuda")
    outs = []
    for fused in (False, True):
        q, kc, vc = qkv.clone(), kc0.clone(), vc0.clone()
        out = torch.zeros((B, n_heads * D), dtype=torch.bfloat16, device="cuda")
        corr = torch.zeros((B, n_heads), dtype=torch.float32, device="cuda")
        if fused:
            _lib.check(L.mesw_attention_decode_rope(q.data_ptr(), q.stride(0), kc.data_ptr(), vc.data_ptr(),
                                                    ln.data_ptr(), B, n_heads, n_kv, D, C.c_float(theta), ctx_max,
                                                    out.data_ptr(), out.stride(0), 0, ws.data_ptr(), ws.numel(),
                                                    corr.data_ptr(), corr.stride(0), s))
            assert torch.equal(q, qkv)  # the fused form leaves the qkv row untouched
        else:
            _lib.check(L.mesw_rope_append(q.data_ptr(), q.stride(0), pos.data_ptr(), B, n_heads, n_kv, D,
                                          C.c_float(theta), kc.data_ptr(), vc.data_ptr(), ctx_max, s))
            _lib.check(L.mesw_attention_decode(q.data_ptr(), q.stride(0), kc.data_ptr(), vc.data_ptr(), ln.data_ptr(),
                                               B, n_heads, n_kv, D, ctx_max, out.data_ptr(), out.stride(0), 0,
                                               ws.data_ptr(), ws.numel(), corr.data_ptr(), corr.stride(0), s))
        torch.cuda.synchronize()
        outs.append((out, corr, kc, vc))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    # the new position was written, the rest of the caches untouched
    for b, n in enumerate(lens):
        assert torch.equal(outs[1][3][b, :n - 1], vc0[b, :n - 1])
        assert torch.equal(outs[1][3][b, n:], vc0[b, n:])
        assert not torch.equal(outs[1][2][b, n - 1], kc0[b, n - 1])


@pytest.mark.parametrize("V,is_bf16", [(32000, 1), (32003, 1), (1000, 0), (8, 1)])
def test_argmax_first_max(V, is_bf16):
    """mesw_argmax == np.argmax (ties -> lowest id, toylm.py:247) on the vectorised bf16 path,
    the scalar fallback (V % 8 != 0) and f32 logits; rows with planted ties."""
    import torch
    from paper_2406_09041_b200 import _lib
    L = _lib.lib()
    B = 5
    rng = np.random.default_rng(V)
    x = rng.integers(-40, 40, size=(B, V)).astype(np.float32) / 8  # exact in bf16, many ties
    x[1, :] = 0.0
    x[2, V // 3] = x[2, V - 1] = 100.0
    dt = torch.bfloat16 if is_bf16 else torch.float32
    t = torch.from_numpy(x).to(dt).cuda()
    out = torch.full((B,), -1, dtype=torch.int32, device="cuda")
    _lib.check(L.mesw_argmax(t.data_ptr(), is_bf16, B, V, t.stride(0), out.data_ptr(),
                             C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    assert out.cpu().numpy().tolist() == np.argmax(t.float().cpu().numpy(), axis=1).tolist()
