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
