"""Offset-code bias tables (mesw.h mesw_linear_args.x_corr) written by pack_x and the
decoder glue, and the fused linear with them against the oracle."""

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2406_09041_b200 import _lib
from paper_2406_09041_b200.device import canonical_rows, corr_table, pack_x, unpack_x


def _w(m):
    k = np.arange(m)
    l = ((k % 64) // 2) % 8
    return np.where(np.isin(l, (0, 3, 6)), 130.0, np.where(np.isin(l, (1, 4, 7)), 34.0, 10.0))


def _ref_corr(x_bf16: torch.Tensor, NP: int) -> np.ndarray:
    x = x_bf16.float().cpu().numpy().astype(np.float64)
    B, m = x.shape
    n_ks = (m + 127) // 128
    xp = np.zeros((NP, n_ks * 128))
    xp[:B, :m] = x
    return (xp * _w(n_ks * 128)[None, :]).reshape(NP, n_ks, 128).sum(axis=2)


def _close(got: torch.Tensor, ref: np.ndarray):
    g = got.cpu().numpy().astype(np.float64)
    assert g.shape == ref.shape
    np.testing.assert_allclose(g, ref, rtol=1e-5, atol=1e-5 * max(1.0, np.abs(ref).max()))


@pytest.mark.parametrize("B,m", [(1, 128), (8, 4096), (21, 300), (48, 14336)])
def test_pack_x_corr(B, m):
    torch.manual_seed(B)
    x = torch.randn((B, m), device="cuda").to(torch.bfloat16)
    corr = corr_table(B, m, "cuda")
    corr.fill_(7.0)  # padding rows must be (re)written as 0
    pack_x(x, corr=corr)
    torch.cuda.synchronize()
    _close(corr, _ref_corr(x, canonical_rows(B)))


def test_glue_corr_tables():
    L = _lib.lib()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    torch.manual_seed(3)
    B, H, I = 19, 4096, 14336
    NP = canonical_rows(B)
    # rmsnorm -> canonical + corr
    x = torch.randn((B, H), device="cuda").to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn(H, device="cuda")).to(torch.bfloat16)
    yc = torch.zeros(NP * H, dtype=torch.bfloat16, device="cuda")
    corr = corr_table(B, H, "cuda")
    _lib.check(L.mesw_rmsnorm(x.data_ptr(), H, w.data_ptr(), B, H, C.c_float(1e-5), yc.data_ptr(), 0, NP,
                              corr.data_ptr(), corr.stride(0), s))
    _close(corr, _ref_corr(unpack_x(yc, B, H), NP))
    # swiglu -> canonical + corr
    gu = torch.randn((B, 2 * I), device="cuda").to(torch.bfloat16)
    ac = torch.zeros(NP * I, dtype=torch.bfloat16, device="cuda")
    corr = corr_table(B, I, "cuda")
    _lib.check(L.mesw_swiglu(gu.data_ptr(), 2 * I, B, I, ac.data_ptr(), 0, NP, corr.data_ptr(), corr.stride(0), s))
    act = unpack_x(ac, B, I)
    g, u = gu[:, :I].float(), gu[:, I:].float()
    ref_act = (torch.nn.functional.silu(g) * u)
    assert torch.allclose(act.float(), ref_act, rtol=1e-2, atol=1e-2)
    _close(corr, _ref_corr(act, NP))
    # attention merge -> canonical + corr (one head = one k-step)
    n_heads, n_kv, D, ctx = 32, 8, 128, 96
    q = torch.randn((B, (n_heads + 2 * n_kv) * D), device="cuda").to(torch.bfloat16)
    kc = torch.randn((B, ctx, n_kv, D), device="cuda").to(torch.bfloat16)
    vc = torch.randn((B, ctx, n_kv, D), device="cuda").to(torch.bfloat16)
    ln = torch.randint(1, ctx + 1, (B,), dtype=torch.int32, device="cuda")
    ws = torch.empty(int(L.mesw_attention_workspace_bytes(B, n_heads, ctx)), dtype=torch.uint8, device="cuda")
    oc = torch.zeros(NP * n_heads * D, dtype=torch.bfloat16, device="cuda")
    corr = corr_table(B, n_heads * D, "cuda")
    _lib.check(L.mesw_attention_decode(q.data_ptr(), q.stride(0), kc.data_ptr(), vc.data_ptr(), ln.data_ptr(), B,
                                       n_heads, n_kv, D, ctx, oc.data_ptr(), 0, NP, ws.data_ptr(), ws.numel(),
                                       corr.data_ptr(), corr.stride(0), s))
    _close(corr, _ref_corr(unpack_x(oc, B, n_heads * D), NP))
