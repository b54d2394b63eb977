"""Decode attention in isolation: B requests x 32 heads (8 kv heads), context lengths ~U(129, 256)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_09041_b200 import _lib  # noqa: E402

L = _lib.lib()
for B in (32, 128):
    n_heads, n_kv, D, ctx = 32, 8, 128, int(os.environ.get("CTX", 256))
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn((B, (n_heads + 2 * n_kv) * D), device="cuda", generator=g).to(torch.bfloat16)
    kc = torch.randn((B, ctx, n_kv, D), device="cuda", generator=g).to(torch.bfloat16)
    vc = torch.randn((B, ctx, n_kv, D), device="cuda", generator=g).to(torch.bfloat16)
    ln = torch.randint(ctx // 2 + 1, ctx + 1, (B,), device="cuda", dtype=torch.int32, generator=g)
    out = torch.empty((B, n_heads * D), device="cuda", dtype=torch.bfloat16)
    ws = torch.empty(int(L.mesw_attention_workspace_bytes(B, n_heads, ctx)), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()

    def run():
        _lib.check(L.mesw_attention_decode_rope(q.data_ptr(), q.stride(0), kc.data_ptr(), vc.data_ptr(), ln.data_ptr(),
                                                B, n_heads, n_kv, D, C.c_float(1e6), ctx, out.data_ptr(), out.stride(0),
                                                0, ws.data_ptr(), ws.numel(), None, 0, C.c_void_p(s.cuda_stream)))
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(100):
        run()
    en.record()
    torch.cuda.synchronize()
    us = st.elapsed_time(en) * 10
    kv = float(ln.sum()) * n_kv * D * 2 * 2
    print(f"B={B} ctx<={ctx}: {us:7.2f} us per call, KV {kv / 1e6:6.1f} MB -> {kv / us / 1e3:7.1f} GB/s", flush=True)
