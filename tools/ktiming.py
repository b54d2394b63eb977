"""Per-CTA phase timing of one fused-linear launch (MESW_TIMING=1)."""
import ctypes as C, os, sys
os.environ["MESW_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2406_09041_b200 import _lib
from paper_2406_09041_b200.device import LinearPlan, corr_table, pack_x
from kbench import make
L = _lib.lib()
L.mesw_debug_timing_copy.argtypes = [C.c_void_p, C.c_int]
m, n = int(sys.argv[1]), int(sys.argv[2])
E, rows = int(sys.argv[3]), int(sys.argv[4])
sets = [make(m, n, max(E, 1), r) for r in range(3)]  # rotate replicas: the timed launch is HBM-cold
if os.environ.get("ALIGNED"):  # B = rows tokens split evenly over E experts, serving-engine alignment
    from paper_2406_09041_b200.device import align_segments
    per = [rows // E + (1 if i < rows % E else 0) for i in range(E)]
    segs, cur = [], 0
    for e, c_ in enumerate(per):
        segs.append((cur, cur + c_, e))
        cur += c_
    rows, segs, _ = align_segments(rows, segs)
else:
    segs = [(16 * i, 16 * i + 3, i) for i in range(E)] if E else []
    rows = max(rows, 16 * (E - 1) + 3) if E else rows
x = torch.randn((rows, m), device="cuda").to(torch.bfloat16)
y = torch.empty((rows, n), dtype=torch.bfloat16, device="cuda")
corr = corr_table(rows, m, "cuda") if os.environ.get("EXACT") is None else None
xc = pack_x(x, corr=corr)
nobase = os.environ.get("NOBASE") is not None  # delta-only launches (no base weight)
CT = int(os.environ.get("CTAS", "0"))
plans = [LinearPlan(xc, rows, None if nobase else dw, table if E else None, segs, y, geom=geom, x_corr=corr, num_ctas=CT) for geom, dw, table in sets]
for i in range(6): plans[i % 3]()
torch.cuda.synchronize()
plans[0](); torch.cuda.synchronize()
G = min(CT or 148, (n // 128) * (m // 128))
G -= G % 2
buf = np.zeros(60 * 4096, np.uint64)
_lib.check(L.mesw_debug_timing_copy(buf.ctypes.data, G))
t = buf[:G * 8].reshape(G, 8).astype(np.int64)
prof = buf[4096 * 8:4096 * 8 + G * 16].reshape(G, 2, 8).astype(np.int64)
prof3 = buf[4096 * 48:4096 * 48 + G * 8].reshape(G, 8).astype(np.int64)
dprof = buf[4096 * 24:4096 * 24 + G * 16].reshape(G, 2, 8).astype(np.int64)
t0 = t[:, 0].min()
names = ["start", "all_synced", "fin_fenced", "mma_done", "red_done", "last_accfull", "last_tmem", "last_end"]
print(f"m={m} n={n} E={E} rows={rows}  (us from first CTA start)")
for i, nm in enumerate(names):
    v = (t[:, i] - t0) / 1e3
    v = v[t[:, i] > 0]
    if v.size:
        print(f"  {nm:12s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f}")

# per-CTA phase durations (us): differences within one CTA, so clock skew between SMs cancels
pairs = [("start->mma_done", 0, 3), ("mma_done->accfull", 3, 5), ("accfull->tmem", 5, 6), ("tmem->epi_end", 6, 7),
         ("epi_end->synced", 7, 1), ("synced->fin", 1, 2), ("fin->red_done", 2, 4)]
for nm, a_, b_ in pairs:
    ok = (t[:, a_] > 0) & (t[:, b_] > 0)
    if ok.any():
        d = (t[ok, b_] - t[ok, a_]) / 1e3
        print(f"  {nm:18s} med {np.median(d):7.2f}  min {d.min():7.2f}  max {d.max():7.2f}  n={ok.sum()}")
t2 = buf[4096:4096 + G * 8].reshape(G, 8).astype(np.int64)
print("  tail (bank 2, per-CTA us):")
flag = t2[:, 7]
print("    epilogue done when thread 0 passed the final barrier:", int((flag == 1001).sum()), "of", int((flag >= 1000).sum()))
print("  tail (bank 2: SM clock cycles, per CTA):")
for nm, a_, b_ in [("atomic", 0, 1), ("atomic->synced(epi)", 1, 2), ("synced->copies_landed", 2, 3),
                   ("copies->summed", 3, 4), ("summed->reduced", 4, 5), ("cluster_sync", 5, 6),
                   ("summed->pass1 (MESW_EXP_WARM)", 4, 7), ("pass1->reduced", 7, 5)]:
    ok = (t2[:, a_] > 0) & (t2[:, b_] > 0)
    if ok.any():
        d = (t2[ok, b_] - t2[ok, a_])
        print(f"    {nm:26s} med {np.median(d):9.0f}  min {d.min():9.0f}  max {d.max():9.0f}  n={ok.sum()}")
pm = ["wait_x", "wait_w", "base_issue", "wait_afull", "delta_issue", "unit_sum", "total", "jobs"]
pd = ["wait_cfull", "wait_aempty", "dequant+st", "wait_st+arrive", "-", "-", "total", "jobs"]
lead = prof[0::2, 0, :]
print("  mma   ", " ".join(f"{pm[i]}={np.median(lead[:, i]):.0f}" for i in range(8)))
print("  mma2  ", " ".join(f"{pm[i]}={np.median(prof[0::2, 1, i]):.0f}" for i in range(8)))
print("  mma3  ", " ".join(f"{pm[i]}={np.median(prof3[0::2, i]):.0f}" for i in range(8)))
for g in range(2):
    for r, nm in ((0, "lead"), (1, "peer")):
        print(f"  deq{g} {nm}", " ".join(f"{pd[i]}={np.median(dprof[r::2, g, i]):.0f}" for i in range(8) if pd[i] != "-"))
eprof = buf[4096 * 40:4096 * 40 + G * 16].reshape(G, 16).astype(np.int64)
sel = eprof[:, 2] > 0
if sel.any():
  print("  final red (cycles):", " ".join(f"{n}={np.median(eprof[sel, i]):.0f}/{np.max(eprof[sel, i]):.0f}" for i, n in enumerate(["prefetch_issue", "stage_wait", "reduce+store", "ncontrib"])), f"n={sel.sum()}")
tl = buf[4096 * 56:4096 * 56 + 260].astype(np.int64)
t0c = tl[256]
if t0c:
    for nm, off in (("issuer0 unit ends", 0), ("issuer1 unit ends", 64), ("deq grp0 chunk ends", 128), ("deq grp1 chunk ends", 192)):
        v = tl[off:off + 64]
        v = v[v > 0]
        if v.size:
            print(f"  {nm:22s}", " ".join(f"{(x - t0c):6d}" for x in v[:30]))
jb = buf[4096 * 56 + 512:4096 * 56 + 1024].astype(np.int64)
if t0c:
    for r in range(3):
        v = jb[r * 64:r * 64 + 64].reshape(32, 2)
        v = v[v[:, 0] > 0]
        if v.size:
            print(f"  issuer{r} jobs (afull-ready, committed):", " ".join(f"{a - t0c}/{b - a}" for a, b in v[:16]))
    for g in range(2):
        v = jb[256 + g * 128:256 + g * 128 + 128].reshape(32, 4)
        v = v[v[:, 0] > 0]
        if v.size:
            print(f"  deq{g} jobs (start, +slot, +stored, +arrived):",
                  " ".join(f"{a - t0c}/{b - a}/{c - b}/{d - c}" for a, b, c, d in v[:14]))
fs = buf[4096 * 12:4096 * 12 + G * 8].reshape(G, 8).astype(np.int64)
t4 = t2[:, 4]
ok = (t4 > 0) & (fs[:, 1] > 0) & (fs[:, 2] > 0)
if ok.any():
    print("  final reduce, thread 0 (cycles): summed->chunk_sum", int(np.median(fs[ok, 1] - t4[ok])),
          " chunk_sum->outputs", int(np.median(fs[ok, 2] - fs[ok, 1])), " outputs->reduced", int(np.median(t2[ok, 5] - fs[ok, 2])))
