"""GPU-resident packed delta format, loader and the fused multi-expert linear call.

Everything here drives the C ABI (include/mesw.h) with device pointers owned by
torch tensors (torch is only the allocator/stream plumbing).  There is no CPU
path: every compute call launches a CUDA kernel from libmesw.so.

Layouts: a linear with m inputs and output blocks n_0, n_1, ...
(fused q|k|v or gate|up) is padded to m_pad = ceil128(m); block b starts at
output column col_base[b] (multiple of 128).  Each expert's linear owns
  codes    uint8 [m_pad * n_pad * DB / 8]   fragment-ordered DB-bit codes, d = q + OFF
  steps    f32   [n_pad]
  sal_off  int32 [n_pad/128 + 1], sal_idx int32 [*], sal_rows fp16 [*][128]
and the shared base owns a bf16 fragment-ordered weight [m_pad * n_pad].
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .compress import CompressedDelta

TILE = 128
MAX_ROWS = 192  # padded token rows per fused-linear launch (TMEM budget)


def _ceil(v: int, q: int = TILE) -> int:
    return (v + q - 1) // q * q


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


@dataclass(frozen=True)
class LinearGeometry:
    """Input width m and output blocks of a (possibly fused) linear."""

    m: int
    block_n: tuple

    @property
    def m_pad(self) -> int:
        return _ceil(self.m)

    @property
    def col_base(self) -> tuple:
        out, acc = [], 0
        for nb in self.block_n:
            out.append(acc)
            acc += _ceil(nb)
        return tuple(out)

    @property
    def n_pad(self) -> int:
        """Device columns: blocks padded to 128, total padded to 256 (the fused kernel's
        CTA pairs own two 128-column groups each)."""
        return _ceil(sum(_ceil(nb) for nb in self.block_n), 2 * TILE)

    @property
    def n(self) -> int:
        """Output width the kernel writes (up to the end of the last block)."""
        return self.col_base[-1] + self.block_n[-1]

    @property
    def n_cg(self) -> int:
        return self.n_pad // TILE


# --------------------------------------------------------------------------- deltas

@dataclass
class DeviceDelta:
    """One expert's compressed delta for one (fused) linear, resident in HBM."""

    geom: LinearGeometry
    bits: int
    code_bits: int
    codes: torch.Tensor
    steps: torch.Tensor
    sal_off: torch.Tensor
    sal_idx: torch.Tensor
    sal_rows: torch.Tensor
    nbytes: int = 0

    @classmethod
    def from_blocks(cls, blocks: list, geom: LinearGeometry | None = None, device="cuda",
                    stream=None, staging: list | None = None) -> "DeviceDelta":
        """Upload + repack MESW layer blocks (one per output block) into the device layout.

        Host bytes are staged in pinned buffers and copied asynchronously on `stream` (the
        registry's copy stream), where the K1 repack kernels run too.  With a stream, the
        pinned buffers are appended to `staging` and must stay alive until the stream has
        been synchronised (the caller does that once per expert); without one, the call
        synchronises the current stream itself."""
        L = _lib.lib()
        blocks = list(blocks)
        if geom is None:
            geom = LinearGeometry(blocks[0].rows, tuple(b.cols for b in blocks))
        if len(blocks) != len(geom.block_n):
            raise ValueError("block count does not match geometry")
        bits = blocks[0].bits
        for b, nb in zip(blocks, geom.block_n):
            if b.rows != geom.m or b.cols != nb:
                raise ValueError(f"block shape {(b.rows, b.cols)} != geometry {(geom.m, nb)}")
            if b.salient.k and int(np.asarray(b.salient.indices)[-1]) >= b.rows:
                # reference: reconstruct() indexes the dense delta with them (compress.py:119-120)
                raise IndexError(f"salient index {int(np.asarray(b.salient.indices)[-1])} out of range "
                                 f"for {b.rows} input channels")
            if b.bits != bits:
                raise NotImplementedError("mixed bit widths inside one fused linear")
        db = L.mesw_device_code_bits(bits)
        if db == 0:
            raise ValueError(f"bits must be one of (1, 2, 3, 4, 8), got {bits}")
        dev = torch.device(device)
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        stage = staging if staging is not None else []

        def h2d(host: torch.Tensor) -> torch.Tensor:  # pinned staging + async copy on `st`
            pinned = host.pin_memory()
            stage.append(pinned)
            return pinned.to(dev, non_blocking=True)

        m_pad, n_pad = geom.m_pad, geom.n_pad
        off, sidx, srows = build_salient_tables(blocks, geom)  # host; validates the salient indices
        with torch.cuda.stream(st):
            s = _stream(st)
            codes = torch.empty(int(L.mesw_codes_device_bytes(m_pad, n_pad, db)), dtype=torch.uint8, device=dev)
            steps_h = torch.zeros(n_pad, dtype=torch.float32)
            for b, cb in zip(blocks, geom.col_base):
                idx = h2d(torch.as_tensor(np.ascontiguousarray(b.salient.indices, dtype=np.int32)))
                raw = np.frombuffer(b.packed.data, dtype=np.uint8) if b.packed.data else np.zeros(1, np.uint8)
                packed = h2d(torch.from_numpy(raw.copy()))
                _lib.check(L.mesw_repack_codes(packed.data_ptr(), b.rows, b.cols, bits, idx.data_ptr(),
                                               b.salient.k, codes.data_ptr(), m_pad, n_pad, cb, s))
                steps_h[cb:cb + b.cols] = torch.from_numpy(np.ascontiguousarray(b.steps, np.float32))
            d = cls(geom=geom, bits=bits, code_bits=db, codes=codes, steps=h2d(steps_h),
                    sal_off=h2d(off), sal_idx=h2d(sidx), sal_rows=h2d(srows))
        d.nbytes = sum(t.numel() * t.element_size() for t in (d.codes, d.steps, d.sal_off, d.sal_idx, d.sal_rows))
        if stream is None:
            st.synchronize()
        return d

    @staticmethod
    def device_nbytes(blocks: list, geom: LinearGeometry | None = None) -> int:
        """HBM bytes `from_blocks(blocks, geom)` will occupy, computed on the host before
        loading (the registry charges its budget in these device bytes): codes, steps and
        the per-column-group salient tables."""
        L = _lib.lib()
        blocks = list(blocks)
        if geom is None:
            geom = LinearGeometry(blocks[0].rows, tuple(b.cols for b in blocks))
        db = L.mesw_device_code_bits(blocks[0].bits)
        rows = 0  # salient table rows: every column group of block b holds its k_b rows
        for b, cb in zip(blocks, geom.col_base):
            rows += b.salient.k * (_ceil(cb + b.cols) // TILE - cb // TILE)
        rows = max(rows, 1)
        return (int(L.mesw_codes_device_bytes(geom.m_pad, geom.n_pad, db)) + 4 * geom.n_pad
                + 4 * (geom.n_cg + 1) + 4 * rows + 2 * TILE * rows)

    def descriptor(self) -> tuple:
        return (self.codes.data_ptr(), self.steps.data_ptr(), self.sal_off.data_ptr(),
                self.sal_idx.data_ptr(), self.sal_rows.data_ptr())

    # ---- K6 debug views -------------------------------------------------------
    def unpack_codes(self, block: int = 0, stream=None) -> torch.Tensor:
        """int8 [m, n] codes of one block (reference orientation, salient rows read 0)."""
        L = _lib.lib()
        g = self.geom
        out = torch.empty((g.m, g.block_n[block]), dtype=torch.int8, device=self.codes.device)
        _lib.check(L.mesw_unpack_codes_debug(self.codes.data_ptr(), self.code_bits, g.m, g.block_n[block],
                                             g.m_pad, g.n_pad, g.col_base[block], out.data_ptr(),
                                             _stream(stream)))
        return out

    def reconstruct(self, block: int = 0, stream=None) -> torch.Tensor:
        """Dense f32 [m, n] = CompressedDelta.reconstruct() (compress.py:115-121), on the GPU."""
        L = _lib.lib()
        g = self.geom
        out = torch.empty((g.m, g.block_n[block]), dtype=torch.float32, device=self.codes.device)
        _lib.check(L.mesw_dequant_debug(self.codes.data_ptr(), self.code_bits, self.steps.data_ptr(),
                                        self.sal_off.data_ptr(), self.sal_idx.data_ptr(),
                                        self.sal_rows.data_ptr(), g.m, g.block_n[block], g.m_pad, g.n_pad,
                                        g.col_base[block], out.data_ptr(), _stream(stream)))
        return out


def build_salient_tables(blocks: list, geom: LinearGeometry):
    """Per-column-group salient tables (host C ABI helper) -> (off, idx, rows) CPU tensors."""
    L = _lib.lib()
    nb = len(blocks)
    U32 = C.c_uint32 * nb
    col_base = U32(*geom.col_base)
    ns = U32(*[b.cols for b in blocks])
    ks = U32(*[b.salient.k for b in blocks])
    idx_arrs = [np.ascontiguousarray(b.salient.indices, dtype=np.uint32) for b in blocks]
    row_arrs = [np.ascontiguousarray(np.asarray(b.salient_rows, np.float16).view(np.uint16)) for b in blocks]
    idx_ptrs = (C.c_void_p * nb)(*[a.ctypes.data if a.size else None for a in idx_arrs])
    row_ptrs = (C.c_void_p * nb)(*[a.ctypes.data if a.size else None for a in row_arrs])
    total = C.c_uint64()
    _lib.check(L.mesw_build_salient_tables(geom.m, nb, col_base, ns, ks, idx_ptrs, row_ptrs, geom.n_pad,
                                           None, None, None, C.byref(total)))
    off = np.zeros(geom.n_cg + 1, np.int32)
    sidx = np.zeros(max(total.value, 1), np.int32)
    srows = np.zeros((max(total.value, 1), TILE), np.uint16)
    _lib.check(L.mesw_build_salient_tables(geom.m, nb, col_base, ns, ks, idx_ptrs, row_ptrs, geom.n_pad,
                                           off.ctypes.data, sidx.ctypes.data, srows.ctypes.data,
                                           C.byref(total)))
    return torch.from_numpy(off), torch.from_numpy(sidx), torch.from_numpy(srows.view(np.int16))


# --------------------------------------------------------------------------- base weights

@dataclass
class DeviceWeight:
    """Shared base weight (bf16) of one (fused) linear in fragment layout."""

    geom: LinearGeometry
    frag: torch.Tensor

    @classmethod
    def empty(cls, geom: LinearGeometry, device="cuda") -> "DeviceWeight":
        L = _lib.lib()
        nel = int(L.mesw_weight_device_bytes(geom.m_pad, geom.n_pad)) // 2
        return cls(geom, torch.zeros(nel, dtype=torch.bfloat16, device=device))

    def load_block(self, block: int, w: torch.Tensor, transposed: bool = False, stream=None) -> None:
        """Write block `block` from a bf16 device matrix: [m, n] (reference orientation)
        or [n, m] if `transposed` (torch nn.Linear weight)."""
        L = _lib.lib()
        g = self.geom
        w = w.to(dtype=torch.bfloat16).contiguous()
        rows, cols = w.shape
        m, n = (cols, rows) if transposed else (rows, cols)
        if m != g.m or n != g.block_n[block]:
            raise ValueError(f"weight shape {tuple(w.shape)} does not match block {block}")
        _lib.check(L.mesw_repack_weight(w.data_ptr(), m, n, cols, 1 if transposed else 0, self.frag.data_ptr(),
                                        g.m_pad, g.n_pad, g.col_base[block], _stream(stream)))

    @classmethod
    def from_dense(cls, blocks: list, device="cuda", transposed: bool = False) -> "DeviceWeight":
        ts = [torch.as_tensor(b) for b in blocks]
        m = ts[0].shape[1] if transposed else ts[0].shape[0]
        ns = tuple(t.shape[0] if transposed else t.shape[1] for t in ts)
        dw = cls.empty(LinearGeometry(m, ns), device)
        for i, t in enumerate(ts):
            dw.load_block(i, t.to(device=device, dtype=torch.bfloat16), transposed)
        return dw

    def dense(self, block: int = 0, stream=None) -> torch.Tensor:
        L = _lib.lib()
        g = self.geom
        out = torch.empty((g.m, g.block_n[block]), dtype=torch.bfloat16, device=self.frag.device)
        _lib.check(L.mesw_unpack_weight_debug(self.frag.data_ptr(), g.m, g.block_n[block], g.m_pad, g.n_pad,
                                              g.col_base[block], out.data_ptr(), _stream(stream)))
        return out


# --------------------------------------------------------------------------- expert table

class ExpertTable:
    """Device array of mesw_expert_dev descriptors (one slot per resident expert)
    for one linear.  Slots are stable handles used in segment lists."""

    def __init__(self, device="cuda", capacity: int = 8):
        self.device = torch.device(device)
        self.host = np.zeros((capacity, 5), np.int64)
        self.dev = torch.zeros((capacity, 5), dtype=torch.int64, device=self.device)
        self.deltas: list = [None] * capacity
        self.code_bits = None

    def _grow(self, need: int):
        cap = self.host.shape[0]
        if need <= cap:
            return
        new = max(need, 2 * cap)
        h = np.zeros((new, 5), np.int64)
        h[:cap] = self.host
        self.host = h
        self.deltas += [None] * (new - cap)
        self.dev = torch.as_tensor(self.host).to(self.device)

    def set(self, slot: int, delta: DeviceDelta | None) -> None:
        self._grow(slot + 1)
        self.deltas[slot] = delta
        self.host[slot] = delta.descriptor() if delta is not None else 0
        self.dev[slot] = torch.as_tensor(self.host[slot]).to(self.device)
        if delta is not None:
            if self.code_bits not in (None, delta.code_bits):
                raise NotImplementedError("experts with different device code widths in one table")
            self.code_bits = delta.code_bits


# --------------------------------------------------------------------------- workspace

class Workspace:
    """Split-K partials + self-resetting column-group counters.  Launches that may run
    concurrently must not share one: `get(device, stream)` keys it by stream (launches on one
    stream are serialised, so they can)."""

    _per_device: dict = {}

    def __init__(self, device):
        L = _lib.lib()
        self.device = torch.device(device)
        idx = self.device.index if self.device.index is not None else torch.cuda.current_device()
        with torch.cuda.device(idx):
            self.sms = L.mesw_device_sm_count()
        self.nbytes = int(L.mesw_linear_workspace_bytes(MAX_ROWS, self.sms))
        self.ws = torch.empty(self.nbytes, dtype=torch.uint8, device=self.device)
        self.counters = torch.zeros(1 << 14, dtype=torch.int32, device=self.device)

    @classmethod
    def get(cls, device, stream=None) -> "Workspace":
        device = torch.device(device)
        idx = device.index if device.index is not None else torch.cuda.current_device()
        key = (idx, None if stream is None else int(stream.cuda_stream))
        if key not in cls._per_device:
            cls._per_device[key] = cls(torch.device("cuda", idx))
        return cls._per_device[key]


# --------------------------------------------------------------------------- K2 call

def canonical_rows(B: int) -> int:
    """Rows of the canonical activation layout: B padded to a multiple of 16."""
    return (B + 15) // 16 * 16


def canonical_numel(B: int, m: int) -> int:
    return _ceil(m) * canonical_rows(B)


def corr_table(B: int, m: int, device) -> torch.Tensor:
    """Zeroed offset-code bias table [canonical_rows(B), ceil(m/128)] f32 (mesw.h x_corr)."""
    return torch.zeros((canonical_rows(B), _ceil(m) // 128), dtype=torch.float32, device=device)


def pack_x(x: torch.Tensor, out: torch.Tensor | None = None, stream=None,
           corr: torch.Tensor | None = None) -> torch.Tensor:
    """Row-major bf16 [B, m] -> canonical tile layout (include/mesw.h, mesw_pack_x);
    optionally also the offset-code bias table `corr` (corr_table)."""
    if x.dtype != torch.bfloat16 or x.dim() != 2 or not x.is_cuda or x.stride(1) != 1:
        raise ValueError("x must be a row-contiguous 2-D bf16 CUDA tensor")
    B, m = x.shape
    if out is None:
        out = torch.empty(canonical_numel(B, m), dtype=torch.bfloat16, device=x.device)
    cp, cld = 0, 0
    if corr is not None:
        if corr.dtype != torch.float32 or not corr.is_contiguous() or tuple(corr.shape) != (canonical_rows(B), _ceil(m) // 128):
            raise ValueError("corr must be a contiguous f32 [canonical_rows(B), ceil(m/128)] tensor")
        cp, cld = corr.data_ptr(), corr.stride(0)
    _lib.check(_lib.lib().mesw_pack_x(x.data_ptr(), B, m, x.stride(0), out.data_ptr(), cp or None, cld,
                                      _stream(stream)))
    return out


def unpack_x(xc: torch.Tensor, B: int, m: int, stream=None) -> torch.Tensor:
    y = torch.empty((B, m), dtype=torch.bfloat16, device=xc.device)
    _lib.check(_lib.lib().mesw_unpack_x(xc.data_ptr(), B, m, y.data_ptr(), m, _stream(stream)))
    return y


class LinearPlan:
    """Pre-built launch of the fused multi-expert linear (pointers bound once).

    `xc` holds the B input rows in the canonical tile layout (pack_x / the decoder
    glue write it).  Calling the plan issues one `mesw_me_linear` on the current (or
    given) stream; this keeps per-launch host cost to one ctypes call and makes the
    launch capturable in a CUDA graph.
    """

    def __init__(self, xc: torch.Tensor, B: int, weight: DeviceWeight | None, table: ExpertTable | None,
                 segments, out: torch.Tensor, residual: torch.Tensor | None = None,
                 geom: LinearGeometry | None = None, num_ctas: int = 0, activation: str | None = None,
                 x_corr: torch.Tensor | None = None, stream=None, swiglu: tuple | None = None):
        """swiglu = (I, act, act_corr or None): the SwiGLU epilogue of mesw_linear_args (the
        engine's gate|up linear writes the down projection's canonical input itself)."""
        L = _lib.lib()
        if geom is None:
            geom = weight.geom if weight is not None else next(
                d.geom for d in table.deltas if d is not None)
        if xc.dtype != torch.bfloat16 or not xc.is_cuda or not xc.is_contiguous():
            raise ValueError("xc must be a contiguous bf16 CUDA tensor (canonical layout)")
        if xc.numel() < canonical_numel(B, geom.m):
            raise ValueError("xc too small for the canonical layout of B rows")
        if out.stride(1) != 1:
            raise ValueError("out must be row-contiguous")
        if out.dtype not in (torch.bfloat16, torch.float32):
            raise ValueError("output must be bf16 or f32")
        segs = [(int(b), int(e), int(s)) for b, e, s in segments]
        if any(b % 8 for b, _, _ in segs):
            raise ValueError("LinearPlan segments must start on 8-row boundaries (see align_segments)")
        if len(segs) > _lib.MAX_SEGMENTS:
            raise NotImplementedError(f"more than {_lib.MAX_SEGMENTS} expert segments in one launch")
        self.geom = geom
        self.keep = (xc, weight, table, out, residual, x_corr)  # keep buffers alive
        # the stream this plan is launched on (None: the default / engine stream); plans that
        # run concurrently on different streams get different split-K workspaces
        ws = Workspace.get(xc.device, stream)
        self.ws = ws
        a = _lib.LinearArgs()
        a.x = xc.data_ptr()
        a.B, a.m, a.n, a.x_layout = B, geom.m, geom.n, 0
        a.w = _ptr(weight.frag) if weight is not None else None
        a.expert_table = table.dev.data_ptr() if table is not None else None
        a.code_bits = table.code_bits if (table is not None and table.code_bits) else 2
        a.n_segments = len(segs)
        for i, (b, e, s) in enumerate(segs):
            a.seg_begin[i], a.seg_end[i], a.seg_slot[i] = b, e, s
        a.y = out.data_ptr()
        a.y_bf16 = 1 if out.dtype == torch.bfloat16 else 0
        a.ldy = out.stride(0)
        if residual is not None:
            if residual.dtype != torch.bfloat16:
                raise ValueError("residual must be bf16")
            a.residual, a.ld_res = residual.data_ptr(), residual.stride(0)
        a.workspace, a.workspace_bytes = ws.ws.data_ptr(), ws.nbytes
        a.counters = ws.counters.data_ptr()
        a.num_ctas = num_ctas
        a.activation = {None: 0, "relu": 1}[activation]
        if x_corr is not None:  # offset-code bias table written with xc (2-bit codes only)
            if (x_corr.dtype != torch.float32 or not x_corr.is_contiguous() or x_corr.dim() != 2
                    or x_corr.shape[0] < canonical_rows(B) or x_corr.shape[1] < _ceil(geom.m) // 128):
                raise ValueError("x_corr must be a contiguous f32 [canonical_rows(B), ceil(m/128)] tensor")
            a.x_corr, a.x_corr_ld = x_corr.data_ptr(), x_corr.stride(0)
        if swiglu is not None:
            I, act, act_corr = swiglu
            a.swiglu_I, a.act, a.act_np = int(I), act.data_ptr(), canonical_rows(B)
            if act.numel() < canonical_numel(B, int(I)):
                raise ValueError("act too small for the canonical layout of B rows")
            if act_corr is not None:
                a.act_corr, a.act_corr_ld = act_corr.data_ptr(), act_corr.stride(0)
            self.keep = self.keep + (act, act_corr)
        self.args = a
        self._fn = L.mesw_me_linear

    def __call__(self, stream=None) -> None:
        _lib.check(self._fn(C.byref(self.args), _stream(stream)))


PREFILL_GROUP = 128  # tokens per expert group of the prefill kernel (K3)
PREFILL_TILE = 256


class PrefillPlan:
    """Pre-built launch of the prefill fused multi-expert linear (K3, mesw_me_linear_prefill).

    `xc`: canonical layout of NP rows (NP % 256 == 0); `group_slots[g]` = expert-table slot of
    rows [128g, 128g+128) or -1 (base only).  y[t] = x[t] . bf16(W + Dtilde_e): the delta is
    folded into the tensor-core A operand, so the tensor work is the base GEMM's."""

    def __init__(self, xc: torch.Tensor, NP: int, B: int, weight: DeviceWeight, table: ExpertTable | None,
                 group_slots, out: torch.Tensor, residual: torch.Tensor | None = None, num_ctas: int = 0):
        if NP % PREFILL_TILE or B > NP or B < 1:
            raise ValueError("prefill: NP must be a multiple of 256 and 1 <= B <= NP")
        geom = weight.geom
        if xc.numel() < canonical_numel(NP, geom.m) or xc.dtype != torch.bfloat16:
            raise ValueError("xc too small for the canonical layout of NP rows")
        slots = [int(s) for s in group_slots]
        if len(slots) != NP // PREFILL_GROUP:
            raise ValueError("one slot per 128-token group")
        if any(s >= 0 for s in slots) and (table is None or table.code_bits != 2):
            raise NotImplementedError("prefill kernel: 2-bit codes only")
        if out.stride(1) != 1 or out.dtype not in (torch.bfloat16, torch.float32):
            raise ValueError("out must be a row-contiguous bf16/f32 tensor")
        self.geom = geom
        self.slots_dev = torch.as_tensor(slots, dtype=torch.int32, device=xc.device)
        self.keep = (xc, weight, table, out, residual)
        a = _lib.PrefillArgs()
        a.x, a.NP, a.B, a.m, a.n = xc.data_ptr(), NP, B, geom.m, geom.n
        a.w = weight.frag.data_ptr()
        a.expert_table = table.dev.data_ptr() if table is not None else None
        a.code_bits = 2
        a.group_slot = self.slots_dev.data_ptr()
        a.y, a.y_bf16, a.ldy = out.data_ptr(), 1 if out.dtype == torch.bfloat16 else 0, out.stride(0)
        if residual is not None:
            if residual.dtype != torch.bfloat16:
                raise ValueError("residual must be bf16")
            a.residual, a.ld_res = residual.data_ptr(), residual.stride(0)
        a.num_ctas = num_ctas
        self.args = a
        self._fn = _lib.lib().mesw_me_linear_prefill

    def __call__(self, stream=None) -> None:
        _lib.check(self._fn(C.byref(self.args), _stream(stream)))


def prefill_layout(B: int, segments) -> tuple:
    """Rows -> prefill layout: every expert segment starts on a 128-row group boundary,
    rows in no segment (base only) fill groups of their own.  Returns (NP, group_slots, src)
    with src[new_row] = old row or -1 (padding)."""
    segs = sorted((int(b), int(e), int(s)) for b, e, s in segments)
    src, slots = [], []

    def pad_to_group(slot):
        while len(src) % PREFILL_GROUP:
            src.append(-1)
        return slot

    cur = 0
    for b, e, sl in segs:
        if cur < b:  # base-only rows
            start = len(src)
            src.extend(range(cur, b))
            pad_to_group(None)
            slots.extend([-1] * ((len(src) - start) // PREFILL_GROUP))
        start = len(src)
        src.extend(range(b, e))
        pad_to_group(None)
        slots.extend([sl] * ((len(src) - start) // PREFILL_GROUP))
        cur = e
    if cur < B:
        start = len(src)
        src.extend(range(cur, B))
        pad_to_group(None)
        slots.extend([-1] * ((len(src) - start) // PREFILL_GROUP))
    while len(src) % PREFILL_TILE:
        src.extend([-1] * PREFILL_GROUP)
        slots.append(-1)
    return len(src), slots, src


def me_linear_prefill(x: torch.Tensor, weight: DeviceWeight, table: ExpertTable | None, segments,
                      out: torch.Tensor | None = None, residual: torch.Tensor | None = None,
                      out_dtype=torch.bfloat16, num_ctas: int = 0, stream=None) -> torch.Tensor:
    """Prefill form of me_linear for large token batches (BASELINE config 4): rows grouped by
    expert are laid out in 128-row groups (one device gather when segments are not already
    128-aligned), one K3 launch, results returned in the caller's row order."""
    geom = weight.geom
    B = x.shape[0]
    if out is None:
        out = torch.empty((B, geom.n), dtype=out_dtype, device=x.device)
    NP, slots, src = prefill_layout(B, segments)
    xm = x[:, :geom.m] if x.shape[1] >= geom.m else x
    aligned = src[:B] == list(range(B)) and all(v < 0 for v in src[B:])
    if aligned:
        xp = torch.zeros((NP, geom.m), dtype=torch.bfloat16, device=x.device)
        xp[:B] = xm
        PrefillPlan(pack_x(xp, stream=stream), NP, B, weight, table, slots, out, residual, num_ctas)(stream)
        return out
    src_t = torch.as_tensor(src, dtype=torch.int64, device=x.device)
    valid = src_t >= 0
    xp = torch.zeros((NP, geom.m), dtype=torch.bfloat16, device=x.device)
    xp[valid] = xm[src_t[valid]]
    rp = None
    if residual is not None:
        rp = torch.zeros((NP, residual.shape[1]), dtype=residual.dtype, device=x.device)
        rp[valid] = residual[src_t[valid]]
    yp = torch.empty((NP, out.shape[1]), dtype=out.dtype, device=x.device)
    PrefillPlan(pack_x(xp, stream=stream), NP, NP, weight, table, slots, yp, rp, num_ctas)(stream)
    out[src_t[valid]] = yp[valid]
    return out


# ------------------------------------------------------------------ launch-width tuning
# K2 splits (column-group pair, k-step) units over CTA pairs (stream-K).  When the units
# divide evenly into whole column groups or aligned k-splits, the final reduction has
# fewer contributors and the launch tail shrinks (measured: o_proj 4096x4096 B=32 E=3
# 33.3 us on 148 CTAs -> 27.6 us on 128), while for ALU-heavy expert mixes every SM
# counts.  The best width depends on shape and expert mix, so plans are timed once per
# shape key and the winner cached (tune_num_ctas).

_TUNED: dict = {}


def cta_candidates(geom: "LinearGeometry", sms: int) -> list:
    """Even CTA counts worth timing for a linear: all SMs, a few narrower grids, and the
    widest grid whose pairs each own an aligned k-split of one column-group pair."""
    g2max = sms // 2
    n_cgp = (geom.n_pad + 255) // 256
    n_ks = geom.m_pad // TILE
    cands = {0}
    for d in (1, 2, 3, 4, 6):      # just under the SM count (stream-K boundaries move)
        cands.add(2 * (g2max - d))
    for f in (0.86, 0.75):
        cands.add(2 * max(1, int(g2max * f)))
    best = 0
    for s_ in range(1, n_ks + 1):
        if n_ks % s_ == 0 and n_cgp * s_ <= g2max:
            best = s_
    if best:
        cands.add(2 * n_cgp * best)
    return sorted(c for c in cands if c <= sms)


def tune_num_ctas(key, make_plan, candidates, reps: int = 16, stream=None, trials: int = 3) -> int:
    """Time `make_plan(num_ctas)()` for each candidate (CUDA events, after warm-up) and
    cache the fastest under `key`.  make_plan must build plans on scratch outputs.  Each
    candidate is scored by its slowest of `trials` timings: some partial-grid widths are
    bimodal from run to run (which SMs / L2 halves the pairs land on: C1 at 112 CTAs
    measured 41.9 or 48.5 us), and a width that is only sometimes fast must not win."""
    if key in _TUNED:
        return _TUNED[key]
    best, best_t = 0, None
    for c in candidates:
        plan = make_plan(c)
        for _ in range(2):
            plan(stream)
        t = 0.0
        for _ in range(trials):
            st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            st.record()
            for _ in range(reps):
                plan(stream)
            en.record()
            en.synchronize()
            t = max(t, st.elapsed_time(en))
        if best_t is None or t < best_t:
            best, best_t = c, t
    _TUNED[key] = best
    return best


TMEM_ROW_BUDGET = 384  # base + delta accumulator columns per launch (512 TMEM columns - 2 A slots)


def segment_align(n_rows: int) -> int:
    """Row alignment of an expert group in a fused launch: groups of <= 8 rows take one
    8-row half of a 16-row tcgen05 window (two such experts share a window: the kernel's
    delta MMA for each covers the window and its epilogue reads only its own half), larger
    groups start on a window."""
    return 8 if n_rows <= 8 else 16


def delta_columns(begin: int, end: int) -> int:
    """Delta accumulator columns a segment takes: 16 per window it touches."""
    return 16 * (((end - 1) >> 4) - (begin >> 4) + 1)


def align_segments(B: int, segments) -> tuple:
    """Re-layout rows so every expert segment starts on its alignment (segment_align: an
    8-row half window for <= 8 rows, else a 16-row window -- the kernel's tcgen05 N
    granularity).  Returns (rows_pad, new_segments, src) where src[new_row] = old row or
    -1 for padding rows."""
    segs = sorted((int(b), int(e), int(s)) for b, e, s in segments)
    src, new_segs = [], []
    cur = 0
    for b, e, sl in segs:
        if cur < b:  # uncovered (base-only) rows keep their place in order
            src.extend(range(cur, b))
        while len(src) % segment_align(e - b):
            src.append(-1)
        new_segs.append((len(src), len(src) + (e - b), sl))
        src.extend(range(b, e))
        cur = e
    src.extend(range(cur, B))
    return len(src), new_segs, src


def launch_groups(B: int, segs: list, max_rows: int = None, tmem_cols: int = TMEM_ROW_BUDGET) -> list:
    """Split rows [0, B) into fused launches: each <= max_rows padded rows (MAX_ROWS) with
    base + delta accumulator columns (canonical_rows + sum of delta_columns) <= tmem_cols,
    cut at 16-row boundaries, preferring segment starts; an oversized expert group is cut
    too.  Returns [(r0, r1, segments rebased to r0)]."""
    max_rows = MAX_ROWS if max_rows is None else max_rows
    segs = sorted(segs)

    def fits(r0, r1):
        gs = [(max(b, r0) - r0, min(e, r1) - r0) for b, e, _ in segs if b < r1 and e > r0]
        return (r1 - r0 <= max_rows and
                canonical_rows(r1 - r0) + sum(delta_columns(b, e) for b, e in gs) <= tmem_cols)

    cuts = [0]
    while cuts[-1] < B:
        r0 = cuts[-1]
        bounds = {x for b, e, _ in segs for x in (b, e) if x > r0 and x % 16 == 0} | {B}
        cands = sorted(bounds | set(range(r0 + 16, min(B, r0 + max_rows) + 1, 16)))
        ok = []
        for x in cands:
            if not fits(r0, x):
                break
            ok.append(x)
        if not ok:
            raise NotImplementedError("a 16-row window does not fit one fused launch")
        at_bound = [x for x in ok if x in bounds]  # prefer not to split an expert group
        cuts.append(at_bound[-1] if at_bound else ok[-1])
    groups = []
    for r0, r1 in zip(cuts[:-1], cuts[1:]):
        gs = [(max(b, r0) - r0, min(e, r1) - r0, sl) for b, e, sl in segs if b < r1 and e > r0]
        groups.append((r0, r1, gs))
    return groups


_ME_PLANS: dict = {}
_ME_PLANS_MAX = 64


class _MeLinearPlan:
    """Cached device state of one me_linear call shape: row gather indices, canonical input
    and bias-table buffers and the bound launch plan(s) -- per call only the gather-pack and
    the fused launch run (two kernels, no host-side tensor ops)."""

    def __init__(self, x, weight, table, segs, out, residual, geom, num_ctas, activation, offset_codes, stream=None):
        B = x.shape[0]
        dev = x.device
        rows, new_segs, src = align_segments(B, segs)
        self.launches = []
        for start, end, csegs in launch_groups(rows, new_segs):
            n_rows = end - start
            src_t = torch.as_tensor(src[start:end], dtype=torch.int32, device=dev)
            xc = torch.empty(canonical_numel(n_rows, geom.m), dtype=torch.bfloat16, device=dev)
            corr = corr_table(n_rows, geom.m, dev) if (offset_codes and csegs) else None
            plan = None
            if weight is not None or csegs:
                plan = LinearPlan(xc, n_rows, weight, table if csegs else None, csegs, out, residual, geom,
                                  num_ctas, activation, x_corr=corr, stream=stream)
                plan.args.y_rows = src_t.data_ptr()  # grouped launch row -> caller's row (or -1)
            self.launches.append((src_t, n_rows, xc, corr, plan))
        self.keep = (weight, table)  # identity-checked by me_linear (ids alone could be reused)

    def __call__(self, x, out, residual, stream=None):
        L = _lib.lib()
        s = _stream(stream)
        for src_t, n_rows, xc, corr, plan in self.launches:
            if plan is None:
                continue
            plan.args.y = out.data_ptr()  # per-call tensors: rebinding two pointers is all it takes
            plan.args.residual = residual.data_ptr() if residual is not None else None
            _lib.check(L.mesw_pack_x_gather(x.data_ptr(), x.stride(0), src_t.data_ptr(), n_rows, plan.geom.m,
                                            xc.data_ptr(), corr.data_ptr() if corr is not None else None,
                                            corr.stride(0) if corr is not None else 0, s))
            plan(stream)


class MeLinearGraph:
    """`me_linear` on fixed buffers captured once in a CUDA graph (the form a serving loop
    uses for a repeated call shape): the device-side row gather, the bias table and the fused
    launch replay as one graph launch.  Callers copy new inputs into `x` (and `residual`)
    and read `out` after `__call__`, on the stream they replay on."""

    def __init__(self, x: torch.Tensor, weight: "DeviceWeight | None", table: "ExpertTable | None", segments,
                 out: torch.Tensor, residual: torch.Tensor | None = None, **kw):
        self.x, self.out, self.residual = x, out, residual
        dev = x.device
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):  # warm: plan, kernel attributes, launch-width tuning
            me_linear(x, weight, table, segments, out=out, residual=residual, stream=s, **kw)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            g.capture_begin()
            me_linear(x, weight, table, segments, out=out, residual=residual, stream=s, **kw)
            g.capture_end()
        torch.cuda.current_stream(dev).wait_stream(s)
        self.graph = g

    def __call__(self) -> torch.Tensor:
        self.graph.replay()
        return self.out


def me_linear(x: torch.Tensor, weight: DeviceWeight | None, table: ExpertTable | None,
              segments, out: torch.Tensor | None = None, residual: torch.Tensor | None = None,
              out_dtype=torch.bfloat16, geom: LinearGeometry | None = None, num_ctas: int = 0,
              activation: str | None = None, stream=None, offset_codes: bool = False) -> torch.Tensor:
    """y = x.W + x.Dtilde_{expert(t)} (+ residual) -- the fused kernel on row-major inputs.

    offset_codes: pass the activation bias table so 2-bit codes expand in offset form
    (mesw.h x_corr; the bf16 serving engine's choice, ~1e-5 relative on the delta term).
    The default keeps the exact q expansion (the f32 provider path holds 1e-4).

    x: bf16 [B, >= m] on the GPU (row-contiguous), rows in any order; segments: iterable of
    (begin, end, slot) into `table`.  The device gathers the rows into expert groups on
    16-row boundaries (mesw_pack_x_gather) and the kernel's epilogue writes every result
    straight back to the caller's row (mesw_linear_args.y_rows): no host-side gathers or
    scatters, and the launch state is cached per call shape (one pack + one fused launch
    per <= 192 grouped rows).  Rows in no segment get the base term only.
    """
    if geom is None:
        geom = weight.geom if weight is not None else next(
            d.geom for d in table.deltas if d is not None)
    if x.dtype != torch.bfloat16 or not x.is_cuda or x.dim() != 2 or x.stride(1) != 1:
        raise ValueError("x must be a row-contiguous 2-D bf16 CUDA tensor")
    if x.shape[1] < geom.m:
        raise ValueError(f"x has {x.shape[1]} columns, the linear needs {geom.m}")
    B = x.shape[0]
    if out is None:
        out = torch.empty((B, geom.n), dtype=out_dtype, device=x.device)
    segs = tuple((int(b), int(e), int(s)) for b, e, s in segments)
    if weight is None and not segs:
        out.zero_()
        return out
    if out.shape[0] < B or out.stride(1) != 1 or out.dtype not in (torch.bfloat16, torch.float32):
        raise ValueError("out must be a row-contiguous bf16/f32 tensor with >= B rows")
    if residual is not None and (residual.dtype != torch.bfloat16 or residual.stride(1) != 1):
        raise ValueError("residual must be a row-contiguous bf16 tensor")
    # per stream: concurrent calls on two streams must not share the cached canonical buffers
    # or the split-K workspace
    key = (x.device, tuple(x.shape), x.stride(0), id(weight), id(table), segs, out.dtype, out.stride(0),
           residual.stride(0) if residual is not None else None, geom, num_ctas, activation, bool(offset_codes),
           table.dev.data_ptr() if table is not None else None,
           None if stream is None else int(stream.cuda_stream))
    plan = _ME_PLANS.get(key)
    if plan is None or plan.keep[0] is not weight or plan.keep[1] is not table:
        if len(_ME_PLANS) >= _ME_PLANS_MAX:
            _ME_PLANS.pop(next(iter(_ME_PLANS)))
        plan = _MeLinearPlan(x, weight, table, segs, out, residual, geom, num_ctas, activation, offset_codes,
                             stream)
        _ME_PLANS[key] = plan
    plan(x, out, residual, stream)
    return out
