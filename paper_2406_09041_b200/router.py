"""Model-level router: multinomial Naive Bayes over hashed character 2/3-grams.

Mirrors SPEC router: `train_router`, `classify`, `evaluate_router`,
`render_prompt`, the MERT model file.  The forward (`classify_batch`) runs batched on the
GPU through `mesw_router_classify` (K4, csrc/mesw_router.cu); the hashing convention and
the f64 summation order are pinned in oracle/router.py and the GPU decision is
bit-identical to it.  Training, evaluation bookkeeping and the prompt are host plumbing.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["Router", "train_router", "save_router", "load_router", "DeviceRouter", "classify",
           "classify_batch", "evaluate_router", "render_prompt", "ngram_buckets", "N_BUCKETS"]

N_BUCKETS = 1 << 16
MAX_DOMAINS = 64  # classification: two domains per warp lane (K4); the prompt template caps at 6
PROMPT_MAX_OPTIONS = 6  # render_prompt enumerates A..F
MERT_MAGIC = b"MERT"
MERT_VERSION = 1

_FNV_OFFSET, _FNV_PRIME = 2166136261, 16777619


def _fnv1a32(data: bytes) -> int:
    h = _FNV_OFFSET
    for b in data:
        h = ((h ^ b) * _FNV_PRIME) & 0xFFFFFFFF
    return h


def ngram_buckets(query: str) -> np.ndarray:
    """Bucket ids of all 2-grams then all 3-grams (code points, FNV-1a of UTF-8, low 16 bits)."""
    out = [_fnv1a32(query[i:i + n].encode("utf-8")) & (N_BUCKETS - 1)
           for n in (2, 3) for i in range(len(query) - n + 1)]
    return np.asarray(out, dtype=np.int64)


@dataclass(frozen=True)
class Router:
    """RouterModel: domains (index = id), f32 log-priors, f32 log-likelihoods."""
    domains: tuple
    logprior: np.ndarray  # f32[D]
    loglik: np.ndarray    # f32[D, 2^16]

    def __post_init__(self):
        D = len(self.domains)
        if not 1 <= D <= MAX_DOMAINS:
            raise ValueError(f"router needs 1..{MAX_DOMAINS} domains, got {D}")
        if len(set(self.domains)) != D:
            raise ValueError("domain names must be unique")
        if self.logprior.shape != (D,) or self.loglik.shape != (D, N_BUCKETS):
            raise ValueError("router table shapes do not match the domain list")


def train_router(records, domains) -> Router:
    """Fit on (query, domain name) records; deterministic in the input."""
    domains = tuple(domains)
    if not 1 <= len(domains) <= MAX_DOMAINS:
        raise ValueError(f"router needs 1..{MAX_DOMAINS} domains")
    index = {d: i for i, d in enumerate(domains)}
    counts = np.zeros((len(domains), N_BUCKETS), dtype=np.int64)
    ndoc = np.zeros(len(domains), dtype=np.int64)
    for query, dom in records:
        if dom not in index:
            raise ValueError(f"record domain {dom!r} is not in the router's domain list")
        d = index[dom]
        ndoc[d] += 1
        np.add.at(counts[d], ngram_buckets(query), 1)
    missing = [domains[i] for i in range(len(domains)) if ndoc[i] == 0]
    if missing:
        raise ValueError(f"domains without training examples: {missing}")
    total = counts.sum(axis=1, keepdims=True)
    loglik = np.log((counts + 1).astype(np.float64) / (total + N_BUCKETS).astype(np.float64))
    logprior = np.log(ndoc.astype(np.float64) / float(ndoc.sum()))
    return Router(domains, logprior.astype(np.float32), loglik.astype(np.float32))


def save_router(router: Router) -> bytes:
    """MERT file: magic, u16 version, u32 D, per domain (u16 len, utf-8 name),
    f32 logprior[D], f32 loglik[D][2^16]; little-endian."""
    out = bytearray(MERT_MAGIC + struct.pack("<HI", MERT_VERSION, len(router.domains)))
    for name in router.domains:
        b = name.encode("utf-8")
        out += struct.pack("<H", len(b)) + b
    out += router.logprior.astype("<f4").tobytes() + router.loglik.astype("<f4").tobytes()
    return bytes(out)


def load_router(blob: bytes) -> Router:
    from .errors import BadMagicError, TruncatedArtifactError, UnsupportedVersionError
    if blob[:4] != MERT_MAGIC:
        raise BadMagicError("not a MERT router file")
    if len(blob) < 10:
        raise TruncatedArtifactError("router header truncated")
    ver, D = struct.unpack_from("<HI", blob, 4)
    if ver != MERT_VERSION:
        raise UnsupportedVersionError(f"router version {ver}")
    off, names = 10, []
    for _ in range(D):
        if off + 2 > len(blob):
            raise TruncatedArtifactError("router domain table truncated")
        (ln,) = struct.unpack_from("<H", blob, off)
        names.append(blob[off + 2:off + 2 + ln].decode("utf-8"))
        off += 2 + ln
    need = off + 4 * D + 4 * D * N_BUCKETS
    if len(blob) != need:
        raise TruncatedArtifactError(f"router file is {len(blob)} bytes, expected {need}")
    lp = np.frombuffer(blob, "<f4", D, off).astype(np.float32)
    ll = np.frombuffer(blob, "<f4", D * N_BUCKETS, off + 4 * D).reshape(D, N_BUCKETS).astype(np.float32)
    return Router(tuple(names), lp, ll)


class DeviceRouter:
    """Router tables resident on the GPU (256 KiB per domain: 4 MiB at 16 domains, L2-resident)."""

    def __init__(self, router: Router, device="cuda"):
        import torch
        self.router = router
        self.device = torch.device(device)
        self.loglik = torch.from_numpy(np.ascontiguousarray(router.loglik)).to(self.device)
        self.logprior = torch.from_numpy(np.ascontiguousarray(router.logprior)).to(self.device)

    def classify_codepoints(self, cps, offsets, stream=None):
        """cps int32 / offsets int64[B+1] CUDA tensors -> (domain i32[B], conf f32[B], prior_only i32[B])."""
        import torch
        B = offsets.numel() - 1
        dom = torch.empty(B, dtype=torch.int32, device=self.device)
        conf = torch.empty(B, dtype=torch.float32, device=self.device)
        flag = torch.empty(B, dtype=torch.int32, device=self.device)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        _lib.check(_lib.lib().mesw_router_classify(
            C.c_void_p(cps.data_ptr() if cps.numel() else offsets.data_ptr()), C.c_void_p(offsets.data_ptr()), B,
            C.c_void_p(self.loglik.data_ptr()), C.c_void_p(self.logprior.data_ptr()), len(self.router.domains),
            C.c_void_p(dom.data_ptr()), C.c_void_p(conf.data_ptr()), C.c_void_p(flag.data_ptr()),
            C.c_void_p(s.cuda_stream)))
        return dom, conf, flag

    def classify_batch(self, queries):
        """-> list of (domain name, confidence, prior_only) in query order."""
        import torch
        cps = [np.frombuffer(q.encode("utf-32-le"), dtype="<u4").astype(np.int32) for q in queries]
        offsets = np.zeros(len(queries) + 1, dtype=np.int64)
        offsets[1:] = np.cumsum([len(c) for c in cps])
        flat = np.concatenate(cps) if offsets[-1] else np.zeros(1, dtype=np.int32)
        d_cps = torch.from_numpy(flat).pin_memory().to(self.device, non_blocking=True)
        d_off = torch.from_numpy(offsets).pin_memory().to(self.device, non_blocking=True)
        dom, conf, flag = self.classify_codepoints(d_cps, d_off)
        dom, conf, flag = dom.cpu().numpy(), conf.cpu().numpy(), flag.cpu().numpy()
        names = self.router.domains
        return [(names[int(d)], float(c), bool(f)) for d, c, f in zip(dom, conf, flag)]


def classify_batch(router: Router | DeviceRouter, queries):
    dr = router if isinstance(router, DeviceRouter) else DeviceRouter(router)
    return dr.classify_batch(list(queries))


def classify(router: Router | DeviceRouter, query: str):
    """-> (domain name, confidence, prior_only)."""
    return classify_batch(router, [query])[0]


def evaluate_router(router: Router | DeviceRouter, records) -> dict:
    """overall / per-domain accuracy and the confusion matrix (exact counts)."""
    records = list(records)
    if not records:
        raise ValueError("empty dataset")
    dr = router if isinstance(router, DeviceRouter) else DeviceRouter(router)
    names = dr.router.domains
    index = {d: i for i, d in enumerate(names)}
    preds = dr.classify_batch([q for q, _ in records])
    conf = np.zeros((len(names), len(names)), dtype=np.int64)
    for (q, truth), (p, _, _) in zip(records, preds):
        conf[index[truth], index[p]] += 1
    per = {names[i]: (float(conf[i, i]) / conf[i].sum() if conf[i].sum() else None) for i in range(len(names))}
    return {"accuracy": float(np.trace(conf)) / len(records), "per_domain": per, "confusion": conf}


_TEMPLATE_HEAD = ("Classify the query based on the required expertise. Route the query to the appropriate "
                  "model for a precise response. Only output the letter corresponding to the best category "
                  "(A, B, C, …, F).")


def render_prompt(query: str, domains) -> str:
    """The paper's routing prompt (Appendix A, Table A) with lettered options."""
    domains = list(domains)
    if len(domains) > PROMPT_MAX_OPTIONS:
        raise ValueError("the template enumerates at most 6 options (A..F)")
    opts = " ".join(f"{chr(65 + i)}) {name} - {desc}" for i, (name, desc) in enumerate(domains))
    letters = ", ".join(f"'{chr(65 + i)}'" for i in range(len(domains)))
    return (f"{_TEMPLATE_HEAD}\n\nQuery: {query}\n\nOptions: {opts}\n\n"
            f"Response should be only {letters}, with no additional text.")
