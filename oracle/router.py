"""CPU restatement of the model-level router (TEST INFRASTRUCTURE ONLY).

Follows SPEC.md:516-573 (the reference ships no router code: SURVEY.md §8(c), H7).  The
SPEC leaves hashing details open; this restatement pins them and the GPU kernel
(paper_2406_09041_b200/csrc/mesw_router.cu) must match it bit-for-bit on the decision:

* text unit: Unicode code points of the query string (no case folding, no padding);
* n-grams: n in {2, 3}; all 2-grams in order, then all 3-grams in order;
* hash: 32-bit FNV-1a over the UTF-8 bytes of the n-gram, bucket = low 16 bits
  (2^16 buckets);
* model: multinomial Naive Bayes, add-one smoothing:
  loglik[d][b] = f32(ln((count[d][b] + 1) / (total[d] + 2^16))) computed in f64,
  logprior[d] = f32(ln(n_d / N));
* score[d] = f64(logprior[d]) + sum over n-grams, in the order above, of f64(loglik[d][b])
  -- sequential f64, so both sides round identically;
* decision: argmax score, ties -> lowest domain id; confidence =
  softmax-normalised posterior of the winner, 1 / sum_d exp(score_d - score_win) in f64
  (SPEC.md:549); a query with no n-gram (length < 2) predicts from the priors alone and is
  flagged "prior-only".
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

N_BUCKETS = 1 << 16
FNV_OFFSET = 2166136261
FNV_PRIME = 16777619
MAX_DOMAINS = 64  # two domains per warp lane in K4; render_prompt alone caps at 6


def fnv1a32(data: bytes) -> int:
    h = FNV_OFFSET
    for b in data:
        h ^= b
        h = (h * FNV_PRIME) & 0xFFFFFFFF
    return h


def ngram_buckets(query: str) -> list:
    """Bucket ids of the query's 2-grams then 3-grams, in order."""
    out = []
    for n in (2, 3):
        for i in range(len(query) - n + 1):
            out.append(fnv1a32(query[i:i + n].encode("utf-8")) & (N_BUCKETS - 1))
    return out


@dataclass(frozen=True)
class OracleRouter:
    domains: tuple            # names, index = domain id
    logprior: np.ndarray      # f32[D]
    loglik: np.ndarray        # f32[D, 2^16]


def train_router(records, domains) -> OracleRouter:
    """records: iterable of (query, domain name).  SPEC.md:540-545."""
    domains = tuple(domains)
    if not domains or len(domains) > MAX_DOMAINS:
        raise ValueError(f"1..{MAX_DOMAINS} domains")
    index = {d: i for i, d in enumerate(domains)}
    counts = np.zeros((len(domains), N_BUCKETS), dtype=np.int64)
    ndoc = np.zeros(len(domains), dtype=np.int64)
    for query, dom in records:
        if dom not in index:
            raise ValueError(f"unknown domain {dom!r}")
        d = index[dom]
        ndoc[d] += 1
        for b in ngram_buckets(query):
            counts[d, b] += 1
    missing = [domains[i] for i in range(len(domains)) if ndoc[i] == 0]
    if missing:
        raise ValueError(f"domains without training examples: {missing}")
    total = counts.sum(axis=1)
    loglik = np.log((counts + 1).astype(np.float64) / (total[:, None] + N_BUCKETS).astype(np.float64))
    logprior = np.log(ndoc.astype(np.float64) / float(ndoc.sum()))
    return OracleRouter(domains, logprior.astype(np.float32), loglik.astype(np.float32))


def scores(router: OracleRouter, query: str):
    """Sequential f64 posterior scores; returns (scores list, prior_only)."""
    buckets = ngram_buckets(query)
    out = []
    for d in range(len(router.domains)):
        s = float(np.float64(router.logprior[d]))
        row = router.loglik[d]
        for b in buckets:
            s += float(np.float64(row[b]))
        out.append(s)
    return out, len(buckets) == 0


def classify(router: OracleRouter, query: str):
    """-> (domain id, confidence f32, prior_only).  SPEC.md:546-551."""
    sc, prior_only = scores(router, query)
    win = 0
    for d in range(1, len(sc)):
        if sc[d] > sc[win]:
            win = d
    z = 0.0
    for d in range(len(sc)):
        z += math.exp(sc[d] - sc[win])
    return win, float(np.float32(1.0 / z)), prior_only
