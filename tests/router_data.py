"""Synthetic 4-domain routing dataset: disjoint keyword pools
per domain, deterministic per seed."""
import numpy as np

DOMAINS = ("instruct", "code", "math", "chinese")
POOLS = {
    "instruct": ["explain", "advice", "guide", "summarize", "recommend", "describe", "plan", "tips"],
    "code": ["python", "debug", "function", "compile", "segfault", "refactor", "lambda", "pointer"],
    "math": ["integral", "prove", "theorem", "matrix", "derivative", "prime", "equation", "lemma"],
    "chinese": ["翻译", "语法", "成语", "汉字", "拼音", "诗词", "句子", "词语"],
}
FILLER = ["the", "a", "please", "how", "to", "of", "my", "for", "with", "this"]


def make_records(n_per_domain: int, seed: int):
    rng = np.random.default_rng(seed)
    out = []
    for d in DOMAINS:
        for _ in range(n_per_domain):
            words = list(rng.choice(POOLS[d], size=3)) + list(rng.choice(FILLER, size=3))
            rng.shuffle(words)
            out.append((" ".join(words), d))
    return out
