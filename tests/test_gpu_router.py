"""K4 parity: batched GPU router forward vs the CPU restatement (decisions bit-exact)."""
import numpy as np
import pytest

from oracle import router as orc
from router_data import DOMAINS, make_records

pytestmark = pytest.mark.gpu


def _queries(seed, n):
    rng = np.random.default_rng(seed)
    alphabet = list("abcdefghijklmnopqrstuvwxyz     ") + list("翻译语法成语汉字拼音诗词") + ["é", "ß", "😀"]
    out = ["", "x", "ab", "abc"]
    for _ in range(n):
        L = int(rng.integers(0, 120))
        out.append("".join(rng.choice(alphabet, size=L)))
    out += [q for q, _ in make_records(10, seed=seed + 1)]
    return out


def test_router_gpu_matches_oracle():
    from paper_2406_09041_b200 import router as pr
    r = pr.train_router(make_records(60, seed=5), DOMAINS)
    o = orc.OracleRouter(r.domains, r.logprior, r.loglik)
    dr = pr.DeviceRouter(r)
    qs = _queries(6, 300)
    got = dr.classify_batch(qs)
    for q, (name, conf, flag) in zip(qs, got):
        d, c, f = orc.classify(o, q)
        assert name == r.domains[d], q
        assert flag == f
        assert abs(conf - c) <= 1e-6 * max(1.0, abs(c))


def test_router_gpu_ties_and_single_domain():
    from paper_2406_09041_b200 import router as pr
    # two domains with identical tables: every query ties -> lowest id, conf 1/2
    ll = np.full((2, pr.N_BUCKETS), -11.0, np.float32)
    r = pr.Router(("a", "b"), np.log(np.array([0.5, 0.5], np.float32)), ll)
    for name, conf, _ in pr.classify_batch(r, ["hello", "", "xyz" * 50]):
        assert name == "a" and abs(conf - 0.5) < 1e-6
    one = pr.train_router([("python code", "code")], ("code",))
    assert [x[0] for x in pr.classify_batch(one, ["anything", ""])] == ["code", "code"]


def test_router_gpu_accuracy_and_evaluate():
    from paper_2406_09041_b200 import router as pr
    r = pr.train_router(make_records(100, seed=7), DOMAINS)
    ev = pr.evaluate_router(r, make_records(25, seed=8))
    assert ev["accuracy"] == 1.0
    assert ev["confusion"].sum(axis=1).tolist() == [25] * 4


@pytest.mark.parametrize("D", [16, 33, 64])
def test_router_gpu_many_domains_match_oracle(D):
    """C3/C5 routing: 16 and 64 expert domains (two per warp lane past 32), decisions and
    confidences equal to the restatement; synthetic keyword pools are separable."""
    from paper_2406_09041_b200 import router as pr
    rng = np.random.default_rng(D)
    doms = tuple(f"dom{i}" for i in range(D))
    pools = {d: [f"{d}w{j}" for j in range(10)] for d in doms}
    rec = [(" ".join(rng.choice(pools[d], size=5)), d) for d in doms for _ in range(8)]
    r = pr.train_router(rec, doms)
    o = orc.OracleRouter(r.domains, r.logprior, r.loglik)
    qs = [" ".join(rng.choice(pools[d], size=4)) for d in doms] + _queries(D, 60)
    got = pr.DeviceRouter(r).classify_batch(qs)
    for i, (q, (name, conf, flag)) in enumerate(zip(qs, got)):
        d, c, f = orc.classify(o, q)
        assert name == r.domains[d], q
        assert flag == f
        assert abs(conf - c) <= 1e-6 * max(1.0, abs(c))
        if i < D:
            assert name == doms[i]
