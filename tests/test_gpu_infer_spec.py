"""SPEC `infer` examples and invariants on the GPU providers:
Zero / Exact / LowRank / Compressed `delta_matvec`, the fused-kernel equivalence over
b in {1, 2, 4} x k in {0, 1, 8}, the decoupling identity of Eq. 4, and `bench_decode`."""

import numpy as np
import pytest

from oracle import mesw as om

pytestmark = pytest.mark.gpu

MAN = {"model_id": "spec", "domain": "d", "base_digest": "0", "layer_count": 1}


def _layer(ol):
    from paper_2406_09041_b200 import compress
    return compress.deserialize_artifact(om.serialize_artifact(MAN, [ol])).layers[0]


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


def test_zero_exact_lowrank_providers():
    """Zero -> zeros; Exact -> plain matvec; LowRank -> (x.A).B."""
    from paper_2406_09041_b200.infer import ExactProvider, LowRankProvider, ZeroProvider, delta_matvec
    rng = np.random.default_rng(1)
    m, n, r = 64, 48, 5
    x = rng.normal(0, 1, m).astype(np.float32)
    assert not np.any(delta_matvec(x, ZeroProvider((m, n))))
    d = rng.normal(0, 0.1, (m, n)).astype(np.float32)
    assert _rel(delta_matvec(x, ExactProvider(d)), x.astype(np.float64) @ d) <= 1e-5
    a = rng.normal(0, 0.3, (m, r)).astype(np.float32)
    b = rng.normal(0, 0.3, (r, n)).astype(np.float32)
    want = (x.astype(np.float64) @ a) @ b
    assert _rel(delta_matvec(x, LowRankProvider(a, b)), want) <= 1e-5
    with pytest.raises(ValueError):
        delta_matvec(x, None)


@pytest.mark.parametrize("bits", [1, 2, 4])
@pytest.mark.parametrize("k", [0, 1, 8])
def test_fused_kernel_equivalence(bits, k):
    """delta_matvec(Compressed) == x . reconstruct() within 1e-5 relative, from the packed
    codes without materialising the dense delta."""
    from paper_2406_09041_b200.infer import GpuCompressedProvider, delta_matvec
    rng = np.random.default_rng(10 * bits + k)
    m, n = 96, 80
    ol = om.random_layer(rng, m, n, bits, k if bits != 1 else 0)
    dense = ol.reconstruct().astype(np.float64)
    p = GpuCompressedProvider(_layer(ol))
    for _ in range(3):
        x = rng.normal(0, 1, m).astype(np.float32)
        assert _rel(delta_matvec(x, p), x.astype(np.float64) @ dense) <= 1e-5
    h = rng.normal(0, 1, (7, m)).astype(np.float32)
    assert _rel(p.matvec_batch(h), h.astype(np.float64) @ dense) <= 1e-5


def test_decoupling_identity():
    """matvec(x, W + D) == matvec(x, W) + delta_matvec(x, Exact(D)) within 1e-5 relative
    (Eq. 4); and the same with the Compressed provider for D = reconstruct()."""
    from paper_2406_09041_b200.infer import ExactProvider, GpuCompressedProvider, delta_matvec
    rng = np.random.default_rng(3)
    m, n = 128, 96
    W = rng.normal(0, 0.05, (m, n)).astype(np.float32)
    ol = om.random_layer(rng, m, n, 2, 8)
    D = ol.reconstruct().astype(np.float32)
    x = rng.normal(0, 1, m).astype(np.float32)
    lhs = delta_matvec(x, ExactProvider(W + D))
    assert _rel(lhs, delta_matvec(x, ExactProvider(W)) + delta_matvec(x, ExactProvider(D))) <= 1e-5
    assert _rel(lhs, delta_matvec(x, ExactProvider(W)) + delta_matvec(x, GpuCompressedProvider(_layer(ol)))) <= 1e-5


def test_bench_decode_decomposition():
    """bench_decode: median / p90 per stage; zero providers -> no delta
    stage; repetitions=1 -> flagged "no-variance"; the delta stage grows with the expert
    count of the batch."""
    import torch
    from paper_2406_09041_b200.device import DeviceDelta, DeviceWeight, ExpertTable, LinearGeometry
    from paper_2406_09041_b200.infer import bench_decode
    rng = np.random.default_rng(5)
    m, n = 1024, 2048
    geom = LinearGeometry(m, (n,))
    dw = DeviceWeight.from_dense([rng.normal(0, 0.02, (m, n)).astype(np.float32)])
    table = ExpertTable("cuda")
    for e in range(8):
        table.set(e, DeviceDelta.from_blocks([_layer(om.random_layer(rng, m, n, 2, 8))], geom))
    x = torch.from_numpy(rng.normal(0, 1, (64, m)).astype(np.float32)).to(torch.bfloat16).cuda()
    zero = bench_decode(dw, table, [], x, repetitions=5)
    assert zero["delta_stage_ms"]["median"] == 0.0
    assert set(zero) == {"base_gemm_ms", "delta_stage_ms", "total_ms"}
    one = bench_decode(dw, table, [(0, 64, 0)], x, repetitions=1)
    assert one["total_ms"]["flag"] == "no-variance" and one["total_ms"]["n"] == 1
    few = bench_decode(dw, table, [(0, 64, 0)], x, repetitions=15)["delta_stage_ms"]["median"]
    many = bench_decode(dw, table, [(8 * e, 8 * e + 8, e) for e in range(8)], x,
                        repetitions=15)["delta_stage_ms"]["median"]
    assert many > few
