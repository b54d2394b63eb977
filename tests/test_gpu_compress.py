"""f2: GPU compress_layer is bit-exact with the reference (golden layers) and with the CPU
restatement on larger random layers (b in {1,2,3,4,8})."""
import os

import numpy as np
import pytest

from oracle import compress as oc
from oracle import mesw as om

from conftest import GOLDEN
from test_compress_cpu import CASES

pytestmark = pytest.mark.gpu


def _same(got, ref):
    assert np.array_equal(got.salient.indices, ref.salient_idx)
    assert np.array_equal(got.steps.view(np.uint32), ref.steps.view(np.uint32))
    assert np.array_equal(got.salient_rows.view(np.uint16), ref.salient_rows.view(np.uint16))
    assert got.packed.data == ref.packed


@pytest.mark.parametrize("name", sorted(CASES))
def test_gpu_compress_matches_reference_artifacts(name):
    from paper_2406_09041_b200 import compress
    z = np.load(os.path.join(GOLDEN, "layer_expected.npz"))
    bits, k = CASES[name]
    got = compress.compress_layer(z[f"{name}_delta"], z[f"{name}_energy"], bits=bits, salient_k=k)
    with open(os.path.join(GOLDEN, f"layer_{name}.mesw"), "rb") as f:
        _, (ref,) = om.parse_artifact(f.read())
    _same(got, ref)


@pytest.mark.parametrize("bits,k,m,n", [(2, 8, 1024, 1536), (3, 4, 640, 384), (4, 16, 512, 1024),
                                        (8, 2, 256, 512), (1, 0, 768, 256), (2, 8, 4096, 520)])
def test_gpu_compress_matches_oracle_random(bits, k, m, n):
    from paper_2406_09041_b200 import compress
    rng = np.random.default_rng(m + n + bits)
    delta = rng.normal(0, 1e-3, size=(m, n)).astype(np.float32)
    planted = rng.choice(m, size=6, replace=False)
    delta[planted] += rng.normal(0, 0.05, size=(6, n)).astype(np.float32)
    delta[:, 3] = 0.0  # an all-zero column -> TINY_F32 step
    energy = (rng.normal(0, 1, size=m) ** 2 * 64).astype(np.float32)
    got = compress.compress_layer(delta, energy, bits=bits, salient_k=k)
    _same(got, oc.compress_layer(delta, energy, bits, k))
