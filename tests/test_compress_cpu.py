"""f2 oracle: the CPU restatement of compress_layer reproduces the reference's own
compressed layers bit-for-bit (tests/golden: layer_*.mesw + their inputs)."""
import json
import os

import numpy as np
import pytest

from oracle import compress as oc
from oracle import mesw as om

from conftest import GOLDEN

CASES = {"l2_256x384_k8": (2, 8), "l2_200x130_k5": (2, 5), "l3_128x256_k4": (3, 4), "l4_192x128_k8": (4, 8),
         "l8_128x128_k2": (8, 2), "l1_256x128_k0": (1, 0), "l2_64x64_k64": (2, 64)}


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_compress_matches_reference(name):
    z = np.load(os.path.join(GOLDEN, "layer_expected.npz"))
    bits, k = CASES[name]
    got = oc.compress_layer(z[f"{name}_delta"], z[f"{name}_energy"], bits, k)
    with open(os.path.join(GOLDEN, f"layer_{name}.mesw"), "rb") as f:
        _, (ref,) = om.parse_artifact(f.read())
    assert np.array_equal(got.salient_idx, ref.salient_idx)
    assert np.array_equal(got.steps.view(np.uint32), ref.steps.view(np.uint32))
    assert np.array_equal(got.salient_rows.view(np.uint16), ref.salient_rows.view(np.uint16))
    assert got.packed == ref.packed


def test_pairwise_sum_restatement():
    rng = np.random.default_rng(5)
    for n in (1, 7, 8, 127, 128, 129, 384, 4096, 14336):
        a = rng.normal(size=n) ** 2 * 10.0 ** rng.uniform(-6, 6, size=n)
        assert oc.pairwise_sum_f64(a) == a.reshape(1, -1).sum(axis=1)[0]
