"""The SPEC known-answer vectors (tests/golden/kat.json, made by the real reference) asserted on
the GPU path: step init / quantisation through the GPU compressor (quant.py:
81-120), dequantisation through the device decode (quant.py:135-139), and the SPEC delta_matvec
example through the fused kernel."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import mesw as om

pytestmark = pytest.mark.gpu


def _kat():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        return json.load(f)


def test_step_and_codes_b2_via_gpu_compress():
    from paper_2406_09041_b200 import compress
    k = _kat()
    delta = np.array([[0.9], [-1.8], [0.45]], np.float32)
    layer = compress.compress_layer(delta, np.ones(3, np.float32), bits=2, salient_k=0)
    assert float(layer.steps[0]) == np.float32(k["step_b2"])  # 1.8
    codes = om.unpack_codes(layer.packed.data, 3, 1, 2)[:, 0].tolist()
    assert codes == k["codes_b2"]                              # [1, -1, 0]


def test_dequant_via_device_decode():
    from paper_2406_09041_b200 import compress
    from paper_2406_09041_b200.device import DeviceDelta
    k = _kat()
    ol = om.OracleLayer(m=3, n=1, bits=2, k=0, salient_idx=np.zeros(0, np.int64),
                        salient_rows=np.zeros((0, 1), np.float16), steps=np.array([1.8], np.float32),
                        packed=om.pack_codes(np.array([[1], [-1], [0]]), 2))
    art = compress.deserialize_artifact(om.serialize_artifact(
        {"model_id": "kat", "domain": "d", "base_digest": "0", "layer_count": 1}, [ol]))
    got = DeviceDelta.from_blocks([art.layers[0]]).reconstruct()[:, 0].cpu().numpy()
    assert got.tolist() == [np.float32(v) for v in k["dequant"]]


def test_delta_matvec_ones_via_fused_kernel():
    """k=0, codes all +1, s_j = 0.5, x = [1,1,1] -> y_j = 1.5 for all j."""
    from paper_2406_09041_b200 import compress, infer
    k = _kat()
    n = len(k["delta_matvec_ones"])
    ol = om.OracleLayer(m=3, n=n, bits=2, k=0, salient_idx=np.zeros(0, np.int64),
                        salient_rows=np.zeros((0, n), np.float16), steps=np.full(n, 0.5, np.float32),
                        packed=om.pack_codes(np.ones((3, n), np.int64), 2))
    art = compress.deserialize_artifact(om.serialize_artifact(
        {"model_id": "kat", "domain": "d", "base_digest": "0", "layer_count": 1}, [ol]))
    p = infer.GpuCompressedProvider(art.layers[0])
    y = infer.delta_matvec(np.ones(3, np.float32), p)
    assert y.tolist() == k["delta_matvec_ones"]
