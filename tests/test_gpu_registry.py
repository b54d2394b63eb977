"""GPU load path of the expert registry: acquire uploads + repacks on a copy stream and the
resident deltas reconstruct bit-exactly to the reference restatement; LRU eviction frees them."""
import numpy as np
import pytest

from oracle import mesw as om
from paper_2406_09041_b200 import synth

pytestmark = pytest.mark.gpu


def test_registry_gpu_load_and_evict():
    from paper_2406_09041_b200 import compress
    from paper_2406_09041_b200.registry import ExpertRegistry, GpuExpert
    blobs = {f"e{i}": synth.synthetic_expert_artifact(50 + i, [(256, 384), (384, 256)], "code") for i in range(3)}
    size = compress.compressed_size_bytes(compress.deserialize_artifact(blobs["e0"])).total
    reg = ExpertRegistry(2 * size, "synthetic")
    for e, b in blobs.items():
        reg.register(e, b)
    for e in ("e0", "e1", "e2"):
        h = reg.acquire(e)
        assert isinstance(h, GpuExpert) and len(h.layers) == 2
        _, ref_layers = om.parse_artifact(blobs[e])
        for dd, ol in zip(h.layers, ref_layers):
            got = dd.reconstruct().cpu().numpy()
            assert np.array_equal(got, ol.reconstruct())
        reg.release(e)
    s = reg.stats()
    assert sorted(s.resident) == ["e1", "e2"] and s.evict_count == 1 and s.current_bytes == 2 * size
