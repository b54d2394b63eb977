"""Mistral-shaped golden block from the REAL reference package (run in the build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_mistral_golden.py

Outputs (committed, ~1.1 MB): tests/golden/ref_kproj_4096x1024.mesw -- one k_proj-shaped
(4096 x 1024) layer compressed by the reference's own `compress_layer` (b=2, k=8, metric
"reconstruction", compress.py:178-215) from a seeded synthetic fine-tuning delta, serialized
with the reference `serialize_artifact` (compress.py:481-495).  The Mistral-dimension parity
test (tests/test_gpu_mistral_full.py) splices it into expert 0's layer-0 k projection so the
serving engine's offset-code path runs on reference-made bytes at real dimensions, and
`tests/test_oracle_golden.py` checks the oracle's parse/reconstruct of it against the
reference's own reconstruct() digest (kat_mistral.json) and x @ reconstruct() for
x = rng(7).normal(0, 1, (4, 4096)) (ref_kproj_y.npy).
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from meswitch import compress, salient  # noqa: E402  (reference package)

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(2406)
    m, n = 4096, 1024
    delta = rng.normal(0, 1e-3, size=(m, n)).astype(np.float32)
    planted = rng.choice(m, size=8, replace=False)
    delta[planted] += rng.normal(0, 0.05, size=(8, n)).astype(np.float32)
    acts = rng.normal(0, 1, size=(256, m)).astype(np.float32)
    stats = salient.stats_from_layer_inputs(acts)
    layer = compress.compress_layer(delta, stats, compress.CompressionConfig(bits=2, salient_k=8))
    man = compress.ArtifactManifest(model_id="ref_kproj", domain="synthetic", base_digest="0" * 64,
                                    layer_count=1)
    blob = compress.serialize_artifact(compress.ExpertArtifact(manifest=man, layers=[layer]))
    with open(os.path.join(HERE, "ref_kproj_4096x1024.mesw"), "wb") as f:
        f.write(blob)
    recon = layer.reconstruct()
    x = np.random.default_rng(7).normal(0, 1, size=(4, m)).astype(np.float32)  # tests regenerate it
    kat = {"file": "ref_kproj_4096x1024.mesw", "m": m, "n": n, "bits": 2, "k": 8,
           "salient": [int(i) for i in layer.salient.indices],
           "recon_sha256": hashlib.sha256(np.ascontiguousarray(recon, "<f4").tobytes()).hexdigest()}
    with open(os.path.join(HERE, "kat_mistral.json"), "w") as f:
        json.dump(kat, f)
    np.save(os.path.join(HERE, "ref_kproj_y.npy"), (x @ recon).astype(np.float32))  # x: rng(7) N(0,1) [4, m]
    print("wrote", len(blob), "bytes")


if __name__ == "__main__":
    main()
