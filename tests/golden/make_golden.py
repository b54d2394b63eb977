"""Generate golden fixtures from the REAL reference package (run in the build
container, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (committed; small):
  tests/golden/kat.json           SPEC known-answer vectors + size arithmetic
  tests/golden/codes.npz          random code matrices and their packed bytes, b in {1,2,3,4,8}
  tests/golden/toy_base.npz       toy base model weights (random_toylm seed 0)
  tests/golden/toy_expert_*.mesw  compressed experts (reference compress_expert)
  tests/golden/toy_expected.npz   reference forward / forward_with_delta / greedy_decode outputs
  tests/golden/layer_*.mesw       single-layer artifacts from reference compress_layer
  tests/golden/layer_expected.npz inputs x and reference x @ reconstruct() for those layers
  tests/golden/bad_*.mesw         malformed containers + expected error class (kat.json)

Nothing at GPU-test run time reads /root/reference: the GPU box only sees these files.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

from meswitch import compress, quant, salient, toylm  # noqa: E402  (reference package)

HERE = os.path.dirname(os.path.abspath(__file__))


class _Dense:
    """Provider over reference reconstruct(); CompressedDelta itself cannot be a
    provider because its `rows` is an int property (toylm.py:175 vs compress.py:96)."""

    def __init__(self, d):
        self.d = d

    def matvec_batch(self, h):
        return h @ self.d

    def rows(self, ids):
        return self.d[ids]


def kat():
    out = {}
    out["pack_b2"] = quant.pack_codes(np.array([[-2], [-1], [0], [1]]), quant.QuantConfig(2)).data.hex()
    out["pack_b1"] = quant.pack_codes(
        np.array([[1], [1], [-1], [-1], [1], [1], [-1], [-1]]), quant.QuantConfig(1)).data.hex()
    out["pack_b3"] = quant.pack_codes(np.array([[-4], [3], [0]]), quant.QuantConfig(3)).data.hex()
    s = quant.init_step_sizes(np.array([[0.9], [-1.8], [0.45]], np.float32), quant.QuantConfig(2)).steps
    out["step_b2"] = float(s[0])
    out["codes_b2"] = quant.quantize_codes(np.array([[0.9], [-1.8], [0.45]], np.float32), s,
                                           quant.QuantConfig(2)).ravel().tolist()
    out["dequant"] = quant.dequantize(np.array([[1], [-1], [0]]), np.array([1.8], np.float32),
                                      quant.QuantConfig(2)).ravel().tolist()
    sizes = compress.layer_block_nbytes(4096, 4096, 2, 8)
    out["size_4096x4096_b2_k8"] = dict(codes=sizes.codes, salient_rows=sizes.salient_rows,
                                       steps=sizes.steps, indices=sizes.indices,
                                       header=sizes.header, total=sizes.total)
    out["size_4096x14336_b2_k8_total"] = compress.layer_block_nbytes(4096, 14336, 2, 8).total
    out["size_4096x4096_b1_k0_total"] = compress.layer_block_nbytes(4096, 4096, 1, 0).total
    out["size_4096x4096_b4_k8_total"] = compress.layer_block_nbytes(4096, 4096, 4, 8).total
    # k=0, codes all +1, s=0.5, x=[1,1,1] -> 1.5
    cd = compress.CompressedDelta(
        salient=salient.top_k(np.zeros(3), 0),
        salient_rows=np.zeros((0, 2), np.float16),
        steps=np.full(2, 0.5, np.float32),
        packed=quant.pack_codes(np.ones((3, 2), np.int8), quant.QuantConfig(2)))
    out["delta_matvec_ones"] = (np.ones(3, np.float32) @ cd.reconstruct()).tolist()
    return out


def codes_fixtures(rng):
    arrs = {}
    shapes = [(1, 1), (3, 2), (37, 5), (64, 64), (130, 3), (257, 9)]
    for bits in (1, 2, 3, 4, 8):
        cfg = quant.QuantConfig(bits)
        for (m, n) in shapes:
            if bits == 1:
                c = rng.choice(np.array([-1, 1]), size=(m, n)).astype(np.int8)
            else:
                c = rng.integers(-cfg.q_n, cfg.q_p + 1, size=(m, n)).astype(np.int8)
            p = quant.pack_codes(c, cfg)
            assert np.array_equal(quant.unpack_codes(p), c)
            key = f"b{bits}_{m}x{n}"
            arrs[key + "_codes"] = c
            arrs[key + "_packed"] = np.frombuffer(p.data, np.uint8)
    np.savez_compressed(os.path.join(HERE, "codes.npz"), **arrs)


def toy_fixtures(rng, kat_out):
    base = toylm.random_toylm(0)
    np.savez_compressed(os.path.join(HERE, "toy_base.npz"), embedding=base.embedding,
                        head=base.head, **{f"layer{i}": w for i, w in enumerate(base.layers)})
    seqs = [list(rng.integers(0, 256, size=16)) for _ in range(8)]
    specs = [toylm.ExpertSpec(domain=d, seed=s) for d, s in (("instruct", 11), ("math", 12), ("code", 13))]
    expected = {"base_digest": toylm.base_digest(base)}
    arrays = {}
    tokens = np.array(rng.integers(0, 256, size=12), np.int64)
    arrays["tokens"] = tokens
    arrays["base_logits"] = toylm.forward(base, tokens)
    prompt = [72, 101, 108, 108, 111]
    for e, spec in enumerate(specs):
        ft = toylm.synthesize_expert(base, spec)
        cfg = compress.CompressionConfig(bits=2, salient_k=8,
                                         distill=compress.DistillConfig(epochs=1 if e == 0 else 0))
        res = compress.compress_expert(base, ft, seqs, cfg, model_id=f"toy-{spec.domain}",
                                       domain=spec.domain)
        blob = compress.serialize_artifact(res.artifact)
        with open(os.path.join(HERE, f"toy_expert_{e}.mesw"), "wb") as f:
            f.write(blob)
        provs = [_Dense(l.reconstruct()) for l in res.artifact.layers]
        arrays[f"fwd_delta_{e}"] = toylm.forward_with_delta(base, provs, tokens)
        arrays[f"greedy_{e}"] = np.array(toylm.greedy_decode(base, prompt, 12, provs), np.int64)
        for li, l in enumerate(res.artifact.layers):
            arrays[f"recon_{e}_{li}"] = l.reconstruct()
            arrays[f"codes_{e}_{li}"] = l.codes()
    arrays["greedy_base"] = np.array(toylm.greedy_decode(base, prompt, 12), np.int64)
    arrays["prompt"] = np.array(prompt, np.int64)
    np.savez_compressed(os.path.join(HERE, "toy_expected.npz"), **arrays)
    kat_out["toy"] = expected


def layer_fixtures(rng, kat_out):
    """Single layers compressed by the reference at shapes that exercise the GPU tiling."""
    cases = [("l2_256x384_k8", 256, 384, 2, 8), ("l2_200x130_k5", 200, 130, 2, 5),
             ("l3_128x256_k4", 128, 256, 3, 4), ("l4_192x128_k8", 192, 128, 4, 8),
             ("l8_128x128_k2", 128, 128, 8, 2), ("l1_256x128_k0", 256, 128, 1, 0),
             ("l2_64x64_k64", 64, 64, 2, 64)]
    arrays = {}
    names = []
    for name, m, n, bits, k in cases:
        delta = (rng.normal(0, 1e-3, size=(m, n))).astype(np.float32)
        planted = rng.choice(m, size=min(4, m), replace=False)
        delta[planted] += rng.normal(0, 0.05, size=(len(planted), n)).astype(np.float32)
        acts = rng.normal(0, 1, size=(64, m)).astype(np.float32)
        stats = salient.stats_from_layer_inputs(acts)
        layer = compress.compress_layer(delta, stats, compress.CompressionConfig(bits=bits, salient_k=k))
        man = compress.ArtifactManifest(model_id=name, domain="synthetic", base_digest="0" * 64,
                                        layer_count=1)
        blob = compress.serialize_artifact(compress.ExpertArtifact(manifest=man, layers=[layer]))
        with open(os.path.join(HERE, f"layer_{name}.mesw"), "wb") as f:
            f.write(blob)
        x = rng.normal(0, 1, size=(9, m)).astype(np.float32)
        arrays[f"{name}_x"] = x
        arrays[f"{name}_y"] = x @ layer.reconstruct()
        arrays[f"{name}_recon"] = layer.reconstruct()
        arrays[f"{name}_codes"] = layer.codes()
        arrays[f"{name}_salient"] = layer.salient.indices
        arrays[f"{name}_delta"] = delta            # compress_layer inputs (GPU compression parity)
        arrays[f"{name}_energy"] = stats.energy
        names.append(name)
    np.savez_compressed(os.path.join(HERE, "layer_expected.npz"), **arrays)
    kat_out["layers"] = names


def bad_fixtures(kat_out):
    with open(os.path.join(HERE, "layer_l2_200x130_k5.mesw"), "rb") as f:
        good = f.read()
    cases = {
        "bad_magic": b"MESX" + good[4:],
        "bad_version": good[:4] + (2).to_bytes(2, "little") + good[6:],
        "truncated": good[:-7],
        "trailing": good + b"\x00\x01",
    }
    expect = {}
    for name, blob in cases.items():
        with open(os.path.join(HERE, f"{name}.mesw"), "wb") as f:
            f.write(blob)
        try:
            compress.deserialize_artifact(blob)
            expect[name] = None
        except Exception as exc:  # record the reference's error class
            expect[name] = type(exc).__name__
    kat_out["bad"] = expect


def main():
    rng = np.random.default_rng(20240613)
    k = kat()
    codes_fixtures(rng)
    toy_fixtures(rng, k)
    layer_fixtures(rng, k)
    bad_fixtures(k)
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(k, f, indent=1, sort_keys=True)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    sys.exit(main())
