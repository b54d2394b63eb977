"""Pin the oracle restatement against the real reference's outputs (golden fixtures
made by tests/golden/make_golden.py from /root/reference)."""

import json
import os

import numpy as np
import pytest

from oracle import mesw as om
from oracle import toylm as ot

from conftest import GOLDEN


def _kat():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        return json.load(f)


def _read(name):
    with open(os.path.join(GOLDEN, name), "rb") as f:
        return f.read()


def test_spec_pack_kats():
    k = _kat()
    assert om.pack_codes(np.array([[-2], [-1], [0], [1]]), 2).hex() == k["pack_b2"] == "e4"
    assert om.pack_codes(np.array([[1], [1], [-1], [-1], [1], [1], [-1], [-1]]), 1).hex() == k["pack_b1"] == "33"
    assert om.pack_codes(np.array([[-4], [3], [0]]), 3).hex() == k["pack_b3"]
    assert om.unpack_codes(bytes.fromhex("e4"), 4, 1, 2).ravel().tolist() == [-2, -1, 0, 1]


def test_size_arithmetic():
    k = _kat()
    s = k["size_4096x4096_b2_k8"]
    assert om.layer_block_nbytes(4096, 4096, 2, 8) == s["total"] == 4276273
    assert om.packed_nbytes(4096, 4096, 2) == s["codes"] == 4194304
    assert om.layer_block_nbytes(4096, 14336, 2, 8) == k["size_4096x14336_b2_k8_total"]
    assert om.layer_block_nbytes(4096, 4096, 1, 0) == k["size_4096x4096_b1_k0_total"]
    assert om.layer_block_nbytes(4096, 4096, 4, 8) == k["size_4096x4096_b4_k8_total"]


@pytest.mark.parametrize("bits", [1, 2, 3, 4, 8])
def test_unpack_matches_reference(bits):
    z = np.load(os.path.join(GOLDEN, "codes.npz"))
    keys = [k[:-6] for k in z.files if k.startswith(f"b{bits}_") and k.endswith("_codes")]
    assert keys
    for key in keys:
        codes = z[key + "_codes"]
        packed = z[key + "_packed"].tobytes()
        m, n = codes.shape
        assert np.array_equal(om.unpack_codes(packed, m, n, bits), codes)
        assert om.pack_codes(codes, bits) == packed


def test_unpack_rejects_bad_length():
    with pytest.raises(ValueError):
        om.unpack_codes(b"\x00" * 3, 4, 4, 2)


def test_parse_and_reconstruct_layers():
    k = _kat()
    z = np.load(os.path.join(GOLDEN, "layer_expected.npz"))
    for name in k["layers"]:
        blob = _read(f"layer_{name}.mesw")
        man, layers = om.parse_artifact(blob)
        assert man["layer_count"] == 1
        L = layers[0]
        assert np.array_equal(L.codes(), z[f"{name}_codes"])
        assert np.array_equal(L.salient_idx, z[f"{name}_salient"])
        assert np.array_equal(L.reconstruct(), z[f"{name}_recon"])
        # the serializer restatement is byte-identical to the reference's
        assert om.serialize_artifact(man, layers) == blob
        # SPEC.md:432 fused delta_matvec == dequantize-then-matvec within 1e-5 rel
        x = z[f"{name}_x"]
        y = om.delta_matvec_batch(x, L)
        ref = z[f"{name}_y"]
        assert np.max(np.abs(y - ref)) <= 1e-5 * np.max(np.abs(ref)) + 1e-12


def test_bad_containers():
    k = _kat()
    cls = {"BadMagicError": om.OracleBadMagic, "UnsupportedVersionError": om.OracleUnsupportedVersion,
           "TruncatedArtifactError": om.OracleTruncated}
    for name, expected in k["bad"].items():
        with pytest.raises(cls[expected]):
            om.parse_artifact(_read(f"{name}.mesw"))


def test_toy_forward_with_delta_matches_reference():
    zb = np.load(os.path.join(GOLDEN, "toy_base.npz"))
    ze = np.load(os.path.join(GOLDEN, "toy_expected.npz"))
    base = ot.ToyWeights(zb["embedding"], [zb[f"layer{i}"] for i in range(4)], zb["head"])
    toks = ze["tokens"]
    np.testing.assert_allclose(ot.forward(base, toks), ze["base_logits"], rtol=1e-5, atol=1e-5)
    assert ot.greedy_decode(base, ze["prompt"], 12) == ze["greedy_base"].tolist()
    for e in range(3):
        _, layers = om.parse_artifact(_read(f"toy_expert_{e}.mesw"))
        for li, L in enumerate(layers):
            assert np.array_equal(L.codes(), ze[f"codes_{e}_{li}"])
            assert np.array_equal(L.reconstruct(), ze[f"recon_{e}_{li}"])
        provs = [ot.OracleCompressedProvider(L) for L in layers]
        np.testing.assert_allclose(ot.forward_with_delta(base, provs, toks), ze[f"fwd_delta_{e}"],
                                   rtol=1e-5, atol=1e-5)
        assert ot.greedy_decode(base, ze["prompt"], 12, provs) == ze[f"greedy_{e}"].tolist()


def test_base_digest_matches_reference_manifests():
    """toylm.base_digest (toylm.py:115-120): the toy experts were compressed against toy_base."""
    from oracle import mesw as om
    from paper_2406_09041_b200.infer import base_digest
    z = np.load(os.path.join(GOLDEN, "toy_base.npz"))
    mats = [z["embedding"]] + [z[f"layer{i}"] for i in range(4)] + [z["head"]]
    with open(os.path.join(GOLDEN, "toy_expert_0.mesw"), "rb") as f:
        man, _ = om.parse_artifact(f.read())
    assert base_digest(mats) == man["base_digest"]


def test_mistral_shape_reference_block():
    """The k_proj-shaped block made by the reference's compress_layer (make_mistral_golden.py):
    the oracle parses it and its reconstruct() hashes to the reference's own; x @ recon matches."""
    import hashlib
    import json
    with open(os.path.join(GOLDEN, "kat_mistral.json")) as f:
        kat = json.load(f)
    _, (L,) = om.parse_artifact(_read(kat["file"]))
    assert (L.m, L.n, L.bits, L.k) == (kat["m"], kat["n"], kat["bits"], kat["k"])
    assert L.salient_idx.tolist() == kat["salient"]
    recon = L.reconstruct()
    assert hashlib.sha256(np.ascontiguousarray(recon, "<f4").tobytes()).hexdigest() == kat["recon_sha256"]
    x = np.random.default_rng(7).normal(0, 1, size=(4, L.m)).astype(np.float32)
    np.testing.assert_allclose(om.delta_matvec_batch(x, L), np.load(os.path.join(GOLDEN, "ref_kproj_y.npy")),
                               rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("m", [4, 7, 200, 4096])
def test_vectorised_2bit_unpack_equals_window_decode(m):
    rng = np.random.default_rng(m)
    L = om.random_layer(rng, m, 37, 2, min(3, m))
    assert np.array_equal(L.codes(), L.unpack_generic())
