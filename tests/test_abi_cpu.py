"""CPU-side checks of the C ABI (no GPU compute): the library loads, exports every
symbol include/mesw.h declares, and its host-side container parser / byte
accounting match the oracle (and through it, the reference)."""

import json
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from oracle import mesw as om
from paper_2406_09041_b200 import _lib, compress, errors


def _header_symbols():
    with open(os.path.join(ROOT, "include", "mesw.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(mesw_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = _header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), f"libmesw.so does not export {s}"
    assert sorted(_lib.SYMBOLS) == syms
    assert L.mesw_abi_version() == 2


def test_packed_and_block_sizes():
    L = _lib.lib()
    for (m, n, b, k) in [(4096, 4096, 2, 8), (4096, 14336, 2, 8), (4096, 4096, 1, 0), (37, 5, 3, 2), (1, 1, 8, 0)]:
        assert L.mesw_packed_nbytes(m, n, b) == om.packed_nbytes(m, n, b)
        assert L.mesw_layer_block_nbytes(m, n, b, k) == om.layer_block_nbytes(m, n, b, k)
        assert compress.layer_block_nbytes(m, n, b, k).total == om.layer_block_nbytes(m, n, b, k)
    assert [L.mesw_device_code_bits(b) for b in (1, 2, 3, 4, 8, 5)] == [4, 2, 4, 4, 8, 0]


def _read(name):
    with open(os.path.join(GOLDEN, name), "rb") as f:
        return f.read()


def test_parse_matches_oracle_on_golden_artifacts():
    names = [f for f in os.listdir(GOLDEN) if f.endswith(".mesw") and not f.startswith(("bad", "trunc", "trail"))]
    assert names
    for name in names:
        blob = _read(name)
        art = compress.deserialize_artifact(blob)
        man, layers = om.parse_artifact(blob)
        assert art.manifest.layer_count == man["layer_count"] == len(layers)
        for a, o in zip(art.layers, layers):
            assert (a.rows, a.cols, a.bits, a.salient.k) == (o.m, o.n, o.bits, o.k)
            assert np.array_equal(a.salient.indices, o.salient_idx)
            assert np.array_equal(a.salient_rows.view(np.uint16), o.salient_rows.view(np.uint16))
            assert np.array_equal(a.steps, o.steps)
            assert a.packed.data == o.packed
        assert compress.serialize_artifact(art) == blob
        assert compress.compressed_size_bytes(art).total == len(blob)


def test_malformed_containers_raise_reference_errors():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        expected = json.load(f)["bad"]
    for name, cls_name in expected.items():
        with pytest.raises(getattr(errors, cls_name)):
            compress.deserialize_artifact(_read(f"{name}.mesw"))
    with pytest.raises(errors.TruncatedArtifactError):
        compress.deserialize_artifact(b"MES")
    with pytest.raises(errors.BadMagicError):
        compress.deserialize_artifact(b"XXXX\x01\x00")
    assert issubclass(errors.TruncatedArtifactError, errors.ArtifactError)


def test_salient_tables_layout():
    from paper_2406_09041_b200.device import LinearGeometry, build_salient_tables
    rng = np.random.default_rng(3)
    blocks = [om.random_layer(rng, 200, 300, 2, 5), om.random_layer(rng, 200, 128, 2, 0),
              om.random_layer(rng, 200, 70, 2, 3)]
    art_blocks = [compress.deserialize_artifact(om.serialize_artifact(
        {"model_id": "x", "domain": "d", "base_digest": "0", "layer_count": 1}, [b])).layers[0] for b in blocks]
    geom = LinearGeometry(200, (300, 128, 70))
    assert geom.col_base == (0, 384, 512) and geom.n_pad == 768 and geom.n == 582
    off, idx, rows = build_salient_tables(art_blocks, geom)
    off, idx, rows = off.numpy(), idx.numpy(), rows.numpy().view(np.uint16)
    assert off.tolist() == [0, 5, 10, 15, 15, 18, 18]
    for cg in range(5):
        for r in range(off[cg], off[cg + 1]):
            b = 0 if cg < 3 else 2
            cb = geom.col_base[b]
            rr = r - off[cg]
            assert idx[r] == blocks[b].salient_idx[rr]
            for c in range(128):
                jl = cg * 128 + c - cb
                want = blocks[b].salient_rows.view(np.uint16)[rr, jl] if jl < blocks[b].n else 0
                assert rows[r, c] == want


def test_launch_width_candidates():
    """device.cta_candidates: all-SM default, narrower grids, and the aligned k-split width."""
    from paper_2406_09041_b200.device import LinearGeometry, cta_candidates
    o_proj = LinearGeometry(4096, (4096,))       # 16 column-group pairs x 32 k-steps
    c = cta_candidates(o_proj, 148)
    assert c[0] == 0 and all(x % 2 == 0 and x <= 148 for x in c)
    assert 128 in c                              # 16 pairs x 4 aligned k-splits = 64 pairs
    down = LinearGeometry(14336, (4096,))        # 112 k-steps: 4 splits of 28
    assert 128 in cta_candidates(down, 148)
    gu = LinearGeometry(4096, (14336, 14336))    # 112 pairs > 74: no aligned split
    assert all(x <= 148 for x in cta_candidates(gu, 148))
