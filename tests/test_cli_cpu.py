"""CLI surface on the CPU (SPEC cli-analytics): the compression-ratio
report reproduces the paper's Fig. 6 / Fig. 7 numbers (acceptance criterion 1), `inspect`
reads a reference-made artifact, errors are one machine-parseable line with a non-zero exit."""
import os

import pytest

from paper_2406_09041_b200 import cli

HERE = os.path.dirname(os.path.abspath(__file__))


def test_compression_ratio_paper_numbers():
    assert abs(cli.compression_ratio(13.48, 2.13, 3.42, 3) - 1.74) <= 0.005    # abstract "1.74x"
    assert abs(cli.compression_ratio(24.23, 3.60, 3.42, 9) - 3.63) <= 0.005    # §4.3 "3.63x"
    assert cli.compression_ratio(1.0, 1.0, 0.0, 1) == 0.5
    r = [cli.compression_ratio(13.48, 2.13, 3.42, m) for m in range(1, 10)]
    assert all(b > a for a, b in zip(r, r[1:]))                                  # monotone in M
    assert abs(cli.compression_ratio(13.48, 2.13, 3.42, 10 ** 6) - 13.48 / 2.13) <= 1e-3 * 13.48 / 2.13


def test_report_ratio_csv(capsys):
    assert cli.main(["report", "ratio", "--psi", "13.48", "--psit", "2.13", "--phi", "3.42", "--m-range", "1..9"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "m,ratio" and len(lines) == 10
    m3 = lines[3].split(",")
    assert m3[0] == "3" and abs(float(m3[1]) - 1.74) <= 0.005


def test_inspect_reference_artifact(capsys):
    assert cli.main(["inspect", os.path.join(HERE, "golden", "layer_l2_256x384_k8.mesw")]) == 0
    out = capsys.readouterr().out
    assert '"layer_count": 1' in out and "0,256,384,2,8," in out


def test_errors_are_one_line_nonzero(tmp_path, capsys):
    bad = tmp_path / "bad.mesw"
    bad.write_bytes(b"NOPE" + b"\0" * 20)
    assert cli.main(["inspect", str(bad)]) == 1
    err = capsys.readouterr().err.strip().splitlines()
    assert len(err) == 1 and err[0].startswith("error: BadMagicError")
    assert cli.main(["report", "ratio", "--psi", "1", "--psit", "1", "--m-range", "5..2"]) == 1


def test_toyl_roundtrip(tmp_path):
    import numpy as np
    from types import SimpleNamespace
    rng = np.random.default_rng(0)
    m = SimpleNamespace(vocab=7, width=4, depth=2, embedding=rng.normal(size=(7, 4)).astype(np.float32),
                        layers=[rng.normal(size=(4, 4)).astype(np.float32) for _ in range(2)],
                        head=rng.normal(size=(4, 7)).astype(np.float32))
    cli.save_toyl(m, tmp_path / "m.toyl")
    back = cli.load_toyl(tmp_path / "m.toyl")
    assert np.array_equal(back.head, m.head) and back.depth == 2
    with pytest.raises(ValueError):
        (tmp_path / "t.toyl").write_bytes((tmp_path / "m.toyl").read_bytes()[:-5])
        cli.load_toyl(tmp_path / "t.toyl")
