"""ETE1 / CSV / JSON formats pinned to the reference's bytes, and the CLI surface
(mirror of /root/reference/pkg/tests/test_io_cli.py's format and exit-code checks)."""

import json
import os
import struct

import numpy as np
import pytest

from paper_1401_4068_b200 import cli, io_formats
from paper_1401_4068_b200.data import AnalysisConfig, EnsembleSeries, TEResult
from paper_1401_4068_b200.exceptions import GridIncomplete, MagicMismatch, ParseError

GOLD = os.path.join(os.path.dirname(__file__), "golden")
VALS = np.random.default_rng(7).standard_normal((3, 5))


def test_reads_reference_files():
    for fmt in ("bin", "csv"):
        s = io_formats.load_ensemble(os.path.join(GOLD, f"io_ref.{fmt}"), fmt)
        assert np.array_equal(s.values, VALS)
    assert io_formats.load_ensemble(os.path.join(GOLD, "io_ref.bin")).channel_name == "chan-α"


def test_writes_reference_bytes(tmp_path):
    s = EnsembleSeries("chan-α", VALS)
    for fmt in ("bin", "csv"):
        out = tmp_path / f"x.{fmt}"
        io_formats.save_ensemble(s, out, fmt)
        assert out.read_bytes() == open(os.path.join(GOLD, f"io_ref.{fmt}"), "rb").read()


def test_results_json_matches_reference(tmp_path):
    res = TEResult(source="X", target="Y", window=(10, 20), u_selected=3, te_value=0.125,
                   surrogate_values=np.array([0.01, 0.02, 0.5]), p_value=1 / 3,
                   significant=False, significant_corrected=False,
                   te_minus_median_surrogate=0.105, te_curve=[(1, 0.1), (3, 0.125)])
    cfg = AnalysisConfig(u_candidates=(1, 3), window=(10, 20), k=4, n_surrogates=3, seed=5)
    out = tmp_path / "r.json"
    io_formats.write_results([res], out, cfg, timestamp=False)
    assert json.load(open(out)) == json.load(open(os.path.join(GOLD, "io_ref_results.json")))


def test_format_errors(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"XXXX" + b"\0" * 12)
    with pytest.raises(MagicMismatch):
        io_formats.load_ensemble(bad)
    trunc = tmp_path / "t.bin"
    trunc.write_bytes(b"ETE1" + struct.pack("<III", 2, 3, 1) + b"a" + b"\0" * 20)
    with pytest.raises(ParseError):
        io_formats.load_ensemble(trunc)
    holes = tmp_path / "h.csv"
    holes.write_text("rep,t,value\n1,1,0.5\n2,2,0.25\n")
    with pytest.raises(GridIncomplete):
        io_formats.load_ensemble(holes, "csv")


def test_cli_exit_codes(tmp_path, capsys):
    assert cli.main(["validate", str(tmp_path / "missing.bin")]) == 2
    assert cli.main(["bench", "--chunks", "x,y", "--out", str(tmp_path / "b.csv")]) == 1
    assert cli.main(["nonsense"]) == 1
    prefix = str(tmp_path / "sim")
    assert cli.main(["simulate", "ar", "--scenario", "unidirectional", "--reps", "4",
                     "--samples", "60", "--out", prefix]) == 0
    assert cli.main(["validate", prefix + "_X.bin"]) == 0
    assert cli.main(["analyze", "--source", prefix + "_X.bin", "--target", prefix + "_Y.bin",
                     "--window", "30:40", "--u", "1:2", "--ragwitz", "--ragwitz-dims", "x",
                     "--out", str(tmp_path / "o.json")]) == 1
    assert cli.main(["analyze", "--source", prefix + "_X.bin", "--target", prefix + "_Y.bin",
                     "--window", "40:30", "--u", "1", "--out", str(tmp_path / "o.json")]) == 1


@pytest.mark.gpu
def test_cli_analyze_matches_api(tmp_path):
    from paper_1401_4068_b200 import EmbeddingSpec, analyze_pair
    prefix = str(tmp_path / "sim")
    cli.main(["simulate", "ar", "--scenario", "unidirectional", "--reps", "12",
              "--samples", "200", "--seed", "3", "--out", prefix])
    out = tmp_path / "o.json"
    curve = tmp_path / "c.csv"
    assert cli.main(["scan-delay", "--source", prefix + "_X.bin", "--target", prefix + "_Y.bin",
                     "--window", "100:140", "--u", "1:3", "--dim", "2", "--surrogates", "20",
                     "--out", str(out), "--curve-out", str(curve)]) == 0
    doc = json.load(open(out))["results"][0]
    x = io_formats.load_ensemble(prefix + "_X.bin")
    y = io_formats.load_ensemble(prefix + "_Y.bin")
    res = analyze_pair(x, y, EmbeddingSpec(2, 1), EmbeddingSpec(2, 1),
                       AnalysisConfig(u_candidates=(1, 2, 3), window=(100, 140), k=4,
                                      n_surrogates=20, seed=0))
    assert doc["te_value"] == res.te_value and doc["p_value"] == res.p_value
    assert doc["te_curve"] == [[u, t] for u, t in res.te_curve]
    assert curve.read_text().splitlines()[0] == "u,te_nats"
