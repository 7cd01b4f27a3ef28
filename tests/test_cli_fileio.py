"""File formats and the command line (reference fileio.py, cli.py:45-129).

CPU: PGM/PNG round trips, 8-bit rounding, and the CLI's exit codes for inputs
rejected before the fill.  GPU: a full `inpaint` run against the oracle.
"""

import json

import numpy as np
import pytest
from click.testing import CliRunner

from paper_1611_05319_b200 import FillParams, Spline, dumps, fileio
from paper_1611_05319_b200.cli import main


def test_to_uint8_rounds_half_away():
    v = np.array([0.0, 0.5 / 255, 1.5 / 255, 254.5 / 255, 1.0, -0.2, 1.3])
    assert fileio.to_uint8(v).tolist() == [0, 1, 2, 255, 255, 0, 255]


def test_pgm_round_trip_and_ascii(tmp_path):
    lab = np.zeros((5, 7), np.uint8)
    lab[1:3, 2:5] = 255
    lab[4, 0] = 128
    fileio.save_labels(tmp_path / "m.pgm", lab)
    assert np.array_equal(fileio.load_labels(tmp_path / "m.pgm"), lab)
    text = "P2\n# comment\n7 5\n255\n" + " ".join(str(int(x)) for x in lab.ravel()) + "\n"
    assert np.array_equal(fileio.parse_labels(text.encode()), lab)
    with pytest.raises(ValueError, match="maxval"):
        fileio.parse_labels(b"P5\n7 5\n65535\n" + lab.tobytes())
    with pytest.raises(ValueError, match="truncated"):
        fileio.parse_labels(b"P5\n7 5\n255\n" + lab.tobytes()[:10])
    bad = lab.copy()
    bad[0, 0] = 7
    with pytest.raises(ValueError, match="label mask holds value 7"):
        fileio.parse_labels(b"P5\n7 5\n255\n" + bad.tobytes())


def test_png_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    img = fileio.to_uint8(rng.random((6, 9, 3))).astype(np.float64) / 255.0
    fileio.save_image(tmp_path / "a.png", img)
    assert np.array_equal(fileio.load_image(tmp_path / "a.png"), img)


def test_cli_rejects_before_the_fill(tmp_path):
    fileio.save_image(tmp_path / "a.png", np.full((6, 9, 3), 0.5))
    fileio.save_labels(tmp_path / "m.pgm", np.zeros((6, 8), np.uint8))
    r = CliRunner().invoke(main, ["inpaint", "--image", str(tmp_path / "a.png"),
                                  "--mask", str(tmp_path / "m.pgm")])
    assert r.exit_code == 2 and "mask is 8x6 but image is 9x6" in r.output
    r = CliRunner().invoke(main, ["inpaint", "--image", str(tmp_path / "nope.png"),
                                  "--mask", str(tmp_path / "m.pgm")])
    assert r.exit_code == 3 and "cannot read image" in r.output
    r = CliRunner().invoke(main, ["inpaint", "--image", str(tmp_path / "a.png"),
                                  "--mask", str(tmp_path / "m.pgm"), "--mu", "-1"])
    assert r.exit_code != 0


@pytest.mark.gpu
def test_cli_inpaint_matches_oracle(tmp_path):
    from oracle import guidefill_oracle as orc
    from paper_1611_05319_b200 import scenes

    sc = scenes.small_scene(64, 96, band=6, gx=3, gy=2, n_spl=2, seed=4)
    img = fileio.to_uint8(sc.image).astype(np.float64) / 255.0  # what the PNG holds
    fileio.save_image(tmp_path / "in.png", img)
    fileio.save_labels(tmp_path / "m.pgm", sc.labels)
    spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"],
                  kind=s["kind"]) for s in sc.splines]
    (tmp_path / "s.json").write_text(dumps(spl))
    r = CliRunner().invoke(main, ["inpaint", "--image", str(tmp_path / "in.png"),
                                  "--mask", str(tmp_path / "m.pgm"),
                                  "--splines", str(tmp_path / "s.json"),
                                  "--out", str(tmp_path / "out.png"),
                                  "--report", str(tmp_path / "rep.json"), "--r", "3"])
    assert r.exit_code == 0, r.output
    field = orc.guide_field([orc.polyline(s["points"], s["kind"]) for s in sc.splines],
                            [s["direction"] for s in sc.splines], sc.labels)
    ref = orc.fill(img, sc.labels, field, orc.Params.of(FillParams.guidefill(r=3)), tracked=True)
    out = fileio.load_image(tmp_path / "out.png")
    assert np.abs(out - fileio.to_uint8(ref["u"]) / 255.0).max() <= 1.0 / 255 + 1e-12
    rep = json.loads((tmp_path / "rep.json").read_text())
    assert rep["iterations"] == ref["iterations"] and rep["tracked"] is True


@pytest.mark.gpu
def test_cli_coherence_preset_matches_oracle(tmp_path):
    """`guidefill inpaint --preset coherence_transport` needs no splines (cli.py:97-106):
    g comes from the masked structure tensor on the device."""
    from oracle import guidefill_oracle as orc
    from paper_1611_05319_b200 import scenes

    sc = scenes.small_scene(64, 96, band=6, gx=3, gy=2, n_spl=2, seed=5)
    img = fileio.to_uint8(sc.image).astype(np.float64) / 255.0
    fileio.save_image(tmp_path / "in.png", img)
    fileio.save_labels(tmp_path / "m.pgm", sc.labels)
    r = CliRunner().invoke(main, ["inpaint", "--image", str(tmp_path / "in.png"),
                                  "--mask", str(tmp_path / "m.pgm"),
                                  "--preset", "coherence_transport",
                                  "--out", str(tmp_path / "out.png"),
                                  "--report", str(tmp_path / "rep.json")])
    assert r.exit_code == 0, r.output
    ref = orc.fill(img, sc.labels, None, orc.Params.of(FillParams.coherence_transport()),
                   tracked=True)
    out = fileio.load_image(tmp_path / "out.png")
    assert np.abs(out - fileio.to_uint8(ref["u"]) / 255.0).max() <= 1.0 / 255 + 1e-12
    rep = json.loads((tmp_path / "rep.json").read_text())
    assert rep["iterations"] == ref["iterations"]
    assert rep["frontier_sizes"] == [x[1] for x in ref["rows"]]
    assert rep["filled_per_iteration"] == [x[4] for x in ref["rows"]]


@pytest.mark.gpu
def test_cli_inpaint_autodetects_splines(tmp_path):
    """Without --splines the default guidefill preset detects splines
    (cli.py:104-105, guide.detect_splines on the device): the fill equals the
    oracle's with the oracle's detected splines; `splines detect` writes the
    canonical JSON (test_cli.py:136-148)."""
    from oracle import detect_oracle as det
    from oracle import guidefill_oracle as orc
    from paper_1611_05319_b200 import loads, scenes

    sc = scenes.small_scene(120, 160, band=6, gx=3, gy=2, n_spl=2, seed=9)
    img = fileio.to_uint8(sc.image).astype(np.float64) / 255.0
    fileio.save_image(tmp_path / "in.png", img)
    fileio.save_labels(tmp_path / "m.pgm", sc.labels)
    r = CliRunner().invoke(main, ["inpaint", "--image", str(tmp_path / "in.png"),
                                  "--mask", str(tmp_path / "m.pgm"),
                                  "--out", str(tmp_path / "out.png"),
                                  "--report", str(tmp_path / "rep.json")])
    assert r.exit_code == 0, r.output
    want = det.detect_splines(img, sc.labels)
    field = orc.guide_field([np.stack([s, e]) for s, e, _ in want], [d for _, _, d in want],
                            sc.labels)
    ref = orc.fill(img, sc.labels, field, orc.Params.of(FillParams.guidefill()), tracked=True)
    rep = json.loads((tmp_path / "rep.json").read_text())
    assert rep["filled_per_iteration"] == [x[4] for x in ref["rows"]]
    out = fileio.load_image(tmp_path / "out.png")
    assert np.abs(out - fileio.to_uint8(ref["u"]) / 255.0).max() <= 1.0 / 255 + 1e-12
    r = CliRunner().invoke(main, ["splines", "detect", "--image", str(tmp_path / "in.png"),
                                  "--mask", str(tmp_path / "m.pgm"),
                                  "--out", str(tmp_path / "det.json")])
    assert r.exit_code == 0, r.output
    text = (tmp_path / "det.json").read_text()
    assert dumps(loads(text)) == text
    assert len(loads(text)) == len(want)
