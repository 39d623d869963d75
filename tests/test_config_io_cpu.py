"""CPU parity of the §8(f) host rows against fixtures generated from the real
reference (tests/golden/make_golden_io.py -> io_golden.json): JSON config
documents (parse, validation messages, canonical serialisation) and the SRTF
and CSV writers/readers on host-resident fields."""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2603_28160_b200 as ms
from paper_2603_28160_b200 import config as cfgmod
from paper_2603_28160_b200 import surface_io

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "io_golden.json")))


def _bits_equal(a, b):
    if isinstance(a, float) and isinstance(b, float):
        return np.float64(a).tobytes() == np.float64(b).tobytes()
    if isinstance(a, dict) and isinstance(b, dict):
        return a.keys() == b.keys() and all(_bits_equal(a[k], b[k]) for k in a)
    if isinstance(a, (list, tuple)) and isinstance(b, (list, tuple)):
        return len(a) == len(b) and all(_bits_equal(x, y) for x, y in zip(a, b))
    return a == b and type(a) is type(b)


@pytest.mark.parametrize("name", sorted(GOLD["configs"]["good"]))
def test_parse_and_serialize_match_reference(name):
    g = GOLD["configs"]["good"][name]
    doc = ms.parse_config(g["text"])
    ser = ms.serialize_config(doc)
    assert _bits_equal(json.loads(json.dumps(ser)), g["serialized"]), (ser, g["serialized"])
    p = doc.process
    assert _bits_equal([p.angular_velocity_rad_s, p.feed_speed_mm_s, p.feed_per_tooth_mm, p.spindle_speed_rpm],
                       g["kinematics"])
    assert [doc.grid.m, doc.grid.n] == g["grid_mn"]
    # parse(serialize(doc)) == doc (config.py:392-398 round trip)
    assert ms.parse_config(json.dumps(ser)) == doc


@pytest.mark.parametrize("name", sorted(GOLD["configs"]["bad"]))
def test_config_errors_match_reference(name):
    g = GOLD["configs"]["bad"][name]
    with pytest.raises(ms.MillsurfError) as err:
        ms.parse_config(g["text"])
    assert type(err.value).__name__ == g["type"]
    assert str(err.value) == g["message"]


def test_extensions_block_round_trip():
    raw = json.loads(GOLD["configs"]["good"]["case1_raw"]["text"])
    raw["extensions"] = {"profile": "ball", "tilt_rad": 0.2, "passes": 3, "stepover_mm": 0.3}
    doc = ms.parse_config(json.dumps(raw))
    assert doc.extensions == ms.Extensions(profile="ball", tilt_rad=0.2, passes=3, stepover_mm=0.3)
    again = ms.parse_config(json.dumps(ms.serialize_config(doc)))
    assert again == doc
    raw["extensions"]["bogus"] = 1
    with pytest.raises(ms.ConfigError, match="extensions.bogus: unknown key"):
        ms.parse_config(json.dumps(raw))
    # a reference document never carries the block and serialises without it
    assert "extensions" not in ms.serialize_config(ms.parse_config(GOLD["configs"]["good"]["case1_raw"]["text"]))


def _field(case):
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", f"{case}.npz"))
    gr = json.loads(str(g["config_json"]))["grid"]
    sent = json.loads(str(g["counters_json"]))["initial_height"]
    spec = ms.GridSpec(gr["spacing_mm"], gr["x_min_mm"], gr["y_min_mm"], gr["m"], gr["n"])
    return ms.HeightField(spec, sent, np.array(g["heights"], dtype=np.float64))


def _sha(p):
    return hashlib.sha256(open(p, "rb").read()).hexdigest()


@pytest.mark.parametrize("case", ["small_0", "cusp"])
def test_srtf_and_csv_bytes_match_reference(case, tmp_path):
    gold = GOLD["exports"][case]
    f = _field(case)
    surface_io.write_surface(f, tmp_path / "s.srtf")
    assert _sha(tmp_path / "s.srtf") == gold["srtf_sha256"]
    back = surface_io.read_surface(tmp_path / "s.srtf")
    assert back.spec == f.spec and back.initial_height_mm == f.initial_height_mm
    assert np.array_equal(back.heights, f.heights)
    assert not list(tmp_path.glob("*.tmp"))
    for name, ent in gold["rois"].items():
        roi = tuple(ent["roi"]) if ent["roi"] else None
        surface_io.write_heights_csv(f, tmp_path / f"{name}.csv", roi)
        assert _sha(tmp_path / f"{name}.csv") == ent["csv_sha256"], name


def test_srtf_reader_rejects_corrupt_files(tmp_path):
    f = _field("small_0")
    p = tmp_path / "s.srtf"
    surface_io.write_surface(f, p)
    blob = p.read_bytes()
    cases = {"short": blob[:20], "truncated": blob[:-8], "oversized": blob + b"\0" * 8,
             "magic": b"XRTF" + blob[4:], "version": blob[:4] + (2).to_bytes(4, "little") + blob[8:]}
    msgs = {"short": "shorter than the 48-byte header", "truncated": "header promises",
            "oversized": "header promises", "magic": "bad magic", "version": "unsupported format version 2"}
    for k, b in cases.items():
        q = tmp_path / f"{k}.srtf"
        q.write_bytes(b)
        with pytest.raises(ms.SurfaceFormatError, match=msgs[k]):
            surface_io.read_surface(q)
    assert len(blob) == 48 + f.spec.node_count * 8


def test_dataset_overrides_match_reference_semantics():
    from paper_2603_28160_b200.dataset import apply_overrides

    for name, run in GOLD["datasets"].items():
        base = run["base_raw"]
        rows = [json.loads(x) for x in run["manifest"].strip().split("\n")]
        header, rows = rows[0], rows[1:]
        assert header["base_config"] == base
        ranges = [ms.ParameterRange(*r) for r in run["ranges"]]
        samples = ms.lhs_sample(ranges, run["count"], run["seed"])
        names = [r.name for r in ranges]
        for row in rows:
            vals = samples[row["index"]]
            assert _bits_equal(row["params"], {n: float(v) for n, v in zip(names, vals)})
            raw = apply_overrides(base, names, vals)
            if row["status"] == "ok":
                doc = ms.parse_config(json.dumps(raw))
                assert doc.grid.node_count > 0
            else:
                with pytest.raises(ms.MillsurfError) as err:
                    doc = ms.config_from_dict(raw)
                    from paper_2603_28160_b200.planner import plan
                    plan(doc.to_simulation_config())
                assert str(err.value) == row["error"]
