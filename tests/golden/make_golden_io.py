"""Golden fixtures for the §8(f) rows next to the hot path — JSON config
documents, SRTF / CSV / PGM exports and dataset manifests — generated from the
REAL reference (mounted read-only at /root/reference/pkg in the build
container only; the GPU box reads the committed files). Usage:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_io.py

Writes tests/golden/io_golden.json:
  * ``configs``: for every reference config file under pkg/configs and the
    test_config.py variants, ``serialize_config(parse_config(text))`` and the
    derived kinematics; for a list of broken documents the exception class and
    message (config.py error conventions);
  * ``exports``: for the small_0 golden field (tests/golden/small_0.npz) the
    SHA-256 of write_surface's SRTF bytes and, per ROI, of write_graymap's PGM
    and write_heights_csv's CSV bytes, plus export_views' metrics JSON text;
  * ``datasets``: generate_dataset runs of test_dataset.py's base config
    (manifest text, SHA-256 of every surface file) including a run with
    failing samples (grid spacing beyond the patch).
The reference's output directories live under a temporary directory.
"""

from __future__ import annotations

import copy
import hashlib
import json
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg"
sys.dont_write_bytecode = True
sys.path.insert(0, os.path.join(REF, "src"))

import millsurf  # noqa: E402
from millsurf import surface_io  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def case1_raw():
    # test_config.py:9-36 shape (values typed here, not copied)
    return {
        "tool": {"cutting_diameter_mm": 10.0, "insert_radius_mm": 5.0, "tooth_count": 2,
                 "radial_rake_deg": 0.6, "axial_rake_deg": 0.0, "runouts_mm": [[0.0, 0.0], [0.011, 0.003]]},
        "process": {"cutting_speed_m_min": 170.0, "feed_per_tooth_mm": 0.6, "depth_of_cut_mm": 0.5,
                    "initial_position_mm": {"x": 0.0, "y": None, "z": 0.0}},
        "grid": {"spacing_mm": 0.01, "x_min_mm": -5.0, "x_max_mm": 5.0, "y_min_mm": 0.0, "y_max_mm": 5.0},
        "engine": {"edge_points": 40, "workers": 2},
        "output": {"formats": ["surface", "csv"], "basename": "case1"},
    }


def config_docs():
    docs = {}
    for name in sorted(os.listdir(os.path.join(REF, "configs"))):
        if name.endswith(".json") and name != "dataset_example.json":
            docs[name] = open(os.path.join(REF, "configs", name)).read()
    docs["case1_raw"] = json.dumps(case1_raw())
    v = case1_raw()
    v["engine"]["span_s"] = [0.0, 0.0123]
    v["process"]["initial_position_mm"]["y"] = -7.5
    v["process"]["phase_deg"] = 12.75
    docs["span_phase"] = json.dumps(v)
    v = case1_raw()
    for k in ("cutting_speed_m_min", "feed_per_tooth_mm"):
        del v["process"][k]
    v["process"].update(spindle_speed_rpm=995.0, feed_speed_mm_min=125.0, depth_of_cut_mm=2.5)
    v["tool"].update(tooth_count=4, runouts_mm=[[0.0, 0.0]] * 4)
    docs["rpm_feed_speed"] = json.dumps(v)
    v = case1_raw()
    del v["engine"], v["output"]
    docs["no_engine_output"] = json.dumps(v)
    v = case1_raw()
    v["process"]["spindle_speed_rpm"] = 1000.0 * 170.0 / (np.pi * 10.0)
    docs["consistent_speed_pair"] = json.dumps(v)
    v = case1_raw()
    v["tool"]["radial_rake_rad"] = 0.01
    del v["tool"]["radial_rake_deg"]
    v["engine"] = {"max_step_angle_rad": 0.002, "time_step_s": 1e-5, "record_trajectory": True}
    docs["rad_twins"] = json.dumps(v)
    return docs


def broken_docs():
    out = {"malformed": "{not json"}

    def mod(fn):
        r = case1_raw()
        fn(r)
        return json.dumps(r)

    out["unknown_key"] = mod(lambda r: r["tool"].__setitem__("ratial_rake_deg", 0.6))
    out["negative_feed"] = mod(lambda r: r["process"].__setitem__("feed_per_tooth_mm", -0.1))
    out["inconsistent_speed"] = mod(lambda r: r["process"].__setitem__("spindle_speed_rpm", 4000.0))
    out["inconsistent_feed"] = mod(lambda r: r["process"].__setitem__("feed_speed_mm_min", 999.0))
    out["no_speed"] = mod(lambda r: r["process"].pop("cutting_speed_m_min"))
    out["depth_beyond_radius"] = mod(lambda r: r["process"].__setitem__("depth_of_cut_mm", 6.0))
    out["runout_count"] = mod(lambda r: r["tool"].__setitem__("runouts_mm", [[0.0, 0.0]]))
    out["runout_large"] = mod(lambda r: r["tool"].__setitem__("runouts_mm", [[0.0, 0.0], [6.0, 0.0]]))
    out["deg_and_rad"] = mod(lambda r: r["tool"].__setitem__("radial_rake_rad", 0.01))
    out["span_needs_y"] = mod(lambda r: r["engine"].__setitem__("span_s", [0.0, 0.01]))
    out["bad_span"] = mod(lambda r: (r["engine"].__setitem__("span_s", [0.02, 0.01]),
                                     r["process"]["initial_position_mm"].__setitem__("y", -7.5)))
    out["unknown_format"] = mod(lambda r: r["output"].__setitem__("formats", ["surface", "tiff"]))
    out["empty_grid"] = mod(lambda r: r["grid"].__setitem__("x_max_mm", -5.0))
    out["sub_cell_grid"] = mod(lambda r: r["grid"].update(spacing_mm=20.0))
    out["bool_teeth"] = mod(lambda r: r["tool"].__setitem__("tooth_count", True))
    out["null_required"] = mod(lambda r: r["grid"].__setitem__("spacing_mm", None))
    out["not_object"] = json.dumps([1, 2])
    out["missing_tool"] = mod(lambda r: r.pop("tool"))
    out["rake_90"] = mod(lambda r: r["tool"].__setitem__("axial_rake_deg", 90.0))
    out["edge_points_1"] = mod(lambda r: r["engine"].__setitem__("edge_points", 1))
    out["record_not_bool"] = mod(lambda r: r["engine"].__setitem__("record_trajectory", 1))
    out["basename_empty"] = mod(lambda r: r["output"].__setitem__("basename", ""))
    out["inf_number"] = mod(lambda r: r["tool"].__setitem__("cutting_diameter_mm", float("inf")))
    out["string_number"] = mod(lambda r: r["grid"].__setitem__("x_min_mm", "-5"))
    out["float_teeth"] = mod(lambda r: r["tool"].__setitem__("tooth_count", 2.0))
    out["bad_pos_key"] = mod(lambda r: r["process"]["initial_position_mm"].__setitem__("w", 1.0))
    out["span_not_list"] = mod(lambda r: r["engine"].__setitem__("span_s", 5))
    out["formats_empty"] = mod(lambda r: r["output"].__setitem__("formats", []))
    return out


def gen_configs():
    good = {}
    for k, text in config_docs().items():
        doc = millsurf.parse_config(text)
        p = doc.process
        good[k] = {"text": text, "serialized": millsurf.serialize_config(doc),
                   "kinematics": [p.angular_velocity_rad_s, p.feed_speed_mm_s, p.feed_per_tooth_mm,
                                  p.spindle_speed_rpm], "grid_mn": [doc.grid.m, doc.grid.n]}
    bad = {}
    for k, text in broken_docs().items():
        try:
            millsurf.parse_config(text)
            raise SystemExit(f"broken doc {k} parsed")
        except millsurf.MillsurfError as exc:
            bad[k] = {"text": text, "type": type(exc).__name__, "message": str(exc)}
    return {"good": good, "bad": bad}


def _golden_field(name):
    g = np.load(os.path.join(OUT, f"{name}.npz"), allow_pickle=False)
    gr = json.loads(str(g["config_json"]))["grid"]
    sentinel = json.loads(str(g["counters_json"]))["initial_height"]
    spec = millsurf.GridSpec(gr["spacing_mm"], gr["x_min_mm"], gr["y_min_mm"], gr["m"], gr["n"])
    return spec, millsurf.HeightField(spec, sentinel, np.array(g["heights"], dtype=np.float64))


def gen_exports(tmp):
    out = {}
    for case in ("small_0", "cusp"):
        spec, field = _golden_field(case)
        ent_case = {}
        p = os.path.join(tmp, "s.srtf")
        surface_io.write_surface(field, p)
        ent_case["srtf_sha256"] = sha(open(p, "rb").read())
        rois = {"full": None, "inner": [2, 3, spec.m - 4, spec.n - 2], "strip": [0, 5, spec.m, 9]}
        ent_case["rois"] = {}
        for name, roi in rois.items():
            ent = {"roi": roi}
            rt = tuple(roi) if roi else None
            q = os.path.join(tmp, f"{name}.pgm")
            try:
                surface_io.write_graymap(field, q, rt)
                ent["pgm_sha256"] = sha(open(q, "rb").read())
            except millsurf.MillsurfError as exc:
                ent["pgm_error"] = str(exc)
            q = os.path.join(tmp, f"{name}.csv")
            surface_io.write_heights_csv(field, q, rt)
            ent["csv_sha256"] = sha(open(q, "rb").read())
            try:
                ent["metrics_json"] = json.dumps(millsurf.areal_metrics(field, rt).to_json_dict(), indent=2) + "\n"
            except millsurf.MillsurfError as exc:
                ent["metrics_error"] = str(exc)
            ent_case["rois"][name] = ent
        out[case] = ent_case
    spec, _ = _golden_field("small_0")
    flat = millsurf.HeightField(spec, 1.0, np.full(spec.node_count, 0.25))
    q = os.path.join(tmp, "flat.pgm")
    surface_io.write_graymap(flat, q)
    out["flat_pgm_sha256"] = sha(open(q, "rb").read())
    try:
        surface_io.write_graymap(millsurf.HeightField(spec, 1.0, None), q)
    except millsurf.MillsurfError as exc:
        out["uncut_pgm_error"] = str(exc)
    return out


def dataset_base():
    # test_dataset.py:9-22 shape
    return {"tool": {"cutting_diameter_mm": 10.0, "insert_radius_mm": 5.0, "tooth_count": 2},
            "process": {"cutting_speed_m_min": 170.0, "feed_per_tooth_mm": 0.3, "depth_of_cut_mm": 0.2,
                        "initial_position_mm": {"x": 0.0, "y": None, "z": 0.0}},
            "grid": {"spacing_mm": 0.05, "x_min_mm": -0.3, "x_max_mm": 0.3, "y_min_mm": 0.0, "y_max_mm": 0.3},
            "engine": {"max_step_angle_deg": 0.4}}


def gen_datasets(tmp):
    runs = {
        "feed_axial": ([("feed_per_tooth_mm", 0.2, 0.4), ("runout_axial_mm", -0.005, 0.005)], 3, 5, None),
        "feed4": ([("feed_per_tooth_mm", 0.2, 0.4)], 4, 9, None),
        "spacing_fail": ([("grid_spacing_mm", 0.05, 1.8)], 6, 2, None),
        "speed_depth_phase": ([("cutting_speed_m_min", 150.0, 250.0), ("depth_of_cut_mm", 0.1, 0.4),
                               ("phase_deg", 0.0, 90.0), ("radial_rake_deg", -5.0, 5.0)], 5, 11, None),
        "radial_runout_fine": ([("runout_radial_mm", 0.004, 0.005)], 2, 1, {"spacing_mm": 0.02}),
    }
    out = {}
    for name, (rg, count, seed, grid_over) in runs.items():
        base = dataset_base()
        if grid_over:
            base["grid"].update(grid_over)
        d = os.path.join(tmp, name)
        ranges = [millsurf.ParameterRange(*r) for r in rg]
        millsurf.generate_dataset(ranges, count, seed=seed, base_raw=copy.deepcopy(base), out_dir=d, workers=1)
        files = {}
        for f in sorted(os.listdir(d)):
            if f.endswith(".srtf"):
                files[f] = sha(open(os.path.join(d, f), "rb").read())
        out[name] = {"ranges": rg, "count": count, "seed": seed, "base_raw": base,
                     "manifest": open(os.path.join(d, "manifest.jsonl")).read(), "surfaces": files}
    return out


def main():
    with tempfile.TemporaryDirectory() as tmp:
        doc = {"configs": gen_configs(), "exports": gen_exports(tmp), "datasets": gen_datasets(tmp)}
    with open(os.path.join(OUT, "io_golden.json"), "w") as fh:
        json.dump(doc, fh, indent=1, sort_keys=True)
    print("wrote", os.path.join(OUT, "io_golden.json"))


if __name__ == "__main__":
    main()
