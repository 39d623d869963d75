"""CPU-only tests: C-ABI library loads and exports every declared symbol,
the host planner reproduces the reference plan bit-exactly (vs the oracle,
itself pinned to the reference goldens), the extended planner equals the
extended oracle, key encoding is order-preserving, samplers are bit-exact,
and configuration errors raise the reference's exception types."""

import ctypes
import math
import os
import re
from types import SimpleNamespace as NS

import numpy as np
import pytest

import golden_io
import paper_2603_28160_b200 as ms
from paper_2603_28160_b200 import _native, planner
from oracle import fsm_ext_oracle as xorc
from oracle import fsm_oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = golden_io.case_names()


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    header = open(os.path.join(ROOT, "include", "msurf.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char\*|void\*)\s+(msurf_\w+)\s*\(", header, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_native.EXPORTS), declared ^ set(_native.EXPORTS)
    for name in declared:
        assert getattr(lib, name) is not None
    assert lib.msurf_abi_version() == _native.ABI_VERSION
    assert lib.msurf_sizeof_job() == ctypes.sizeof(_native.MsurfJob)
    assert lib.msurf_tile_steps() > 0 and lib.msurf_tile_steps() % 32 == 0


def test_error_path_without_gpu_reports_message():
    lib = _native.load_library()
    assert lib.msurf_sweep(None, 0, None, 0, 0, 1, None, None) != 0
    assert b"bad arguments" in lib.msurf_last_error()


@pytest.mark.parametrize("name", CASES)
def test_ref_plan_matches_oracle_plan(name):
    g = golden_io.load(name)
    cfg = golden_io.product_config(g["config"])
    p = planner.plan(cfg)
    o = orc.plan(golden_io.namespace_config(g["config"]))
    assert p.mode == planner.MODE_REF
    assert (p.steps, p.points, p.teeth) == (o.steps, o.points, o.teeth)
    assert p.dt == o.dt and p.t_start == o.t_start and p.y0 == o.y0
    assert p.initial_height == o.initial_height == g["counters"]["initial_height"]
    assert p.trajectory_points == g["counters"]["trajectory_points"]
    assert np.array_equal(p.px, o.xp) and np.array_equal(p.pz, o.zp)
    for k in range(p.teeth):
        assert np.array_equal(p.zw[k], o.zw[k])
        assert p.min_index[k] == o.min_index[k]
        e = o.rows[k]
        assert list(p.tooth_rows[k]) == [e[0][0], e[0][1], e[0][2], e[0][3], e[1][0], e[1][1], e[1][2], e[1][3]]
        assert p.tooth_base[k] == orc.tooth_base(cfg.process.phase_rad, k + 1, p.teeth)
    assert np.array_equal(planner.decode_keys(p.zkey), p.zw + 0.0)
    # chunk boxes enclose the tool-frame points
    nchunk = (p.points + 31) // 32
    assert p.chunk_box.shape == (p.teeth, nchunk, 6)


EXT_CASES = {
    "helix_insert": dict(helix_angle_rad=math.radians(30)),
    "ball_tilt": dict(profile="ball", tilt_rad=math.radians(15), helix_angle_rad=math.radians(30),
                      runout_offset_mm=0.005, runout_phase_rad=math.radians(40), passes=3, stepover_mm=0.3),
    "vib_runout": dict(runout_offset_mm=0.003, vib_amplitude_mm=0.002, vib_frequency_hz=300.0),
    "ball_noise": dict(profile="ball", tilt_rad=math.radians(10), runout_offset_mm=0.004,
                       noise_sigma_mm=0.001, noise_corr_mm=0.02, noise_seed=7),
}


def _ext_cfg(profile="insert"):
    if profile == "ball":
        tool = ms.ToolDefinition(cutting_diameter_mm=6.0, insert_radius_mm=3.0, tooth_count=2)
        proc = ms.derive_kinematics(tooth_count=2, cutting_diameter_mm=6.0, depth_of_cut_mm=0.2,
                                    spindle_speed_rpm=6000.0, feed_per_tooth_mm=0.08,
                                    initial_position_mm=(-0.3, None, 0.0))
        grid = ms.GridSpec.from_nodes(0.01, -0.5, 0.0, 101, 81)
        return ms.SimulationConfig(tool=tool, process=proc, grid=grid, edge_point_count=77,
                                   time_step_s=(2 * math.pi / 720) / proc.angular_velocity_rad_s)
    tool = ms.ToolDefinition(cutting_diameter_mm=10.0, insert_radius_mm=5.0, tooth_count=4)
    proc = ms.derive_kinematics(tooth_count=4, cutting_diameter_mm=10.0, depth_of_cut_mm=1.0,
                                spindle_speed_rpm=3000.0, feed_per_tooth_mm=0.05,
                                initial_position_mm=(0.0, -2.0, 0.0))
    grid = ms.GridSpec.from_nodes(0.02, -0.99, 0.0, 100, 100)
    om = proc.angular_velocity_rad_s
    return ms.SimulationConfig(tool=tool, process=proc, grid=grid, edge_point_count=61,
                               time_step_s=(2 * math.pi / 720) / om, span_s=(0.0, 4 * 2 * math.pi / om))


@pytest.mark.parametrize("case", sorted(EXT_CASES))
def test_ext_plan_matches_ext_oracle(case):
    kw = EXT_CASES[case]
    cfg = _ext_cfg(kw.get("profile", "insert"))
    ext = ms.Extensions(**kw)
    p = planner.plan(cfg, ext)
    o = xorc.ext_plan(cfg, NS(**kw))
    assert p.mode == (planner.MODE_EXT_TILT if kw.get("tilt_rad") else planner.MODE_EXT)
    assert (p.steps, p.points, p.teeth) == (o.steps, o.points, o.teeth)
    assert p.y0 == o.y0 and p.dt == o.dt
    assert np.array_equal(p.px, o.xt) and np.array_equal(p.py, o.yt) and np.array_equal(p.pz, o.zt)
    assert np.array_equal(p.zw, o.zw) and p.zoff == o.zoff
    assert list(p.pass_x0) == list(o.pass_x0)
    assert (p.tilt_c, p.tilt_s, p.vib_amp, p.vib_omega, p.vib_phase) == \
        (o.tilt_c, o.tilt_s, o.vib_amp, o.vib_omega, o.vib_phase)
    assert list(p.tooth_base) == list(o.base)


def test_ext_zero_formulation_is_reference_on_goldens():
    # the extended formulation with every extension at zero reproduces the
    # reference bit-exactly on the reference's own golden cases
    for name in CASES:
        g = golden_io.load(name)
        cfg = golden_io.namespace_config(g["config"])
        h, _, _, _ = xorc.ext_sweep(cfg, NS(force_extended=True), workers=4)
        assert golden_io.heights_match(g, h), name


def test_key_encoding_is_order_preserving():
    rng = np.random.default_rng(3)
    z = np.concatenate([rng.normal(0, 1, 5000), rng.normal(0, 1e-300, 100), [0.0, -0.0, 1e308, -1e308,
                                                                             5e-324, -5e-324]])
    k = planner.encode_keys(z)
    order_z = np.argsort(z, kind="stable")
    assert np.all(np.diff(k[order_z].astype(np.float64)) >= 0) or np.all(k[order_z][1:] >= k[order_z][:-1])
    assert np.array_equal(planner.decode_keys(k), z + 0.0)
    assert planner.encode_keys(np.array([-0.0]))[0] == planner.encode_keys(np.array([0.0]))[0]


def test_lhs_bit_exact_with_reference_goldens():
    z = np.load(os.path.join(golden_io.GOLDEN, "lhs.npz"))
    names = ["cutting_speed_m_min", "feed_per_tooth_mm", "depth_of_cut_mm", "grid_spacing_mm",
             "radial_rake_deg", "phase_deg"]
    ranges = [ms.ParameterRange(n, *b) for n, b in zip(names, z["bounds"])]
    for key in z.files:
        if key.startswith("lhs_"):
            _, count, seed = key.split("_")
            assert np.array_equal(ms.lhs_sample(ranges, int(count), int(seed)), z[key])


def test_uniform_sampler_shape_and_bounds():
    ranges = [ms.ParameterRange("feed_per_tooth_mm", 0.02, 0.2), ms.ParameterRange("spindle_speed_rpm", 2000, 12000)]
    s = ms.uniform_sample(ranges, 256, 0)
    assert s.shape == (256, 2)
    assert s[:, 0].min() >= 0.02 and s[:, 0].max() <= 0.2
    assert np.array_equal(s, ms.uniform_sample(ranges, 256, 0))


def test_reference_error_types():
    with pytest.raises(ms.ConfigError):
        ms.ParameterRange("helix", 0, 1)
    with pytest.raises(ms.DomainError):
        ms.ToolDefinition(cutting_diameter_mm=-1, insert_radius_mm=1, tooth_count=1)
    with pytest.raises(ms.ConfigError):
        ms.derive_kinematics(tooth_count=2, cutting_diameter_mm=10, depth_of_cut_mm=1)
    g = golden_io.load("tiny")
    cfg = golden_io.product_config(g["config"], time_step_s=-1.0)
    with pytest.raises(ms.ConfigError):
        planner.plan(cfg)
    cfg = golden_io.product_config(g["config"], span_s=(0.0, 0.01))
    with pytest.raises(ms.ConfigError):  # explicit span needs y0 (engine.py:166-167)
        planner.plan(cfg)
    cfg = golden_io.product_config(g["config"], worker_count=0)
    with pytest.raises(ms.ConfigError):
        planner.plan(cfg)
    assert issubclass(ms.DomainError, ValueError) and issubclass(ms.ConfigError, ms.MillsurfError)


def test_time_step_kats():
    # test_engine.py:31-42
    g = golden_io.load("tiny")
    cfg = golden_io.product_config(g["config"], time_step_s=None)
    dt = ms.time_step(cfg)
    assert dt == pytest.approx(1.5400e-5, rel=1e-4)
    assert dt == math.radians(0.5) / cfg.process.angular_velocity_rad_s


def test_locate_kats():
    spec = ms.GridSpec(0.01, 0.0, 0.0, 10, 10)
    assert ms.locate(0.012, 0.0, spec) == (1, 0)
    assert ms.locate(-0.006, 0.0, spec) is None
    assert ms.locate(0.005, 0.0, spec) == (1, 0)


def test_host_heightfield_semantics():
    spec = ms.GridSpec(0.1, 0.0, 0.0, 3, 2)
    f = ms.HeightField(spec, 0.5)
    assert ms.update_min(f, (1, 1), 0.1) and not ms.update_min(f, (1, 1), 0.1)
    assert f.machined_cell_count() == 1
    g = ms.HeightField(spec, 0.5)
    ms.update_min(g, (0, 0), 0.2)
    f.merge_min(g)
    assert f.machined_cell_count() == 2
    with pytest.raises(ms.DomainError):
        ms.update_min(f, (4, 0), 0.0)


def test_device_required_no_cpu_fallback(monkeypatch):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = golden_io.load("tiny")
    with pytest.raises(ms.NativeUnavailableError):
        ms.simulate(golden_io.product_config(g["config"]))


def test_job_dtype_matches_ctypes_layout():
    """SweepBatch writes msurf_job rows through a NumPy structured dtype; every
    field must land where the ctypes mirror (and the C header) puts it."""
    names = [f for f, _ in _native.MsurfJob._fields_]
    assert list(_native.JOB_DTYPE.names) == names
    assert _native.JOB_DTYPE.itemsize == ctypes.sizeof(_native.MsurfJob)
    vals = tuple((k + 1) * (0.5 if _native.JOB_DTYPE[f].kind == "f" else 3) for k, f in enumerate(names))
    vals = tuple(int(v) if _native.JOB_DTYPE[f].kind != "f" else v for v, f in zip(vals, names))
    row = np.array([vals], dtype=_native.JOB_DTYPE)
    j = _native.MsurfJob.from_buffer_copy(row.tobytes())
    for f, v in zip(names, vals):
        assert (getattr(j, f) or 0) == v, f


def test_plan_many_bitwise_equals_per_set_plan():
    """The vectorised batch planner (simulate_batch) reproduces plan() per set."""
    from paper_2603_28160_b200 import configs
    from paper_2603_28160_b200.dataset import ParameterRange, apply_sample, uniform_sample

    base, ext, meta = configs.config3_base()
    ranges = [ParameterRange(n, lo, hi) for n, lo, hi in meta["ranges"]]
    samples = uniform_sample(ranges, 24, 3)
    names = [r.name for r in ranges]
    pairs = [apply_sample(base, ext, names, samples[i], 3600) for i in range(24)]
    # plus a tilt/noise group and a reference-kinematics set
    cfg_b = _ext_cfg("ball")
    for k in range(5):
        pairs.append((cfg_b, ms.Extensions(profile="ball", tilt_rad=0.2, helix_angle_rad=0.3 + 0.05 * k,
                                           runout_offset_mm=0.001 * k, noise_sigma_mm=0.001, noise_corr_mm=0.02)))
    pairs.append((golden_io.product_config(golden_io.load("small_3")["config"]), None))
    many = planner.plan_many([c for c, _ in pairs], [e for _, e in pairs])
    for (c, e), a in zip(pairs, many):
        b = planner.plan(c, e)
        for f in ("px", "py", "pz", "zw", "zkey", "chunk_box", "chunk_circ", "pts", "tooth_box", "pass_x0",
                  "tooth_base", "min_index"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f
        for f in ("steps", "dt", "t_start", "y0", "x0", "zoff", "initial_height", "mode", "tilt_c", "tilt_s",
                  "vib_amp", "vib_omega", "vib_phase", "feed_speed", "omega", "points", "teeth"):
            assert getattr(a, f) == getattr(b, f), f
        if a.group is not None:  # group arrays SweepBatch packs as one slice per field
            g, k = a.group
            assert g.owns(a, k)
            assert np.array_equal(g.arrays["chunk_f32"][k], planner.chunk_f32(b.chunk_circ, b.tooth_box, planner.plan_zfloor(b)))
            assert np.array_equal(g.arrays["tooth_rows"][k], b.tooth_rows)
    assert sum(p.group is not None for p in many) >= 24
    # native planning loops on several threads: the same arrays
    many_mt = planner.plan_many([c for c, _ in pairs], [e for _, e in pairs], threads=2, native_threads=3)
    for a, b in zip(many, many_mt):
        for f in ("pts", "chunk_circ", "tooth_box", "zkey", "min_index"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f


def test_sweep_batch_descriptors_point_at_plan_arrays(monkeypatch):
    """SweepBatch packing (group slices for plan_many sets, per-set arrays
    otherwise): every msurf_job pointer must address the bytes of its own
    plan's array in the uploaded arena. Runs on CPU with the upload faked
    into a host tensor."""
    import torch

    from paper_2603_28160_b200 import configs, engine
    from paper_2603_28160_b200.dataset import ParameterRange, apply_sample, uniform_sample

    monkeypatch.setattr(_native, "require_cuda", lambda: torch)

    def upload(self, device, fill_structs=None):
        dev = torch.zeros(max(self.size, 1), dtype=torch.uint8)
        extra = fill_structs(dev.data_ptr()) if fill_structs else []
        host = dev.numpy()
        for off, a in self._parts:
            if a is not None:
                host[off:off + a.nbytes] = a.view(np.uint8).reshape(-1)
        for off, b in extra:
            b = b if isinstance(b, np.ndarray) else np.frombuffer(b, dtype=np.uint8)
            host[off:off + b.nbytes] = b
        return dev

    monkeypatch.setattr(_native.Arena, "upload", upload)
    base, ext, meta = configs.config3_base()
    ranges = [ParameterRange(n, lo, hi) for n, lo, hi in meta["ranges"]]
    samples = uniform_sample(ranges, 9, 5)
    names = [r.name for r in ranges]
    pairs = [apply_sample(base, ext, names, samples[i], 3600) for i in range(9)]
    many = planner.plan_many([c for c, _ in pairs], [e for _, e in pairs])
    assert all(p.group is not None for p in many)
    single = planner.plan(*pairs[0])
    order = many[:4] + [single] + many[6:] + [many[5]]  # runs broken by a per-set plan and a gap
    b = engine.SweepBatch([(p, 0, p.grid.n) for p in order], device="cpu")
    mem = b.buf.numpy()
    base_ptr = b.base
    jobs = np.concatenate(b.group_host_jobs)
    seen = set()
    for row, (i, lo, hi, s_lo, s_hi) in zip(jobs, [b.jobs[j] for gm in b.group_meta for j in gm[1]]):
        p = order[i]
        seen.add(i)
        want = {"tooth_base": p.tooth_base, "tooth_rows": p.tooth_rows, "pts": p.pts, "tooth_box": p.tooth_box,
                "chunk_circ": p.chunk_circ, "chunk_f32": planner.chunk_f32(p.chunk_circ, p.tooth_box, planner.plan_zfloor(p)),
                "pass_x0": p.pass_x0, "min_index": p.min_index.astype(np.int32)}
        for f, a in want.items():
            off = int(row[f]) - base_ptr
            a = np.ascontiguousarray(a)
            assert np.array_equal(mem[off: off + a.nbytes], a.view(np.uint8).reshape(-1)), (i, f)
        assert row["steps"] == p.steps and row["points"] == p.points and row["dt"] == p.dt
        assert (row["step_lo"], row["step_hi"], row["j_lo"], row["j_hi"]) == (s_lo, s_hi, lo, hi)
        assert int(row["counters"]) - base_ptr == b.ctr_off + i * _native.NUM_CTRS * 8
    assert seen == set(range(len(order)))


def test_vectorised_profile_finish_equals_per_row():
    """roughness._finish_profiles (all rows at once) gives the same objects
    and the same first error as _finish_profile row by row."""
    from paper_2603_28160_b200 import roughness as R
    from paper_2603_28160_b200.errors import DomainError

    rng = np.random.default_rng(5)
    rows = np.zeros((9, 8))
    rows[:, 1] = rng.integers(2, 1000, 9)
    rows[:, 3] = rng.normal(size=9) + 2.0
    rows[:, 4] = rng.normal(size=9) - 2.0
    rows[:, 5] = rng.random(9) * rows[:, 1]
    rows[:, 6] = rng.normal(size=9) * 0.1
    idx = list(range(0, 90, 10))
    for uncut in ("raise", "exclude"):
        assert R._finish_profiles(rows, idx, uncut) == [R._finish_profile(r, i, uncut) for r, i in zip(rows, idx)]
    bad = rows.copy()
    bad[4, 2] = 3.0   # uncut cells in profile 4
    bad[6, 1] = 1.0   # too few samples in profile 6
    for uncut, row in (("raise", 4), ("exclude", 6)):
        with pytest.raises(DomainError) as e1:
            R._finish_profiles(bad, idx, uncut)
        with pytest.raises(DomainError) as e2:
            R._finish_profile(bad[row], idx[row], uncut)
        assert str(e1.value) == str(e2.value)


def _same_ext_plan(a, b):
    import dataclasses

    pa, pb = xorc.ext_plan(*a), xorc.ext_plan(*b)
    for f in dataclasses.fields(pa):
        va, vb = getattr(pa, f.name), getattr(pb, f.name)
        if isinstance(va, np.ndarray):
            assert np.array_equal(va, vb), f.name
        else:
            assert va == vb, (f.name, va, vb)
    for part in ("tool", "process", "grid"):
        for f in dataclasses.fields(getattr(a[0], part)):
            assert getattr(getattr(a[0], part), f.name) == getattr(getattr(b[0], part), f.name), (part, f.name)
    for k in ("edge_point_count", "time_step_s", "span_s"):
        assert getattr(a[0], k) == getattr(b[0], k), k


def test_oracle_workloads_equal_product_configs():
    """bench.py's reference arm builds its workloads from oracle/workloads.py
    (no product import): they must equal paper_2603_28160_b200/configs.py,
    including the derived kinematics and the oracle plan, for all five
    BASELINE configs (all 256 config-3 sets)."""
    from oracle import workloads as W
    from paper_2603_28160_b200 import configs as C
    from paper_2603_28160_b200.dataset import ParameterRange, apply_sample, uniform_sample

    for k in (1, 2, 4, 5):
        a, b = W.FACTORIES[k](), C.FACTORIES[k]()
        _same_ext_plan(a[:2], b[:2])
        assert a[2] == {kk: v for kk, v in b[2].items() if kk in a[2]}
    sets, samples, meta = W.config3_sets()
    base, ext, m2 = C.config3_base()
    ranges = [ParameterRange(n, lo, hi) for n, lo, hi in m2["ranges"]]
    assert np.array_equal(uniform_sample(ranges, m2["count"], m2["seed"]), samples)
    names = [r.name for r in ranges]
    for i in range(meta["count"]):
        _same_ext_plan(sets[i], apply_sample(base, ext, names, samples[i], m2["steps_per_rev"]))


def test_bench_reference_arm_imports_no_product_code(tmp_path):
    """`bench.py --impl reference` (the driver's reference arm) runs only the
    oracle: after a full run the product package was never imported and
    libmsurf.so never mapped."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, json; sys.argv=['bench.py','--impl','reference','--config','1','--steps','1',"
            "'--warmup','0','--cpu-seconds','0.5']; sys.path.insert(0, %r); import bench; bench.main(); "
            "mods=[m for m in sys.modules if m.startswith('paper_2603_28160_b200')]; "
            "maps=open('/proc/self/maps').read(); "
            "print('CHECK', json.dumps({'mods': mods, 'lib': 'libmsurf' in maps}))" % root)
    out = subprocess.run([sys.executable, "-c", code], cwd=tmp_path, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = next(l for l in out.stdout.splitlines() if l.startswith("{"))
    import json

    rec = json.loads(line)
    assert rec["impl"] == "reference" and rec["value"] > 0 and rec["e2e"]["h2d_bytes_per_step"] == 0
    chk = json.loads(out.stdout.split("CHECK ", 1)[1])
    assert chk == {"mods": [], "lib": False}, chk


def test_ext_oracle_edge_noise_statistics():
    """Edge noise: Gaussian-smoothed white noise rescaled to
    sigma; its autocorrelation falls to ~1/e at the correlation length."""
    sigma, corr, ds = 1e-3, 0.02, 0.0005
    d = xorc.edge_noise(3, 20000, sigma, corr, ds, seed=7)
    assert abs(float(d.std()) / sigma - 1.0) < 0.1
    lag = int(round(corr / ds))
    x = d[0] - d[0].mean()
    r = float(np.dot(x[:-lag], x[lag:]) / np.dot(x, x))
    assert abs(r - math.exp(-1.0)) < 0.1, r


def test_ext_oracle_tilt_relevels_lowest_reachable_point():
    """Lead tilt: the tool is re-levelled so the lowest point any edge point
    can reach over a revolution sits exactly at z0."""
    from oracle import workloads as W

    for cid in (2, 5):
        cfg, ext, _ = W.FACTORIES[cid]()
        p = xorc.ext_plan(cfg, ext)
        low = np.min(p.tilt_c * p.zt - abs(p.tilt_s) * np.sqrt(p.xt ** 2 + p.yt ** 2)) + p.zoff
        assert abs(low - p.z0) < 1e-12, (cid, low)


def test_ext_oracle_ball_raster_scallop_height():
    """Ball-end raster without tilt: between two passes at stepover s the
    residual ridge is the scallop R - sqrt(R^2 - (s/2)^2) (feed marks made
    negligible by a tiny feed per tooth)."""
    from dataclasses import replace

    from oracle import workloads as W

    r, s = 1.0, 0.2
    tool = W.Tool(2.0 * r, r, 2)
    proc = W.process(2, 2.0 * r, 0.05, 6000.0, 0.002, initial=(0.0, None, 0.0))
    grid = W.Grid(0.002, 0.0, 0.0, int(round(s / 0.002)), 20)
    cfg = W.Config(tool, proc, grid, edge_point_count=400, time_step_s=(2 * math.pi / 720) / proc.angular_velocity_rad_s)
    ext = W.Ext(profile="ball", passes=2, stepover_mm=s)
    h, p, _, _ = xorc.ext_sweep(cfg, ext, workers=4)
    h2 = h.reshape(p.m + 1, p.n + 1)
    expect = r - math.sqrt(r * r - (s / 2) ** 2)
    ridge = float(h2[p.m // 2].mean())  # midway between the pass centres
    assert abs(ridge - expect) < 0.1 * expect, (ridge, expect)
    assert float(h2[0].mean()) < 0.1 * expect  # pass centre: cut to the ball bottom


@pytest.mark.parametrize("cid", [2, 5])
def test_chunk_zfloor_bounds_every_point_at_every_angle(cid):
    """The stock-height / surface-cap culls rest on chunk_zfloor: for every
    point of a chunk and ANY spindle angle, z' >= sin(tau) * v_centre + zfloor
    + stock (v_centre = the chunk circle centre rotated like the kernel's fp32
    test). Checked on the tilt plans of configs 2 and 5 at 720 angles."""
    from paper_2603_28160_b200 import configs

    cfg, ext, _ = configs.FACTORIES[cid]()
    p = planner.plan(cfg, ext)
    zf = planner.plan_zfloor(p)
    circ = p.chunk_circ
    n = p.points
    nch = circ.shape[1]
    th = np.linspace(0.0, 2.0 * math.pi, 720, endpoint=False)
    c, s = np.cos(th)[:, None], np.sin(th)[:, None]
    for k in range(p.teeth):
        x, y, w = p.pts[k, :, 0], p.pts[k, :, 1], p.pts[k, :, 3]
        v = c * y[None] - s * x[None]                      # (angles, points)
        z = p.tilt_s * v + w[None]
        vc = c * circ[k, :, 1][None] - s * circ[k, :, 0][None]  # (angles, chunks)
        bound = p.tilt_s * vc + zf[k][None] + p.initial_height
        q = np.arange(n) // 32
        assert np.all(z >= bound[:, q] - 1e-12), float(np.min(z - bound[:, q]))
    assert zf.shape == (p.teeth, nch)


@pytest.mark.parametrize("case", ["ball_tilt", "ball_noise"])
def test_final_rows_bound_later_passes_deposits(case):
    """engine.final_rows (the progressive row release of launch_by_strip):
    the oracle's own deposits of every raster pass q >= p_next stay at node
    rows >= final_rows(plan, p_next), on a grid wide enough in x that rows
    are released before the last pass."""
    from dataclasses import replace as dc_replace

    from paper_2603_28160_b200 import engine

    kw = dict(EXT_CASES[case], passes=6, stepover_mm=0.5)
    cfg = _ext_cfg(kw.get("profile", "insert"))
    g = cfg.grid
    cfg = dc_replace(cfg, grid=ms.GridSpec.from_nodes(g.spacing_mm, -1.2, g.y_min_mm, 481, 41), edge_point_count=40)
    x_start = cfg.process.initial_position_mm[0]
    p = planner.plan(cfg, ms.Extensions(**kw))
    rows = p.grid.m + 1
    first_hit = []
    for q in range(kw["passes"]):
        proc = dc_replace(cfg.process, initial_position_mm=(x_start + q * kw["stepover_mm"],) +
                          tuple(cfg.process.initial_position_mm[1:]))
        h, pq, _, _ = xorc.ext_sweep(dc_replace(cfg, process=proc), NS(**dict(kw, passes=1)), workers=2)
        cut = np.nonzero((h.reshape(rows, -1) < pq.initial_height).any(axis=1))[0]
        first_hit.append(int(cut[0]) if cut.size else rows)
    released = 0
    for p_next in range(1, kw["passes"]):
        r = engine.final_rows(p, p_next)
        assert r <= min(first_hit[p_next:]), (p_next, r, first_hit)
        released = max(released, r)
    assert released > 0  # the test geometry does release rows early
