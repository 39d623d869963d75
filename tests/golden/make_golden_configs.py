"""Full-size oracle fixtures for BASELINE configs 3, 4 and 5.

The extended CPU oracle (oracle/fsm_ext_oracle.py, pinned bit-exact to the
real reference where the reference has the features) is run HERE, in the
build container, on the workloads exactly as oracle/workloads.py pins them
(which equal paper_2603_28160_b200/configs.py field by field,
tests/test_host_cpu.py). The GPU box only reads the committed .npz files
(tests/test_gpu_configs_full.py). Usage:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_configs.py [3] [4] [5]

Per surface the fixture holds:
  * ``sha256`` of the row-major fp64 height map (the bit-exact gate),
  * ``row_bits``: per node row, the sum mod 2^64 of the heights' IEEE bit
    patterns (pinpoints the rows that differ when the hash does not match),
  * ``rows``: every ``row_stride``-th node row in full,
  * counters (time steps, trajectory points, machined cells, deposits),
  * the oracle's areal metrics (Sa Sq Sp Sv Sz Ssk Sku over machined cells,
    ``uncut='exclude'``) and Ra/Rz of every 64th feed profile
    (roughness.py:93-188 restated by oracle/fsm_oracle.py).
Config 3 keeps, per parameter set, the hash, counters, metrics and one row.
Wall time here (8 threads): config 4 ~2 min, config 5 ~10 min, config 3 ~10 min.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.dont_write_bytecode = True

from oracle import fsm_ext_oracle as xorc  # noqa: E402
from oracle import fsm_oracle as orc  # noqa: E402
from oracle import workloads as W  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "full")
WORKERS = int(os.environ.get("ORACLE_WORKERS", os.cpu_count() or 1))
AREAL_KEYS = ("Sa", "Sq", "Sp", "Sv", "Sz", "Ssk", "Sku", "cell_count")


def row_bits(h2d: np.ndarray) -> np.ndarray:
    return h2d.view(np.uint64).sum(axis=1, dtype=np.uint64)


def metrics(h2d, init, every):
    am = orc.areal_metrics(h2d, init, uncut="exclude")
    out = {"areal": {k: am[k] for k in AREAL_KEYS if k in am}}
    if every:
        prof = []
        for i in range(0, h2d.shape[0], every):
            try:
                r = orc.profile_roughness(h2d[i], init, uncut="exclude")
                prof.append([i, r["Ra"], r["Rz"]])
            except ValueError:
                prof.append([i, None, None])
        out["profiles"] = prof
    return out


def run_single(cfg_id: int, stride: int) -> None:
    cfg, ext, meta = W.FACTORIES[cfg_id]()
    t0 = time.perf_counter()
    h, p, ctr, _ = xorc.ext_sweep(cfg, ext, workers=WORKERS)
    wall = time.perf_counter() - t0
    h2 = h.reshape(p.m + 1, p.n + 1)
    met = metrics(h2, p.initial_height, meta["profiles_every"])
    info = {"counters": ctr, "initial_height": p.initial_height, "oracle_wall_s": wall,
            "workers": WORKERS, "metrics": met}
    np.savez_compressed(os.path.join(OUT, f"{meta['name']}_full.npz"),
                        sha256=np.array(hashlib.sha256(h.tobytes()).hexdigest()),
                        row_bits=row_bits(h2), row_stride=np.array(stride),
                        rows=np.ascontiguousarray(h2[::stride]), info_json=np.array(json.dumps(info)))
    print(meta["name"], f"{wall:.1f} s", ctr, met["areal"], flush=True)


def run_config3() -> None:
    sets, samples, meta = W.config3_sets()
    hashes, rows, infos = [], [], []
    t0 = time.perf_counter()
    for i, (cfg, ext) in enumerate(sets):
        h, p, ctr, _ = xorc.ext_sweep(cfg, ext, workers=WORKERS)
        h2 = h.reshape(p.m + 1, p.n + 1)
        hashes.append(hashlib.sha256(h.tobytes()).hexdigest())
        rows.append(h2[p.m // 2].copy())
        try:
            met = metrics(h2, p.initial_height, None)
        except ValueError as exc:
            met = {"error": str(exc)}
        infos.append({"counters": ctr, "initial_height": p.initial_height, "metrics": met})
        if i % 32 == 0:
            print("config3", i, f"{time.perf_counter() - t0:.1f} s", flush=True)
    np.savez_compressed(os.path.join(OUT, "config3_full.npz"), sha256=np.array(hashes),
                        mid_rows=np.stack(rows), samples=samples,
                        info_json=np.array(json.dumps({"sets": infos, "workers": WORKERS,
                                                       "oracle_wall_s": time.perf_counter() - t0})))
    print("config3", f"{time.perf_counter() - t0:.1f} s", flush=True)


def main(argv) -> None:
    which = [int(a) for a in argv] or [4, 5, 3]
    for c in which:
        if c == 3:
            run_config3()
        elif c == 4:
            run_single(4, 1250)
        elif c == 5:
            run_single(5, 512)
        else:
            raise SystemExit(f"no full-size fixture for config {c}")


if __name__ == "__main__":
    main(sys.argv[1:])
