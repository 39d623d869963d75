"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: feed-strip
partitioning, the two-round all-reduce of partial roughness moments
(sharded.combine) and the metric finish, against the single-field oracle.
The per-strip partial sums are computed here with NumPy exactly as the
device passes define them (include/msurf.h msurf_areal_pass1/2,
msurf_profiles); the kernels themselves are covered by tests/test_gpu_*."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_28160_b200 import sharded
from paper_2603_28160_b200.roughness import _finish_areal, _finish_profile


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _field():
    rng = np.random.default_rng(42)
    h = 0.2 + 0.01 * rng.standard_normal((37, 53))
    h[0, :5] = 0.5  # a few uncut cells (sentinel 0.5)
    h[12, 40] = 0.5
    return h, 0.5


def _stats1(block, sent, exclude):
    cut = block < sent
    z = (block[cut] if exclude else block.ravel()) * 1000.0
    if z.size == 0:
        return np.array([0.0, -np.inf, np.inf, 0.0, float((~cut).sum()), 0.0])
    return np.array([z.sum(), z.max(), z.min(), float(z.size), float((~cut).sum()), 0.0])


def _moments(block, sent, exclude, mean):
    cut = block < sent
    z = (block[cut] if exclude else block.ravel()) * 1000.0
    d = z - mean
    return np.array([np.abs(d).sum(), (d * d).sum(), (d ** 3).sum(), (d ** 4).sum()])


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h, sent = _field()
    j_lo, j_hi = sharded.strip_bounds(h.shape[1], world)[rank]
    strip = h[:, j_lo:j_hi + 1]
    res = {}
    for exclude in (True, False):
        st1 = torch.tensor(_stats1(strip, sent, exclude)).view(1, 6)
        sharded.combine(st1, sharded.STATS1_SUM, sharded.STATS1_MAX, sharded.STATS1_MIN)
        st1[0, 5] = st1[0, 0] / st1[0, 3]
        mean = float(st1[0, 5])
        st2 = torch.tensor(_moments(strip, sent, exclude, mean)).view(1, 4)
        sharded.combine(st2, (0, 1, 2, 3), (), ())
        try:
            m = _finish_areal(st1[0].numpy(), st2[0].numpy(), "exclude" if exclude else "raise")
            res[exclude] = (m.sa_um, m.sq_um, m.sz_um, m.ssk, m.sku, m.cell_count)
        except Exception as exc:  # DomainError expected for raise mode
            res[exclude] = type(exc).__name__
    # profiles: every 8th feed row, spanning both strips
    rows = list(range(0, h.shape[0], 8))
    first = []
    for i in rows:
        z = strip[i][strip[i] < sent] * 1000.0
        first.append([z.sum(), z.size, (strip[i] >= sent).sum(), z.max() if z.size else -np.inf,
                      z.min() if z.size else np.inf, 0, 0, 0])
    first = torch.tensor(np.array(first, dtype=np.float64))
    sharded.combine(first, sharded.PROF_SUM, sharded.PROF_MAX, sharded.PROF_MIN)
    first[:, 6] = first[:, 0] / first[:, 1]
    sabs = []
    for k, i in enumerate(rows):
        mean = float(first[k, 0] / first[k, 1])
        z = strip[i][strip[i] < sent] * 1000.0
        sabs.append([np.abs(z - mean).sum()])
    sabs = torch.tensor(np.array(sabs))
    sharded.combine(sabs, (0,), (), ())
    first[:, 5:6] = sabs
    res["profiles"] = [(p.ra_um, p.rz_um) for p in
                       (_finish_profile(r, i, "exclude") for r, i in zip(first.numpy(), rows))]
    out[rank] = res
    dist.destroy_process_group()


def test_strip_bounds_partition():
    for nodes in (1000, 1001, 4096, 7):
        for world in (1, 2, 3, 4, 8):
            if nodes < world:
                continue
            b = sharded.strip_bounds(nodes, world)
            assert b[0][0] == 0 and b[-1][1] == nodes - 1
            assert all(b[k][1] + 1 == b[k + 1][0] for k in range(world - 1))
            assert max(hi - lo for lo, hi in b) - min(hi - lo for lo, hi in b) <= 1
    assert sharded.batch_slice(256, 3, 8) == slice(96, 128)


def test_strip_roi():
    from paper_2603_28160_b200 import GridSpec

    g = GridSpec(0.01, 0.0, 0.0, 9, 99)
    assert sharded.strip_roi(g, None, 50, 99) == (0, 0, 10, 50)
    assert sharded.strip_roi(g, (2, 10, 5, 60), 50, 99) == (2, 0, 4, 11)
    assert sharded.strip_roi(g, (2, 10, 5, 40), 50, 99) is None


def test_two_rank_gloo_moment_allreduce_matches_single_field():
    from oracle import fsm_oracle as orc

    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    h, sent = _field()
    exp = orc.areal_metrics(h, sent, uncut="exclude")
    for rank in range(world):
        got = out[rank][True]
        ref = (exp["Sa"], exp["Sq"], exp["Sz"], exp["Ssk"], exp["Sku"], exp["cell_count"])
        for a, b in zip(got, ref):
            assert a == pytest.approx(b, rel=1e-12)
        assert out[rank][False] == "DomainError"  # uncut cells present, reference semantics
        for (ra, rz), i in zip(out[rank]["profiles"], range(0, h.shape[0], 8)):
            pr = orc.profile_roughness(h[i], sent, uncut="exclude")
            assert ra == pytest.approx(pr["Ra"], rel=1e-12)
            assert rz == pytest.approx(pr["Rz"], rel=1e-12)
