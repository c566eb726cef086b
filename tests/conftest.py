import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")
REF_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        return json.load(fh)


def make_instance(r):
    """Product KernelInstance from a golden record."""
    import paper_1412_6986_b200 as L

    params = L.TemplateParams(
        r["in_h"], r["in_w"], r["out_h"], r["out_w"], L.HomeAccessPattern(r["pattern"]), r["n"], r["m"],
        L.StencilPattern(L.StencilShape(r["shape"]), r["radius"]), r["num_comp_ilb"], r["num_comp_ep"],
        r["num_coal_ilb"], r["num_coal_ep"], r["num_uncoal_ilb"], r["num_uncoal_ep"])
    return L.KernelInstance(params, L.LaunchConfig(r["grid_x"], r["grid_y"], r["wg_x"], r["wg_y"]))


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "lmtune"))


@pytest.fixture(scope="session")
def lmtune_ref():
    if not reference_available():
        pytest.skip("reference package not present (only in the build container)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import lmtune

    return lmtune
