import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    import json
    d = os.path.join(ROOT, "tests", "golden")
    return {n[:-5]: json.load(open(os.path.join(d, n))) for n in os.listdir(d) if n.endswith(".json")}


# decode / fused-update implementations (slc_plan_set_option: OPT_AGG_KERNEL = 1, OPT_AGG_GRID_CAP = 2);
# a capped grid makes every CTA of a persistent kernel walk many chunks
AGG_KERNEL_VARIANTS = {"batch": {1: 1}, "batch-grid5": {1: 1, 2: 5}, "pipe": {1: 2}, "pipe-grid3": {1: 2, 2: 3},
                       "simple": {1: 3}}


@pytest.fixture(params=sorted(AGG_KERNEL_VARIANTS))
def agg_kernel(request, monkeypatch):
    from paper_2603_08163_b200 import slc
    monkeypatch.setattr(slc.Plan, "default_options", dict(AGG_KERNEL_VARIANTS[request.param]))
    return request.param
