import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
REF_SRC = "/root/reference/pkg/src"
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA executor")
    config.addinivalue_line("markers", "reference: needs the read-only reference tree "
                                       "(/root/reference, build container only)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def reference_available():
    return os.path.isdir(os.path.join(REF_SRC, "gpumux"))


@pytest.fixture(scope="session")
def golden_traces():
    return load_golden("traces.json")


@pytest.fixture(scope="session")
def golden_costs():
    return load_golden("costs.json")


@pytest.fixture(scope="session")
def golden_models():
    return load_golden("models.json")


@pytest.fixture(scope="session")
def golden_profiles():
    return load_golden("profiles.json")
