import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def rng_for(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


class Golden:
    """Lazy accessor over a golden .npz written by tests/golden/make_golden.py."""

    def __init__(self, name):
        self.z = np.load(os.path.join(GOLDEN, name), allow_pickle=False)

    def __getitem__(self, key):
        return self.z[key]

    def names(self, key="names"):
        return [str(s) for s in self.z[key]]

    def obs_args(self, prefix):
        z = self.z
        return (int(z[prefix + "m"]), int(z[prefix + "n"]), z[prefix + "rows"], z[prefix + "cols"],
                z[prefix + "vals"])


@pytest.fixture(scope="session")
def golden():
    return Golden


@pytest.fixture(scope="session")
def traces():
    with open(os.path.join(GOLDEN, "traces.json")) as fh:
        return json.load(fh)


def random_obs_arrays(rng, m, n, frac=0.4, scale=1.0):
    mask = rng.random((m, n)) < frac
    mask[0, 0] = True
    rows, cols = np.nonzero(mask)
    vals = scale * rng.standard_normal(rows.size)
    return m, n, rows, cols, vals
