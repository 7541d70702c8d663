import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


class Inst:
    """Duck-typed QAP instance built from the golden arrays (the same fields
    as the reference's QapInstance: name, n, flow, distance, known_best)."""

    def __init__(self, name, n, flow, distance, known_best=None):
        self.name, self.n, self.flow, self.distance = name, n, flow, distance
        self.known_best = known_best

    @property
    def is_integral(self):
        return self.flow.dtype.kind in "iu" and self.distance.dtype.kind in "iu"


def load_instances():
    arr = np.load(GOLDEN / "instances.npz")
    meta = json.loads((GOLDEN / "instances.json").read_text())
    out = {}
    for k, m in meta.items():
        if k.endswith("_sln"):
            continue
        out[k] = Inst(m["name"], m["n"], arr[f"{k}__flow"], arr[f"{k}__distance"],
                      m["known_best"])
    return out, meta


@pytest.fixture(scope="session")
def golden_instances():
    return load_instances()[0]


@pytest.fixture(scope="session")
def golden_meta():
    return load_instances()[1]


@pytest.fixture(scope="session")
def trajectories():
    return json.loads((GOLDEN / "trajectories.json").read_text())


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
