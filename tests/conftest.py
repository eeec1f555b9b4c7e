import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def models():
    from paper_1710_08124_b200 import synthetic

    out = {}
    for P in (64, 100):
        m = synthetic.synthetic_gmm(200, P, 0, 0.95)
        out[P] = (m, synthetic.baseline_tree(m))
    return out


def load_golden(name):
    d = np.load(GOLDEN / f"restore_{name}.npz")
    g = {k: d[k] for k in d.files}
    g["meta"] = json.loads(str(g["meta"]))
    return g


def golden_inputs(name):
    """Operator, observation, sigma, spacing, P of a golden case (rebuilt
    from the product-side synthetic generators, checked against the stored y)."""
    from paper_1710_08124_b200 import operators as ops, synthetic

    g = load_golden(name)
    meta = g["meta"]
    if meta["cfg"] == "gain":
        H = meta["size"]
        A = ops.gain_operator(ops.radial_gain_map((H, H), 0.6))
    else:
        A = synthetic.baseline_case(meta["cfg"], meta["size"]).A
    return g, A, g["y"], meta["sigma"], meta["spacing"], meta["patch_dim"]


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
