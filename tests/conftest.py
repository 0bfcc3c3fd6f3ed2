import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def golden_view(rec, prefix="view"):
    return SimpleNamespace(position=rec[f"{prefix}_position"], forward=rec[f"{prefix}_forward"],
                           up=rec[f"{prefix}_up"], right=rec[f"{prefix}_right"],
                           tan_half=float(rec[f"{prefix}_tan_half"]),
                           resolution=tuple(int(v) for v in rec[f"{prefix}_resolution"]))


def golden_camera(rec, prefix="cam"):
    from paper_2301_05262_b200.scenes import CameraPose
    return CameraPose(rec[f"{prefix}_position"], rec[f"{prefix}_forward"], rec[f"{prefix}_up"],
                      float(rec[f"{prefix}_fov_y"]),
                      tuple(int(v) for v in rec[f"{prefix}_resolution"]))


def golden_nets():
    z = load_golden("nets")
    cases = {}
    for k, v in z.items():
        name, _, rest = k.partition("/")
        c = cases.setdefault(name, {"w": {}})
        if rest.startswith("w/"):
            c["w"][rest[2:]] = v
        else:
            c[rest] = v
    return cases


@pytest.fixture(scope="session")
def cfg1():
    return load_golden("cfg1")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
