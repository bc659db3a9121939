import os
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


def load_container(path):
    import json
    z = np.load(path)
    meta = json.loads(bytes(z["meta"]).decode())
    return dict(meta=meta, x=z["x"], blob=z["blob"].tobytes(), y=z["y"], offsets=z["offsets"])


def golden_containers():
    import json
    manifest = json.loads((GOLDEN / "manifest.json").read_text())
    return [m["name"] for m in manifest]


def reference_available() -> bool:
    ref = os.environ.get("APAX_REF", "/root/reference/pkg/src")
    return pathlib.Path(ref, "apax", "codec.py").exists()
