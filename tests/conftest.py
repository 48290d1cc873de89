import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
REF = ROOT / "baseline" / "_ref"
if REF.exists():
    sys.path.insert(0, str(REF))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built libvoxb200.so")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no GPU in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def tiny_cfg():
    from paper_2602_00269_b200.config import tiny

    return tiny()


@pytest.fixture(scope="session")
def tiny_dev(tiny_cfg):
    from paper_2602_00269_b200.build import build
    from paper_2602_00269_b200.device import VoxDevice

    build()
    dev = VoxDevice(tiny_cfg, weight_seed=1234)
    yield dev
    dev.close()


@pytest.fixture(scope="session")
def tiny_oracle(tiny_cfg):
    from oracle.llama import LlamaOracle

    return LlamaOracle(tiny_cfg, 1234)
