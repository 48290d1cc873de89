"""Locate the reference host framework (``speechserve``) that this executor plugs into.

The reference's model-execution interface (types, errors, chunk rule) and its
streaming-aware scheduler stay unchanged: this package is a drop-in executor
behind them, so it imports them from the reference install made by
``pip install --target baseline/_ref`` ("Reference install").
"""

from __future__ import annotations

import importlib
import os
import sys
from pathlib import Path

_REPO = Path(__file__).resolve().parent.parent


def _candidates() -> list[Path]:
    out = []
    env = os.environ.get("VOXB200_REF")
    if env:
        out.append(Path(env))
    out.append(_REPO / "baseline" / "_ref")
    return out


def load():
    try:
        return importlib.import_module("speechserve")
    except ImportError:
        pass
    for p in _candidates():
        if (p / "speechserve" / "__init__.py").exists():
            sys.path.insert(0, str(p))
            return importlib.import_module("speechserve")
    raise ImportError(
        "reference package 'speechserve' not found; install it with "
        "`python -m pip install --no-index --no-build-isolation --no-deps "
        "--target baseline/_ref /root/reference/pkg` (see DESIGN.md)"
    )


speechserve = load()
from speechserve import core, errors, model_api, profiles, scheduler, workload  # noqa: E402
from speechserve import engine as ref_engine  # noqa: E402

__all__ = ["speechserve", "core", "errors", "model_api", "profiles", "scheduler", "workload", "ref_engine"]
