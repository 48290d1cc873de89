"""CPU: `bench.py --gpus 2` outside torchrun launches two ranks itself (gloo probe)."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_gpus_flag_spawns_ranks():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--ranks-probe"],
                         capture_output=True, text=True, timeout=240)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 for d in lines)
