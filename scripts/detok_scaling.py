"""K4 detok call time vs windows per call (steady-state 7-token windows). GPU only."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2602_00269_b200.config import orpheus3b  # noqa: E402
from paper_2602_00269_b200.device import VoxDevice  # noqa: E402

dev = VoxDevice(orpheus3b(max_slots=260, max_detok_frames=1024), 0)
for n in [8, 16, 32, 64, 128, 192]:
    r = bench.detok_roofline(dev, 1412.4, 6423.4, n_win=n, calls=10)
    print(f"windows {n:4d}: {r['ms_per_call']:.3f} ms/call  {r['ms_per_call'] / n * 1e3:.1f} us/window  "
          f"{r['audio_s_per_s']:.0f} audio-s/s", flush=True)
