"""CPU: the C-ABI library loads and exports every symbol include/voxb200.h declares.

No compute calls are made (there is no GPU here); creating a context without
an sm_100 device must fail loudly — there is no CPU fallback.
"""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    text = (ROOT / "include" / "voxb200.h").read_text()
    return sorted(set(re.findall(r"\b(vox_[a-z_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2602_00269_b200.build import build

    build()
    from paper_2602_00269_b200 import _lib

    return _lib.load()


def test_all_declared_symbols_exported(lib):
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    from paper_2602_00269_b200 import _lib

    assert set(names) == set(_lib.EXPORTED), set(names) ^ set(_lib.EXPORTED)


def test_abi_version(lib):
    assert lib.vox_abi_version() == 1


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors vs the C compiler's layout of include/voxb200.h (gcc probe)."""
    import shutil
    import subprocess

    from paper_2602_00269_b200 import _lib

    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc missing")
    src = tmp_path / "p.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "voxb200.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(VoxModelCfg), sizeof(VoxSampling),"
        " sizeof(VoxRow), sizeof(VoxWindow), offsetof(VoxModelCfg, rates), offsetof(VoxModelCfg, max_detok_frames),"
        " offsetof(VoxSampling, top_k));"
        "printf(\"%zu %zu %zu %zu\\n\", sizeof(VoxMimiCfg), offsetof(VoxMimiCfg, ratios), offsetof(VoxMimiCfg, max_frames),"
        " sizeof(VoxMimiReq));return 0;}\n")
    exe = tmp_path / "p"
    subprocess.run([gcc, "-I", str(ROOT / "include"), "-o", str(exe), str(src)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    exp = [ctypes.sizeof(_lib.VoxModelCfg), ctypes.sizeof(_lib.VoxSampling), ctypes.sizeof(_lib.VoxRow),
           ctypes.sizeof(_lib.VoxWindow), _lib.VoxModelCfg.rates.offset, _lib.VoxModelCfg.max_detok_frames.offset,
           _lib.VoxSampling.top_k.offset, ctypes.sizeof(_lib.VoxMimiCfg), _lib.VoxMimiCfg.ratios.offset,
           _lib.VoxMimiCfg.max_frames.offset, ctypes.sizeof(_lib.VoxMimiReq)]
    assert got == exp


def test_create_without_gpu_fails_loudly(lib):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2602_00269_b200.config import tiny
    from paper_2602_00269_b200.device import VoxDevice

    with pytest.raises(RuntimeError):
        VoxDevice(tiny())
    from paper_2602_00269_b200.config import tiny_mimi
    from paper_2602_00269_b200.mimi import MimiDecoder

    with pytest.raises(RuntimeError):
        MimiDecoder(tiny_mimi())


def test_sm100a_cubin_contains_tcgen05_and_tma():
    import shutil
    import subprocess

    so = ROOT / "paper_2602_00269_b200" / "libvoxb200.so"
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(tool).exists():
        pytest.skip("cuobjdump missing")
    sass = subprocess.run([tool, "-sass", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run([tool, "-lelf", str(so)], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnem in sass, mnem
