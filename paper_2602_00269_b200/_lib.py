"""ctypes binding of the C-ABI in include/voxb200.h.

This is the reference-side binding a maintainer would add (the reference is
pure Python, so its FFI is ctypes).  Every status code maps onto the
reference exception class it replaces (errors.py:4-77).  There is no CPU
fallback: if ``libvoxb200.so`` is missing or no sm_100 GPU is present, calls
raise.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

from ._ref import errors

LIB_PATH = Path(__file__).resolve().parent / "libvoxb200.so"

VOX_FWD_SAMPLE = 1
VOX_FWD_FULL_LOGITS = 2
VOX_FWD_SYNC = 4
VOX_FWD_NO_GRAPH = 8


class VoxModelCfg(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
        ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("d_ff", C.c_int32),
        ("vocab", C.c_int32),
        ("rope_theta", C.c_float), ("rms_eps", C.c_float), ("embed_scale", C.c_float),
        ("text_vocab", C.c_int32),
        ("audio_base", C.c_int32), ("codebook_size", C.c_int32), ("frame_tokens", C.c_int32),
        ("page_size", C.c_int32), ("n_pages", C.c_int32), ("max_slots", C.c_int32),
        ("max_ctx", C.c_int32), ("max_rows", C.c_int32),
        ("detok_enabled", C.c_int32),
        ("latent_dim", C.c_int32), ("decoder_dim", C.c_int32), ("n_rates", C.c_int32),
        ("rates", C.c_int32 * 4),
        ("max_detok_frames", C.c_int32),
        ("qkv_bias", C.c_int32),
        ("n_codebooks", C.c_int32),
        ("ext_dim", C.c_int32),
    ]


class VoxSampling(C.Structure):
    _fields_ = [
        ("temperature", C.c_double), ("top_p", C.c_double), ("repetition_penalty", C.c_double),
        ("top_k", C.c_int32), ("penalty_window", C.c_int32),
    ]


class VoxRow(C.Structure):
    _fields_ = [("slot", C.c_int32), ("pos", C.c_int32), ("token", C.c_int32), ("sample", C.c_int32)]


class VoxWindow(C.Structure):
    _fields_ = [
        ("slot", C.c_int32), ("index", C.c_int32), ("start", C.c_int32), ("length", C.c_int32),
        ("new_tokens", C.c_int32), ("final", C.c_int32),
    ]


class VoxMimiCfg(C.Structure):
    _fields_ = [
        ("n_q", C.c_int32), ("n_semantic", C.c_int32), ("cb_size", C.c_int32), ("cb_dim", C.c_int32),
        ("hidden", C.c_int32), ("n_layers", C.c_int32), ("n_heads", C.c_int32), ("ffn", C.c_int32),
        ("window", C.c_int32), ("rope_theta", C.c_float), ("eps", C.c_float),
        ("filters", C.c_int32), ("n_ratios", C.c_int32), ("ratios", C.c_int32 * 4),
        ("kernel", C.c_int32), ("last_kernel", C.c_int32), ("res_kernel", C.c_int32), ("compress", C.c_int32),
        ("max_slots", C.c_int32), ("max_frames", C.c_int32),
    ]


class VoxMimiReq(C.Structure):
    _fields_ = [("slot", C.c_int32), ("n_frames", C.c_int32)]


class VoxCosyCfg(C.Structure):
    _fields_ = [
        ("vocab", C.c_int32), ("ref_tokens", C.c_int32),
        ("d_enc", C.c_int32), ("enc_layers", C.c_int32), ("enc_heads", C.c_int32), ("enc_ffn", C.c_int32),
        ("mel", C.c_int32),
        ("d_est", C.c_int32), ("est_layers", C.c_int32), ("est_heads", C.c_int32), ("est_ffn", C.c_int32),
        ("n_steps", C.c_int32),
        ("cfg_rate", C.c_float), ("rope_theta", C.c_float), ("eps", C.c_float),
        ("voc_ch", C.c_int32), ("n_ratios", C.c_int32), ("ratios", C.c_int32 * 4), ("voc_kernel", C.c_int32),
        ("res_kernel", C.c_int32), ("post_kernel", C.c_int32), ("n_fft", C.c_int32), ("hop", C.c_int32),
        ("slope", C.c_float),
        ("max_slots", C.c_int32), ("max_tokens", C.c_int32), ("max_chunk", C.c_int32),
    ]


class VoxCosyReq(C.Structure):
    _fields_ = [("slot", C.c_int32), ("n_tokens", C.c_int32)]


# status -> exception (VoxStatus in include/voxb200.h)
_STATUS_TO_EXC = {
    1: ValueError,
    2: errors.BatchTooLarge,
    3: errors.DegenerateDistribution,
    4: errors.CodebookMismatch,
    5: errors.WindowRuleViolation,
    6: errors.CacheMissing,
    7: errors.PromptTooLong,
    8: errors.InvalidTokenCount,
    9: ValueError,
    10: MemoryError,
    11: RuntimeError,
    12: RuntimeError,
    13: errors.EmptyBatch,
}

_P = C.c_void_p
_i32p = C.POINTER(C.c_int32)
_u64p = C.POINTER(C.c_uint64)
_f32p = C.POINTER(C.c_float)

_SIGS = {
    "vox_abi_version": (C.c_int, []),
    "vox_last_error": (C.c_char_p, [_P]),
    "vox_create": (C.c_int, [C.c_int, C.POINTER(VoxModelCfg), C.c_uint64, C.POINTER(_P)]),
    "vox_destroy": (None, [_P]),
    "vox_admit": (C.c_int, [_P, C.c_uint64, C.c_int32, C.c_int32, C.POINTER(VoxSampling), _i32p]),
    "vox_release": (C.c_int, [_P, C.c_int32]),
    "vox_page_table": (C.c_int, [_P, C.c_int32, _i32p, C.c_int32, _i32p]),
    "vox_read_tokens": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _i32p]),
    "vox_write_tokens": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _i32p]),
    "vox_slot_info": (C.c_int, [_P, C.c_int32, _i32p, _i32p]),
    "vox_forward": (C.c_int, [_P, C.POINTER(VoxRow), C.c_int32, C.c_uint32, _f32p, _i32p]),
    "vox_forward_steps": (C.c_int, [_P, C.POINTER(VoxRow), C.c_int32, C.c_int32, C.c_uint32]),
    "vox_read_logits": (C.c_int, [_P, _f32p, C.c_int32, C.c_int32, _i32p, _i32p, _i32p]),
    "vox_forward_seq": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "vox_forward_wait": (C.c_int, [_P, C.c_int64]),
    "vox_sample_logits": (C.c_int, [_P, _f32p, C.c_int32, C.c_int32, C.POINTER(VoxSampling),
                                    _i32p, C.c_int32, _i32p, _u64p, _u64p, _i32p, _i32p, _i32p]),
    "vox_detok": (C.c_int, [_P, C.POINTER(VoxWindow), C.c_int32, _f32p, _i32p,
                            C.POINTER(C.c_int64)]),
    "vox_ticket_query": (C.c_int, [_P, C.c_int64, _i32p, C.POINTER(C.c_double)]),
    "vox_ticket_pcm": (C.c_int, [_P, C.c_int64, C.POINTER(_f32p), _i32p]),
    "vox_clock_reset": (C.c_int, [_P]),
    "vox_synchronize": (C.c_int, [_P]),
    "vox_streams": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P)]),
    "vox_timing_enable": (C.c_int, [_P, C.c_int32]),
    "vox_timing_read": (C.c_int, [_P, C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                  C.POINTER(C.c_double)]),
    "vox_launch_count": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "vox_sm_partition": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "vox_trace_arm": (C.c_int, [_P, C.c_int64]),
    "vox_trace_read": (C.c_int, [_P, _P, C.c_int64, C.POINTER(C.c_int64)]),
    "vox_debug_detok": (C.c_int, [_P, C.c_int32, _f32p, C.c_size_t, C.POINTER(C.c_uint16), C.c_size_t]),
    "vox_gemm_test": (C.c_int, [_P, C.POINTER(C.c_uint16), C.POINTER(C.c_uint16), _f32p, C.c_int32, C.c_int32,
                                C.c_int32, C.c_int32, C.c_int32, _f32p, C.POINTER(C.c_double)]),
    "vox_read_weight": (C.c_int, [_P, C.c_char_p, C.c_int32, _P, C.c_size_t]),
    "vox_read_kv": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _f32p, _f32p]),
    "vox_write_frame": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _i32p]),
    "vox_read_frame": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _i32p]),
    "vox_project_ext": (C.c_int, [_P, _P, C.c_int32]),
    "vox_link_tokens": (C.c_int, [_P, _P, _i32p, C.c_int32, C.c_int32, C.c_int32]),
    "vox_copy_tokens": (C.c_int, [_P, _P, _i32p, C.c_int32]),
    "vox_mimi_create": (C.c_int, [C.c_int, C.POINTER(VoxMimiCfg), C.c_uint64, C.POINTER(_P)]),
    "vox_mimi_destroy": (None, [_P]),
    "vox_mimi_last_error": (C.c_char_p, [_P]),
    "vox_mimi_open": (C.c_int, [_P, _i32p]),
    "vox_mimi_close": (C.c_int, [_P, C.c_int32]),
    "vox_mimi_decode": (C.c_int, [_P, C.POINTER(VoxMimiReq), C.c_int32, _i32p, _f32p, C.POINTER(C.c_int64)]),
    "vox_mimi_launch_count": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "vox_mimi_last_ms": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "vox_cosy_create": (C.c_int, [C.c_int, C.POINTER(VoxCosyCfg), C.c_uint64, C.POINTER(_P)]),
    "vox_cosy_destroy": (None, [_P]),
    "vox_cosy_last_error": (C.c_char_p, [_P]),
    "vox_cosy_open": (C.c_int, [_P, C.c_uint64, _i32p]),
    "vox_cosy_close": (C.c_int, [_P, C.c_int32]),
    "vox_cosy_decode": (C.c_int, [_P, C.POINTER(VoxCosyReq), C.c_int32, _i32p, _f32p, C.POINTER(C.c_int64)]),
    "vox_cosy_last_ms": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "vox_cosy_launch_count": (C.c_int, [_P, C.POINTER(C.c_int64)]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path: Path | str = LIB_PATH) -> C.CDLL:
    """Load the library (no compute); raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path)
    if not p.exists():
        raise ImportError(
            f"{p} not built: run `python -m paper_2602_00269_b200.build` (nvcc, sm_100a). "
            "There is no CPU fallback."
        )
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.vox_abi_version() != 1:
        raise ImportError("libvoxb200.so ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int, ctx=None, mimi=None, cosy=None) -> None:
    if rc == 0:
        return
    if cosy is not None:
        msg = load().vox_cosy_last_error(cosy)
    elif mimi is not None:
        msg = load().vox_mimi_last_error(mimi)
    else:
        msg = load().vox_last_error(ctx)
    text = msg.decode() if msg else f"status {rc}"
    raise _STATUS_TO_EXC.get(rc, RuntimeError)(text)
