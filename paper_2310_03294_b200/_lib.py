"""ctypes binding of libdistattn_b200.so (the C ABI in include/distattn_b200.h).

Loading never falls back to anything: a missing or unloadable library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libdistattn_b200.so"

i32, i64, f32, vp = C.c_int32, C.c_int64, C.c_float, C.c_void_p


class FwdArgs(C.Structure):
    _fields_ = [("q", vp), ("k", vp), ("v", vp),
                ("h_q", i64), ("h_kv", i64), ("rows_q", i64), ("rows_kv", i64), ("d", i64),
                ("o_in", vp), ("m_in", vp), ("l_in", vp),
                ("o_acc", vp), ("m_acc", vp), ("l_acc", vp),
                ("o_out", vp), ("lse_out", vp), ("degenerate_flag", vp),
                ("scale", f32), ("mask", C.c_int), ("finalize", C.c_int)]


class BwdArgs(C.Structure):
    _fields_ = [("q", vp), ("k", vp), ("v", vp), ("d_out", vp), ("lse", vp), ("d_vec", vp),
                ("h_q", i64), ("h_kv", i64), ("rows_q", i64), ("rows_kv", i64), ("d", i64),
                ("dq_acc", vp), ("dk_acc", vp), ("dv_acc", vp),
                ("accumulate_kv", C.c_int), ("scale", f32), ("mask", C.c_int),
                ("deterministic", C.c_int)]


class Shards(C.Structure):
    _fields_ = [("workers", i32), ("h_q", i64), ("h_kv", i64), ("rows", i64), ("d", i64),
                ("q", C.POINTER(vp)), ("k", C.POINTER(vp)), ("v", C.POINTER(vp)),
                ("out", C.POINTER(vp)), ("lse", C.POINTER(vp)), ("d_out", C.POINTER(vp)),
                ("dq", C.POINTER(vp)), ("dk", C.POINTER(vp)), ("dv", C.POINTER(vp))]


class RankOptions(C.Structure):
    _fields_ = [("transport", C.c_int), ("deterministic", C.c_int), ("nccl_max_ctas", C.c_int)]


TRANSPORT = {"ipc": 0, "nccl": 1, "none": 2}


class TraceRec(C.Structure):
    _fields_ = [("kind", i32), ("code", i32), ("step", i32), ("peer", i32), ("phase", i32),
                ("pad", i32), ("t0_ms", f32), ("t1_ms", f32)]


class Counters(C.Structure):
    _fields_ = [("kv_scalars", i64), ("q_scalars", i64), ("partial_scalars", i64),
                ("grad_scalars", i64), ("kv_messages", i64), ("q_messages", i64),
                ("partial_messages", i64), ("grad_messages", i64),
                ("attention_kernel_calls", i64), ("max_remote_chunks_held", i32)]

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_}


# exported symbol -> (restype, argtypes); the CPU test suite checks that every
# function declared in include/distattn_b200.h appears here and in the .so.
SIGNATURES = {
    "da_last_error": (C.c_char_p, []),
    "da_abi_version": (C.c_int, []),
    "da_stream_write_u32": (C.c_int, [vp, vp, C.c_uint32]),
    "da_rank_create": (C.c_int, [C.c_int, C.c_int, vp, vp, C.POINTER(vp)]),
    "da_rank_destroy": (None, [vp]),
    "da_rank_set_trace": (None, [vp, C.c_int]),
    "da_rank_trace": (C.c_int, [vp, C.c_int, vp, i64, C.POINTER(i64)]),
    "da_rank_forward_table": (C.c_int, [vp, i32, C.POINTER(i32), i64, C.POINTER(i32), i64, vp,
                                        vp, vp, i64, i64, i64, vp, vp, vp, vp]),
    "da_rank_backward_table": (C.c_int, [vp, i32, C.POINTER(i32), i64, C.POINTER(i32), i64, vp,
                                         vp, vp, vp, vp, vp]),
    "da_rank_restore": (C.c_int, [vp, vp, vp, vp, vp, vp, i64, i64, i64]),
    "da_rank_create_ex": (C.c_int, [C.c_int, C.c_int, vp, vp, vp, C.POINTER(vp)]),
    "da_rank_protocol": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(i32), i64,
                                   C.POINTER(i64)]),
    "da_rank_forward": (C.c_int, [vp, C.c_int, vp, vp, vp, i64, i64, i64, vp, vp, vp, vp]),
    "da_rank_backward": (C.c_int, [vp, C.c_int, vp, vp, vp, vp, vp, vp]),
    "da_stream_wait_u32_geq": (C.c_int, [vp, vp, C.c_uint32]),
    "da_device_supported": (C.c_int, []),
    "da_attn_fwd_chunk": (C.c_int, [C.POINTER(FwdArgs), vp]),
    "da_attn_merge": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, i64, vp]),
    "da_attn_finalize": (C.c_int, [vp, vp, vp, vp, vp, vp, i64, i64, i64, vp]),
    "da_check_degenerate": (C.c_int, [vp, vp]),
    "da_attn_bwd_preprocess": (C.c_int, [vp, vp, vp, i64, i64, i64, vp]),
    "da_attn_bwd_chunk": (C.c_int, [C.POINTER(BwdArgs), vp]),
    "da_convert_f32_bf16": (C.c_int, [vp, vp, i64, vp]),
    "da_schedule_build": (C.c_int, [C.c_int, C.c_int, C.POINTER(i32), C.POINTER(i32),
                                    C.POINTER(i64), C.POINTER(i32), C.POINTER(i64)]),
    "da_schedule_validate": (i64, [C.c_int, i32, C.POINTER(i32), i64, C.POINTER(i32), i64]),
    "da_schedule_validate_backward": (i64, [C.c_int, i32, C.POINTER(i32), i64, C.POINTER(i32),
                                            i64]),
    "da_run_forward": (C.c_int, [C.POINTER(Shards), C.c_int, C.POINTER(Counters), vp]),
    "da_run_backward_sched": (C.c_int, [C.POINTER(Shards), C.c_int, C.POINTER(Counters), vp]),
    "da_run_backward": (C.c_int, [C.POINTER(Shards), C.POINTER(Counters), vp]),
    "da_runtime_release": (None, []),
    "da_pipeline_create": (C.c_int, [i64, i64, i64, i64, i64, C.c_int, C.POINTER(vp)]),
    "da_pipeline_destroy": (None, [vp]),
    "da_pipeline_step": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, C.c_int, vp]),
    "da_pipeline_join": (C.c_int, [vp, vp, C.c_int]),
    "da_pipeline_outputs": (C.c_int, [vp, vp, vp, vp]),
    "da_run_forward_table": (C.c_int, [C.POINTER(Shards), i32, C.POINTER(i32), i64,
                                       C.POINTER(i32), i64, C.POINTER(Counters), vp]),
    "da_run_backward_table": (C.c_int, [C.POINTER(Shards), i32, C.POINTER(i32), i64,
                                        C.POINTER(i32), i64, C.POINTER(Counters), vp]),
    "da_rng_uniform": (C.c_int, [C.c_uint64, i64, C.c_double, C.c_double, C.c_int, vp, vp]),
    "da_debug_set_bwd_trace": (None, [vp]),
    "da_debug_set_fwd_trace": (None, [vp]),
    "da_debug_scores": (C.c_int, [vp, vp, i64, vp, vp]),
    "da_host_attn_update": (C.c_int, [vp, i64, vp, vp, i64, i64, vp, vp, vp, C.c_int,
                                      C.c_double]),
    "da_host_attn_merge": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, i64]),
    "da_host_attn_finalize": (C.c_int, [vp, vp, vp, i64, i64, vp, vp]),
    "da_host_backward_aux": (C.c_int, [vp, vp, i64, i64, vp]),
    "da_host_attn_backward": (C.c_int, [vp, i64, vp, vp, i64, i64, vp, vp, vp, C.c_int,
                                        C.c_double, vp, vp, vp]),
    "da_host_dense_attention": (C.c_int, [vp, i64, vp, vp, i64, i64, C.c_int, C.c_double, vp,
                                          vp]),
}

_lib = None


def lib() -> C.CDLL:
    """Loads the in-tree library (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        path = Path(os.environ.get("DISTATTN_B200_LIB", LIB_PATH))
        if not path.exists():
            raise RuntimeError(
                f"{path} is missing: build it with `python -m paper_2310_03294_b200.build` "
                "(there is no CPU fallback)")
        handle = C.CDLL(str(path), mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib
