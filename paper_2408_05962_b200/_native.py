"""ctypes declarations for libhiccl.so (include/hiccl.h).

The library is built in-tree (``python -m paper_2408_05962_b200.build``);
importing this module loads it and fails loudly if it is missing — there is
no Python or CPU fallback for the executor.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# HICCL_LIB_PATH: an alternative build of the same library (A/B experiments)
LIB_PATH = Path(os.environ.get("HICCL_LIB_PATH") or
                Path(__file__).resolve().parent / "lib" / "libhiccl.so")

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_2408_05962_b200.build` "
        "(there is no fallback implementation)")

lib = C.CDLL(str(LIB_PATH))

P = C.POINTER
vp = C.c_void_p
i32 = C.c_int
i64 = C.c_int64
u64 = C.c_uint64
sz = C.c_size_t
cp = C.c_char_p


class MachineDesc(C.Structure):
    _fields_ = [("hierarchy", P(i32)), ("num_levels", i32), ("gpus_per_node", i32),
                ("transport", P(cp))]


class PlanInfo(C.Structure):
    _fields_ = [(n, i32) for n in ("world_size", "num_transfers", "num_buffers", "num_stages",
                                   "slots", "depth", "stripe", "ring")]


class Transfer(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("id", "src", "dst", "src_buf", "dst_buf", "reduce", "op",
                                         "stage", "slot", "channel", "stripe", "level", "step",
                                         "n_deps")] + \
               [(n, C.c_int64) for n in ("src_off", "dst_off", "count")]


class Model(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("launch", "step", "push_bw", "pull_bw", "hbm_bw",
                                          "ll_launch", "ll_step", "ll_bw", "ll_in_bw",
                                          "ll_bidir_bw", "nvls_read_bw", "nvls_store_bw",
                                          "nvls_bidir_bw", "nvls_reduce_bw", "pull_uni_bw",
                                          "push_uni_bw", "nvls_launch")]


class TuneResult(C.Structure):
    _fields_ = [("formulation", i32), ("ring", i32), ("pipeline", i32), ("seconds", C.c_double),
                ("copy_mode", i32), ("nvls", i32)]


class ExecConfig(C.Structure):
    _fields_ = [("device", i32), ("exec_index", i32), ("num_execs", i32),
                ("rank_to_exec", P(i32)), ("dtype", i32), ("ctas", i32), ("threads", i32),
                ("copy_mode", i32), ("timeout_s", C.c_double), ("execs_per_device", i32)]


class ExecStats(C.Structure):
    _fields_ = [(n, i32) for n in ("num_steps", "num_items", "num_waits", "ctas", "threads")] + \
               [(n, C.c_int64) for n in ("bytes_in", "bytes_out", "remote_bytes", "arena_bytes")] + \
               [("nvls_items", i32), ("paired_waits", i32), ("whole_waits", i32),
                ("copy_mode", i32), ("tma_steps", i32), ("staged_steps", i32)]


_SIGS = {
    "hc_last_error": ([], cp),
    "hc_free": ([vp], None),
    "hc_version": ([], cp),
    "hc_program_create": ([i32, P(vp)], i32),
    "hc_program_destroy": ([vp], None),
    "hc_program_declare_buffer": ([vp, cp, i64, i32, i32], i32),
    "hc_program_add_multicast": ([vp, cp, i64, cp, i64, i64, i32, P(i32), i32], i32),
    "hc_program_add_reduction": ([vp, cp, i64, cp, i64, i64, P(i32), i32, i32, i32], i32),
    "hc_program_add_fence": ([vp], i32),
    "hc_program_validate": ([vp, P(vp)], i32),
    "hc_program_serialize": ([vp, P(vp)], i32),
    "hc_program_deserialize": ([cp, P(vp)], i32),
    "hc_program_id": ([vp, P(vp)], i32),
    "hc_program_preset": ([i32, i32, i32, i64, i32, i32, P(vp)], i32),
    "hc_plan_lower": ([vp, P(MachineDesc), i32, i32, i32, P(vp)], i32),
    "hc_plan_lower_staged_json": ([vp, P(MachineDesc), i32, i32, P(vp)], i32),
    "hc_plan_serialize": ([vp, P(vp)], i32),
    "hc_plan_deserialize": ([cp, P(vp)], i32),
    "hc_plan_destroy": ([vp], None),
    "hc_plan_get_info": ([vp, P(PlanInfo)], i32),
    "hc_plan_get_buffer": ([vp, i32, P(cp), P(i64), P(i32), P(i32)], i32),
    "hc_plan_get_transfers": ([vp, P(Transfer)], i32),
    "hc_plan_comm_matrix": ([vp, i32, P(i64)], i32),
    "hc_plan_schedule_summary": ([vp, i32, P(i32), i32, i32, i32, P(vp)], i32),
    "hc_plan_layout_summary": ([vp, i32, P(i32), i32, i32, i32, cp, P(vp)], i32),
    "hc_model_default": ([P(Model)], i32),
    "hc_plan_predict": ([vp, i32, P(Model), i32, i32, P(C.c_double)], i32),
    "hc_tune": ([i32, i32, i64, i32, P(Model), P(TuneResult)], i32),
    "hc_plan_predict_nvls": ([vp, i32, P(Model), P(C.c_double)], i32),
    "hc_tune_nvls": ([i32, i32, i64, i32, P(Model), P(TuneResult)], i32),
    "hc_t_ring": ([C.c_double, C.c_double, i32, C.c_double, i32, i32, C.c_double, P(C.c_double)], i32),
    "hc_t_tree": ([C.c_double, C.c_double, i32, C.c_double, i32, i32, C.c_double, P(C.c_double)], i32),
    "hc_bound": ([i32, i32, i32, i32, C.c_double, P(C.c_double)], i32),
    "hc_throughput": ([C.c_double, i32, C.c_double, P(C.c_double)], i32),
    "hc_exec_create": ([vp, P(ExecConfig), P(vp)], i32),
    "hc_exec_destroy": ([vp], None),
    "hc_exec_bind_buffer": ([vp, i32, cp, vp, sz], i32),
    "hc_exec_local_arena": ([vp, P(vp), P(sz)], i32),
    "hc_exec_bind_peer_arena": ([vp, i32, vp], i32),
    "hc_exec_local_flags": ([vp, P(vp), P(sz)], i32),
    "hc_exec_bind_peer_flags": ([vp, i32, vp], i32),
    "hc_exec_commit": ([vp], i32),
    "hc_exec_start": ([vp, vp], i32),
    "hc_exec_wait": ([vp], i32),
    "hc_exec_query": ([vp, P(i32)], i32),
    "hc_exec_get_stats": ([vp, P(ExecStats)], i32),
    "hc_exec_get_trace": ([vp, P(i64), i32], i32),
    "hc_enable_peer_access": ([P(i32), i32], i32),
    "hc_nvls_supported": ([i32, P(i32)], i32),
    "hc_window_create": ([P(i32), i32, sz, P(vp)], i32),
    "hc_window_open": ([i32, i32, sz, P(C.c_ubyte), P(vp)], i32),
    "hc_window_export": ([vp, P(C.c_ubyte)], i32),
    "hc_window_bind": ([vp], i32),
    "hc_window_export_memory": ([vp, P(C.c_ubyte)], i32),
    "hc_window_import_memory": ([vp, P(C.c_ubyte), P(vp)], i32),
    "hc_window_pointers": ([vp, i32, P(vp), P(vp), P(sz)], i32),
    "hc_window_destroy": ([vp], None),
    "hc_exec_bind_multicast": ([vp, cp, vp], i32),
    "hc_ipc_export": ([vp, P(C.c_ubyte), P(sz)], i32),
    "hc_ipc_import": ([P(C.c_ubyte), sz, i32, P(vp)], i32),
    "hc_ipc_close": ([vp], i32),
    "hc_device_range": ([vp, P(vp), P(sz)], i32),
    "hc_device_alloc": ([i32, sz, P(vp)], i32),
    "hc_device_free": ([i32, vp], i32),
    "hc_device_count": ([P(i32)], i32),
    "hc_device_sync": ([i32], i32),
    "hc_device_fill": ([i32, vp, i64, i32, u64, i32, i64, vp], i32),
}

for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)
