"""ctypes binding of libhybrimoe.so (include/hybrimoe.h).

This is the only place that touches the native library.  Status codes map
1:1 onto the reference's exception types; there is no Python
fallback for anything the library implements -- if the library cannot be
loaded, importing the package fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .errors import CalibrationError, EvictionError, PlanInvariantError

_LIB_PATH = Path(__file__).resolve().parent / "libhybrimoe.so"

HM_OK, HM_EVALUE, HM_EEVICTION, HM_EPLAN, HM_ERUNTIME, HM_ECALIBRATION, HM_EASSERT, HM_ECUDA = range(8)
HM_PREDICT_LIVE = -1  # forward_layer n_pred: the runtime's live look-ahead predicts
DEV_CPU, DEV_GPU, DEV_PCIE = 0, 1, 2
KIND_COMPUTE, KIND_TRANSFER = 0, 1
ASSIGN_CPU, ASSIGN_GPU_CACHED, ASSIGN_GPU_TRANSFER = 0, 1, 2


class Profile(C.Structure):
    _fields_ = [
        ("gpu_time_per_expert", C.c_double),
        ("cpu_slope", C.c_double),
        ("transfer_bandwidth", C.c_double),
        ("transfer_latency", C.c_double),
        ("gpu_saturation_load", C.c_int64),
        ("gpu_slope", C.c_double),
        ("cpu_first_expert_penalty", C.c_double),
        ("shared_expert_time", C.c_double),
        ("non_expert_time", C.c_double),
    ]


class Task(C.Structure):
    _fields_ = [("ref", C.c_uint32), ("_pad", C.c_int32), ("load", C.c_int64)]


class Event(C.Structure):
    _fields_ = [("device", C.c_int32), ("kind", C.c_int32), ("ref", C.c_uint32), ("_pad", C.c_int32),
                ("start", C.c_double), ("end", C.c_double)]


class Assign(C.Structure):
    _fields_ = [("ref", C.c_uint32), ("how", C.c_int32)]


class Candidate(C.Structure):
    _fields_ = [("ref", C.c_uint32), ("layer_distance", C.c_int32), ("predicted_load", C.c_int64),
                ("gain", C.c_double), ("cost", C.c_double)]


class EngineConfig(C.Structure):
    _fields_ = [
        ("num_layers", C.c_int32), ("num_routed", C.c_int32), ("num_activated", C.c_int32),
        ("scheduling", C.c_int32), ("cache_policy", C.c_int32), ("prefetch", C.c_int32),
        ("validate", C.c_int32), ("split_point", C.c_int32), ("capacity", C.c_int64),
        ("expert_bytes", C.c_double), ("collect", C.c_int32), ("_pad", C.c_int32),
    ]


class PassResult(C.Structure):
    _fields_ = [("latency", C.c_double), ("busy", C.c_double * 3), ("lookups", C.c_int64),
                ("hits", C.c_int64), ("inserts", C.c_int64), ("evictions", C.c_int64),
                ("prefetch_issued", C.c_int64), ("prefetch_hits", C.c_int64),
                ("prefetch_expired", C.c_int64)]


class RecordSizes(C.Structure):
    _fields_ = [("n_lookups", C.c_int32), ("n_events", C.c_int32), ("n_assign", C.c_int32),
                ("n_demand", C.c_int32), ("n_candidates", C.c_int32), ("n_chosen", C.c_int32),
                ("expired", C.c_int32), ("n_selected", C.c_int32), ("prefetch_evict_error", C.c_int32),
                ("_pad", C.c_int32), ("makespan", C.c_double),
                ("budget", C.c_double)]


class Group(C.Structure):
    _fields_ = [("w13", C.c_void_p), ("w2", C.c_void_p), ("row_begin", C.c_int32),
                ("row_count", C.c_int32)]


def _load():
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python -m paper_2504_05897_b200._build` "
            "(or __graft_entry__.build()); there is no Python fallback")
    return C.CDLL(str(_LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)


lib = _load()

P = C.POINTER
vp = C.c_void_p
i32, i64, u32, f64, u8 = C.c_int32, C.c_int64, C.c_uint32, C.c_double, C.c_uint8
_SIGS = {
    "hm_last_error": ([C.c_char_p, C.c_size_t], C.c_int),
    "hm_version": ([], C.c_char_p),
    "hm_profile_check": ([P(Profile)], C.c_int),
    "hm_gpu_time": ([P(Profile), i64, P(f64)], C.c_int),
    "hm_cpu_time": ([P(Profile), i64, i64, P(f64)], C.c_int),
    "hm_transfer_time": ([P(Profile), f64, P(f64)], C.c_int),
    "hm_simulate_schedule": ([P(Task), C.c_int, P(Task), C.c_int, P(Profile), f64, P(Event), P(C.c_int),
                              P(Assign), P(C.c_int), P(f64)], C.c_int),
    "hm_plan_all_cpu": ([P(Task), C.c_int, P(Profile), P(Event), P(C.c_int), P(Assign), P(C.c_int), P(f64)],
                        C.c_int),
    "hm_plan_all_gpu": ([P(Task), C.c_int, P(Task), C.c_int, P(Profile), f64, P(Event), P(C.c_int),
                         P(Assign), P(C.c_int), P(f64)], C.c_int),
    "hm_select_plan_tasks": ([P(Task), C.c_int, P(Task), C.c_int, P(Profile), f64, P(Event), P(C.c_int),
                              P(Assign), P(C.c_int), P(f64)], C.c_int),
    "hm_select_plan": ([vp, C.c_int, P(i64), C.c_int, P(Profile), f64, P(Event), P(C.c_int), P(Assign),
                        P(C.c_int), P(f64)], C.c_int),
    "hm_check_plan": ([P(Event), C.c_int, P(Assign), C.c_int, f64], C.c_int),
    "hm_pcie_idle_budget": ([P(Event), C.c_int, f64, P(f64)], C.c_int),
    "hm_oracle_optimal": ([P(Task), C.c_int, P(u8), P(Profile), f64, C.c_int, P(f64)], C.c_int),
    "hm_evaluator_create": ([P(Profile), f64, P(vp)], C.c_int),
    "hm_evaluator_destroy": ([vp], None),
    "hm_evaluator_makespan": ([vp, P(i64), C.c_int, P(i64), C.c_int, P(f64)], C.c_int),
    "hm_evaluator_size": ([vp, P(i64)], C.c_int),
    "hm_cache_create": ([i64, P(vp)], C.c_int),
    "hm_cache_destroy": ([vp], None),
    "hm_cache_capacity": ([vp, P(i64)], C.c_int),
    "hm_cache_lookup": ([vp, u32, C.c_int, P(C.c_int)], C.c_int),
    "hm_cache_insert": ([vp, u32, C.c_int, vp, P(u32), P(C.c_int)], C.c_int),
    "hm_cache_victim": ([vp, C.c_int, vp, P(u32)], C.c_int),
    "hm_cache_is_resident": ([vp, u32, P(C.c_int)], C.c_int),
    "hm_cache_is_pinned": ([vp, u32, P(C.c_int)], C.c_int),
    "hm_cache_pin": ([vp, u32], C.c_int),
    "hm_cache_unpin": ([vp, u32], C.c_int),
    "hm_cache_clear_pinned": ([vp], C.c_int),
    "hm_cache_add_resident": ([vp, u32], C.c_int),
    "hm_cache_remove_resident": ([vp, u32], C.c_int),
    "hm_cache_clear_resident": ([vp], C.c_int),
    "hm_cache_counts": ([vp, P(i64), P(i64)], C.c_int),
    "hm_cache_resident": ([vp, P(u32), i64, P(i64)], C.c_int),
    "hm_cache_pinned": ([vp, P(u32), i64, P(i64)], C.c_int),
    "hm_cache_last_access": ([vp, u32, P(i64), P(C.c_int)], C.c_int),
    "hm_cache_frequency": ([vp, u32, P(i64), P(C.c_int)], C.c_int),
    "hm_cache_set_last_access": ([vp, u32, i64], C.c_int),
    "hm_cache_set_frequency": ([vp, u32, i64], C.c_int),
    "hm_cache_tick": ([vp, P(i64)], C.c_int),
    "hm_cache_next_tick": ([vp, P(i64)], C.c_int),
    "hm_cache_slot": ([vp, u32, P(i64)], C.c_int),
    "hm_mrs_create": ([C.c_int, C.c_int, f64, C.c_int, P(vp)], C.c_int),
    "hm_mrs_destroy": ([vp], None),
    "hm_mrs_update": ([vp, C.c_int, P(f64), C.c_int], C.c_int),
    "hm_mrs_get": ([vp, u32, P(f64)], C.c_int),
    "hm_mrs_set": ([vp, u32, f64], C.c_int),
    "hm_mrs_table": ([vp, P(f64)], C.c_int),
    "hm_mrs_params": ([vp, P(f64), P(C.c_int), P(C.c_int), P(C.c_int)], C.c_int),
    "hm_top_p_filter": ([P(f64), C.c_int, C.c_int, P(f64)], C.c_int),
    "hm_evaluate_gain": ([u32, C.c_int, P(i64), C.c_int, vp, vp, P(f64)], C.c_int),
    "hm_select_prefetches": ([P(Candidate), C.c_int, f64, P(u32), P(C.c_int)], C.c_int),
    "hm_engine_create": ([P(EngineConfig), P(Profile), vp, vp, vp, P(vp)], C.c_int),
    "hm_engine_destroy": ([vp], None),
    "hm_engine_set_fixed_pinned": ([vp, P(u32), C.c_int], C.c_int),
    "hm_engine_begin_pass": ([vp], C.c_int),
    "hm_engine_run_layer": ([vp, C.c_int, P(i64), P(f64), C.c_int, P(i32), P(i64), C.c_int], C.c_int),
    "hm_engine_end_pass": ([vp, P(PassResult)], C.c_int),
    "hm_engine_layer_makespans": ([vp, P(f64), C.c_int, P(C.c_int)], C.c_int),
    "hm_engine_record_sizes": ([vp, P(RecordSizes)], C.c_int),
    "hm_engine_record": ([vp, P(u32), P(u8), P(Event), P(Assign), P(u32), P(u32), P(u8), P(Candidate), P(u32),
                          P(u32), P(u8), P(u32)], C.c_int),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res


def last_error() -> str:
    buf = C.create_string_buffer(4096)
    lib.hm_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(status: int) -> None:
    """Raise the reference's exception type for a non-zero status."""
    if status == HM_OK:
        return
    msg = last_error()
    if status == HM_EVALUE:
        raise ValueError(msg)
    if status == HM_EEVICTION:
        raise EvictionError(msg)
    if status == HM_EPLAN:
        raise PlanInvariantError(msg)
    if status == HM_ECALIBRATION:
        raise CalibrationError(msg)
    if status == HM_EASSERT:
        raise AssertionError(msg)
    raise RuntimeError(msg)


def pack(layer: int, expert: int) -> int:
    if not (0 <= layer < 65536 and 0 <= expert < 65536):
        raise ValueError(f"ExpertRef({layer}, {expert}) outside the packed 16-bit range")
    return (layer << 16) | expert


def unpack(r: int) -> tuple[int, int]:
    return r >> 16, r & 0xFFFF


def i64_array(values) -> np.ndarray:
    return np.ascontiguousarray(values, dtype=np.int64)


def f64_array(values) -> np.ndarray:
    return np.ascontiguousarray(values, dtype=np.float64)


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(P(ctype))


def symbols_declared() -> list[str]:
    """Every function name declared in include/hybrimoe.h."""
    import re

    hdr = (Path(__file__).resolve().parent.parent / "include" / "hybrimoe.h").read_text()
    body = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(hm_[a-z0-9_]+)\s*\(", body)))


class HmGroup(C.Structure):
    _fields_ = [("slot", C.c_int32), ("row_begin", C.c_int32), ("row_count", C.c_int32), ("_pad", C.c_int32)]


_DEV_SIGS = {
    "hm_router_topk": ([vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp],
                       C.c_int),
    "hm_score_sums": ([vp, C.c_int, C.c_int, vp, vp], C.c_int),
    "hm_router_logits": ([vp, vp, C.c_int, C.c_int, C.c_int, vp, vp], C.c_int),
    "hm_offsets": ([vp, C.c_int, vp, vp], C.c_int),
    "hm_permute": ([vp, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp], C.c_int),
    "hm_gather_rows": ([vp, vp, C.c_int, C.c_int, C.c_int, vp, vp], C.c_int),
    "hm_expert_ffn": ([vp, C.c_int, C.c_int, C.c_int, P(HmGroup), C.c_int, vp, C.c_int, vp, vp, C.c_int, vp],
                      C.c_int),
    "hm_combine": ([vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp, vp], C.c_int),
    "hm_mrs_update_dev": ([vp, vp, C.c_int, C.c_int, C.c_int, f64, vp], C.c_int),
    "hm_router_fused_small": ([vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int,
                               vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "hm_router_fused_mirror": ([vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int,
                                vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_uint32, vp], C.c_int),
    "hm_combine_tail": ([vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int,
                         f64, vp], C.c_int),
}
for _name, (_args, _res) in _DEV_SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res
FFN_AUTO, FFN_GEMV, FFN_GEMM, FFN_GEMV_SPLIT, FFN_GEMV_FUSED, FFN_GEMV_BULK = 0, 1, 2, 3, 4, 5

_HOST_SIGS = {
    "hm_cpu_pool_create": ([C.c_int, P(vp)], C.c_int),
    "hm_cpu_pool_destroy": ([vp], None),
    "hm_cpu_expert": ([vp, vp, C.c_int, C.c_int, vp, C.c_int, vp], C.c_int),
    "hm_cpu_has_avx512bf16": ([], C.c_int),
}
for _name, (_args, _res) in _HOST_SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res


class RuntimeConfig(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_routed", C.c_int32), ("num_activated", C.c_int32),
                ("hidden", C.c_int32), ("inter", C.c_int32), ("n_shared", C.c_int32), ("renormalize", C.c_int32),
                ("shared_gate_col", C.c_int32), ("capacity", C.c_int64), ("host_images", C.c_int64),
                ("cpu_threads", C.c_int32), ("max_tokens", C.c_int32), ("gpu_mrs", C.c_int32),
                ("residual", C.c_int32), ("ep_rank", C.c_int32), ("ep_world", C.c_int32),
                ("weight_bits", C.c_int32), ("_pad", C.c_int32)]


class LayerStats(C.Structure):
    _fields_ = [("makespan_planned", C.c_double), ("t_wait_router_us", C.c_double), ("t_decide_us", C.c_double),
                ("t_cpu_us", C.c_double), ("n_gpu", C.c_int32), ("n_cpu", C.c_int32), ("n_transfer", C.c_int32),
                ("n_prefetch", C.c_int32), ("bytes_gpu", C.c_int64), ("bytes_cpu", C.c_int64),
                ("bytes_h2d", C.c_int64)]


_RT_SIGS = {
    "hm_runtime_create": ([P(RuntimeConfig), vp, P(vp)], C.c_int),
    "hm_runtime_destroy": ([vp], None),
    "hm_runtime_buffers": ([vp, P(vp), P(vp), P(C.c_size_t), P(i64)], C.c_int),
    "hm_runtime_image_of": ([vp, C.c_int, C.c_int, P(i64)], C.c_int),
    "hm_runtime_shared_slot": ([vp, C.c_int, C.c_int, P(i64)], C.c_int),
    "hm_runtime_forward_layer": ([vp, C.c_int, vp, vp, C.c_int, C.c_int, vp, P(i32), P(i64), C.c_int, vp,
                                  P(LayerStats)], C.c_int),
    "hm_runtime_last_request": ([vp, P(i64), P(f64)], C.c_int),
    "hm_runtime_device_mrs": ([vp, P(f64)], C.c_int),
    "hm_runtime_sync": ([vp], C.c_int),
}
for _name, (_args, _res) in _RT_SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res

for _name, (_args, _res) in {
    "hm_runtime_set_kernel_timing": ([vp, C.c_int], C.c_int),
    "hm_runtime_kernel_times": ([vp, P(f64), P(i64), P(i64), P(f64)], C.c_int),
    "hm_runtime_set_copy_timing": ([vp, C.c_int], C.c_int),
    "hm_runtime_copy_times": ([vp, P(f64), P(i64), P(i64), P(f64)], C.c_int),
    "hm_launch_count": ([], C.c_longlong),
}.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res
lib.hm_host_read_bw.argtypes = [vp, vp, C.c_size_t, C.c_int, P(f64)]
lib.hm_host_read_bw.restype = C.c_int

for _name, (_args, _res) in {
    "hm_runtime_set_ep_output": ([vp, vp], C.c_int),
    "hm_mask_nonhome": ([vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp], C.c_int),
    "hm_combine_f32": ([vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp], C.c_int),
    "hm_residual_add": ([vp, vp, C.c_int, C.c_int, vp, vp], C.c_int),
    "hm_runtime_preload": ([vp, P(u32), C.c_int], C.c_int),
    "hm_cpu_experts_amx": ([vp, P(vp), P(vp), P(C.c_int), C.c_int, C.c_int, C.c_int, P(vp)], C.c_int),
    "hm_cpu_experts_decode": ([vp, P(vp), P(vp), C.c_int, C.c_int, C.c_int, P(vp)], C.c_int),
    "hm_cpu_set_prefetch": ([C.c_int, C.c_int], C.c_int),
    "hm_engine_set_profile": ([vp, P(Profile)], C.c_int),
    "hm_runtime_forward_pass": ([vp, vp, P(vp), C.c_int, C.c_int, vp, vp, P(i64), i64, i64, C.c_int, f64, vp, vp,
                                 P(PassResult), P(vp)], C.c_int),
    "hm_predict_layers": ([P(i64), C.c_int, C.c_int, i64, C.c_int, i64, C.c_int, f64, P(i32), P(i64),
                           P(C.c_int)], C.c_int),
    "hm_cpu_set_decode_grain": ([C.c_int], C.c_int),
    "hm_cpu_set_decode_steal": ([C.c_int], C.c_int),
    "hm_cpu_decode_profile": ([C.c_int, vp, C.c_int], C.c_int),
    "hm_cpu_expert_q4": ([vp, vp, C.c_int, C.c_int, vp, C.c_int, vp], C.c_int),
    "hm_cpu_experts_decode_q4": ([vp, P(vp), P(vp), C.c_int, C.c_int, C.c_int, P(vp)], C.c_int),
    "hm_cpu_has_amx_bf16": ([], C.c_int),
    "hm_q4_image_bytes": ([C.c_int, C.c_int, P(C.c_size_t)], C.c_int),
    "hm_q4_quantize": ([vp, C.c_int, C.c_int, vp, vp], C.c_int),
    "hm_q4_dequantize": ([vp, C.c_int, C.c_int, vp, vp], C.c_int),
    "hm_expert_ffn_q4": ([vp, C.c_size_t, C.c_int, C.c_int, C.c_int, P(HmGroup), C.c_int, vp, C.c_int, vp, vp, vp,
                          C.c_int, C.c_int, vp], C.c_int),
    "hm_cpu_decode_profile_accum": ([P(C.c_int64), C.c_int], C.c_int),
    "hm_cpu_decode_profile_hist": ([P(C.c_int64), P(C.c_int64), C.c_int], C.c_int),
    "hm_bench_stream_read": ([vp, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.POINTER(C.c_float)], C.c_int),
    "hm_bench_expert_ffn": ([vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, C.c_int, C.c_int, vp,
                             P(C.c_float)], C.c_int),
    "hm_ep_create": ([C.c_int, C.c_int, C.c_int, C.c_int, P(vp)], C.c_int),
    "hm_ep_destroy": ([vp], None),
    "hm_ep_ipc_handles": ([vp, C.c_char_p, C.c_char_p], C.c_int),
    "hm_ep_open_peer": ([vp, C.c_int, C.c_char_p, C.c_char_p], C.c_int),
    "hm_ep_combine_allreduce": ([vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp], C.c_int),
    "hm_runtime_set_ep_exchange": ([vp, vp], C.c_int),
    "hm_ep_enable_dispatch": ([vp, C.c_int, C.c_int, C.c_int, C.c_char_p], C.c_int),
    "hm_ep_open_peer_dispatch": ([vp, C.c_int, C.c_char_p], C.c_int),
    "hm_runtime_set_ep_dispatch": ([vp, vp], C.c_int),
    "hm_ep_nccl_unique_id": ([C.c_char_p], C.c_int),
    "hm_ep_create_nccl": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int, C.c_int, C.c_int, P(vp)],
                          C.c_int),
    "hm_ep_uses_nccl": ([vp], C.c_int),
    "hm_ep_world": ([vp], C.c_int),
    "hm_ep_a2a_plan": ([vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int, P(C.c_int)], C.c_int),
    "hm_runtime_set_lookahead": ([vp, vp, C.c_int, C.c_int], C.c_int),
    "hm_lookahead": ([vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp], C.c_int),
}.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res


class A2aOp(C.Structure):
    """hm_a2a_op: one step of a rank's all-to-all(v) schedule (include/hybrimoe.h)."""
    _fields_ = [("kind", C.c_int32), ("peer", C.c_int32), ("src_row", C.c_int64), ("dst_row", C.c_int64),
                ("rows", C.c_int64)]


HM_A2A_SEND, HM_A2A_RECV, HM_A2A_COPY = 0, 1, 2
