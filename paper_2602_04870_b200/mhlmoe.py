"""Thin ctypes binding of the C ABI in include/mhlmoe.h (same names, argument
marshalling only: every step of the layer runs in libmhlmoe.so's kernels).

Tensors are passed as raw device pointers (``tensor.data_ptr()``); streams as the
raw ``cudaStream_t`` of ``torch.cuda.current_stream()``.  There is no fallback:
if the shared library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmhlmoe.so")

MHL_F32, MHL_BF16 = 0, 1
MHL_FLAG_LOOPBACK, MHL_FLAG_SIMT, MHL_FLAG_PAIR, MHL_FLAG_ROUTING_TOKENS, MHL_FLAG_FUSED_COMBINE = 1, 2, 4, 8, 16
MHL_FLAG_WINDOWED_COMBINE, MHL_FLAG_DET_DP, MHL_FLAG_REQUIRE_TC, MHL_FLAG_BWD_FUSED = 32, 64, 128, 256
STATUS = {0: "MHL_OK", 1: "MHL_ERR_INVALID_ARGUMENT", 2: "MHL_ERR_CONFIG", 3: "MHL_ERR_WORKSPACE_TOO_SMALL",
          4: "MHL_ERR_UNSUPPORTED", 5: "MHL_ERR_CUDA", 6: "MHL_ERR_NCCL", 7: "MHL_ERR_NONFINITE"}
EXPORTS = ["hp_plan_query", "mhl_get_unique_id", "hp_plan", "hp_plan_info", "hp_plan_destroy", "mhlmoe_forward",
           "mhlmoe_backward", "mhlmoe_train_step_host", "mhlmoe_train_step_host_pipelined", "mhl_host_drain",
           "mhlmoe_update_bias", "mhl_check_device_status",
           "mhl_launch_count",
           "mhl_a2a_bytes_posted", "mhl_set_step_timing", "mhl_step_times", "mhl_kernel_paths", "mhl_dp_reduce",
           "mhl_status_string", "mhl_last_error"]
# mhl_kernel_paths bits (include/mhlmoe.h MHL_PATH_*)
PATHS = {"router_tc": 1 << 0, "router_blk": 1 << 1, "router_simt": 1 << 2, "expert_fwd_tc": 1 << 3,
         "expert_fwd_pair": 1 << 4, "expert_fwd_simt": 1 << 5, "expert_bwd_tc": 1 << 6, "expert_bwd_simt": 1 << 7,
         "router_bwd_tc": 1 << 8, "router_bwd_simt": 1 << 9, "proj_pinned": 1 << 10, "fused_combine": 1 << 11,
         "a2a_nccl": 1 << 12, "a2a_loopback": 1 << 13, "windowed_combine": 1 << 14,
         "expert_bwd_fused": 1 << 15}


class MhlError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: {STATUS.get(status, status)}: {detail}")
        self.status = status


class mhl_config(ctypes.Structure):
    _fields_ = [("tokens", ctypes.c_int64), ("d_model", ctypes.c_int32), ("n_heads", ctypes.c_int32),
                ("d_head", ctypes.c_int32), ("n_experts", ctypes.c_int32), ("top_k", ctypes.c_int32),
                ("d_expert", ctypes.c_int32), ("dtype", ctypes.c_int32), ("world_size", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("flags", ctypes.c_uint32)]


class mhl_plan_info(ctypes.Structure):
    _fields_ = [("head_begin", ctypes.c_int32), ("head_end", ctypes.c_int32), ("tokens_global", ctypes.c_int64),
                ("a2a_bytes_per_peer", ctypes.c_uint64), ("a2a_bytes_per_rank", ctypes.c_uint64),
                ("saved_bytes", ctypes.c_uint64), ("workspace_bytes", ctypes.c_uint64),
                ("io_bytes", ctypes.c_uint64), ("max_tiles", ctypes.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class mhl_weights(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("W_in", "W_out", "W_r", "bias", "W1", "W2")]


class mhl_grads(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("dW_in", "dW_out", "dW_r", "dW1", "dW2")]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run paper_2602_04870_b200.build (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I = ctypes.c_void_p, ctypes.c_int
    sig = {
        "hp_plan_query": (I, [ctypes.POINTER(mhl_config), ctypes.POINTER(mhl_plan_info)]),
        "mhl_get_unique_id": (I, [ctypes.c_char_p]),
        "hp_plan": (I, [ctypes.POINTER(mhl_config), ctypes.c_char_p, ctypes.POINTER(P)]),
        "hp_plan_info": (I, [P, ctypes.POINTER(mhl_plan_info)]),
        "hp_plan_destroy": (I, [P]),
        "mhlmoe_forward": (I, [P, P, ctypes.POINTER(mhl_weights), P, P, P, ctypes.c_size_t, P, P, P]),
        "mhlmoe_backward": (I, [P, P, ctypes.POINTER(mhl_weights), P, P, P, ctypes.POINTER(mhl_grads), P,
                                ctypes.c_size_t, P]),
        "mhlmoe_train_step_host": (I, [P, P, P, ctypes.POINTER(mhl_weights), P, P, ctypes.POINTER(mhl_grads), P,
                                       P, P, ctypes.c_size_t, P]),
        "mhlmoe_train_step_host_pipelined": (I, [P, P, P, ctypes.POINTER(mhl_weights), P, P,
                                                 ctypes.POINTER(mhl_grads), P, P, P, ctypes.c_size_t, P]),
        "mhl_host_drain": (I, [P, P]),
        "mhlmoe_update_bias": (I, [P, P, P, ctypes.c_float, P]),
        "mhl_check_device_status": (I, [P]),
        "mhl_launch_count": (ctypes.c_uint64, [P]),
        "mhl_a2a_bytes_posted": (ctypes.c_uint64, [P]),
        "mhl_set_step_timing": (I, [P, I]),
        "mhl_step_times": (ctypes.c_int32, [P, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_double),
                                            ctypes.POINTER(ctypes.c_int32), ctypes.c_int32]),
        "mhl_kernel_paths": (ctypes.c_uint32, [P, I]),
        "mhl_dp_reduce": (I, [P, P, P, P, ctypes.c_size_t, P]),
        "mhl_status_string": (ctypes.c_char_p, [I]),
        "mhl_last_error": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    return lib


_lib = _load()


def _check(status: int, where: str):
    if status != 0:
        raise MhlError(status, where, _lib.mhl_last_error().decode())


def make_config(T_loc, d, N_h, d_h, N_e, k, d_e, dtype="bf16", world_size=1, rank=0, flags=0) -> mhl_config:
    return mhl_config(int(T_loc), int(d), int(N_h), int(d_h), int(N_e), int(k), int(d_e),
                      MHL_BF16 if dtype == "bf16" else MHL_F32, int(world_size), int(rank), int(flags))


def hp_plan_query(cfg: mhl_config) -> dict:
    info = mhl_plan_info()
    _check(_lib.hp_plan_query(ctypes.byref(cfg), ctypes.byref(info)), "hp_plan_query")
    return info.as_dict()


def mhl_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.mhl_get_unique_id(buf), "mhl_get_unique_id")
    return buf.raw


@dataclass
class Plan:
    handle: ctypes.c_void_p
    cfg: mhl_config
    info: dict

    def __del__(self):
        try:
            if self.handle:
                _lib.hp_plan_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def hp_plan(cfg: mhl_config, nccl_id: bytes | None = None) -> Plan:
    h = ctypes.c_void_p()
    _check(_lib.hp_plan(ctypes.byref(cfg), nccl_id, ctypes.byref(h)), "hp_plan")
    info = mhl_plan_info()
    _check(_lib.hp_plan_info(h, ctypes.byref(info)), "hp_plan_info")
    return Plan(h, cfg, info.as_dict())


def hp_plan_info(plan: Plan) -> dict:
    info = mhl_plan_info()
    _check(_lib.hp_plan_info(plan.handle, ctypes.byref(info)), "hp_plan_info")
    return info.as_dict()


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def weights_struct(W: dict) -> mhl_weights:
    return mhl_weights(*[W[n].data_ptr() for n in ("W_in", "W_out", "W_r", "b", "W1", "W2")])


def grads_struct(g: dict) -> mhl_grads:
    return mhl_grads(*[(g[n].data_ptr() if g.get(n) is not None else None)
                       for n in ("dW_in", "dW_out", "dW_r", "dW1", "dW2")])


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def mhlmoe_forward(plan: Plan, x, W, out, saved, workspace, topk_idx=None, gates=None, stream=None):
    ws = weights_struct(W) if isinstance(W, dict) else W
    _check(_lib.mhlmoe_forward(plan.handle, _ptr(x), ctypes.byref(ws), _ptr(out), _ptr(saved), _ptr(workspace),
                               workspace.numel() * workspace.element_size(), _ptr(topk_idx), _ptr(gates),
                               _stream(stream)), "mhlmoe_forward")


def mhlmoe_backward(plan: Plan, x, W, d_out, saved, dx, grads, workspace, stream=None):
    ws = weights_struct(W) if isinstance(W, dict) else W
    gs = grads_struct(grads) if isinstance(grads, dict) else grads
    _check(_lib.mhlmoe_backward(plan.handle, _ptr(x), ctypes.byref(ws), _ptr(d_out), _ptr(saved), _ptr(dx),
                                ctypes.byref(gs), _ptr(workspace), workspace.numel() * workspace.element_size(),
                                _stream(stream)), "mhlmoe_backward")


def mhlmoe_train_step_host(plan: Plan, x_host, dout_host, W, out_host, dx_host, grads, io, saved, workspace,
                           stream=None):
    ws = weights_struct(W) if isinstance(W, dict) else W
    gs = grads_struct(grads) if isinstance(grads, dict) else grads
    _check(_lib.mhlmoe_train_step_host(plan.handle, _ptr(x_host), _ptr(dout_host), ctypes.byref(ws), _ptr(out_host),
                                       _ptr(dx_host), ctypes.byref(gs), _ptr(io), _ptr(saved), _ptr(workspace),
                                       workspace.numel() * workspace.element_size(), _stream(stream)),
           "mhlmoe_train_step_host")


def mhlmoe_train_step_host_pipelined(plan: Plan, x_host, dout_host, W, out_host, dx_host, grads, io, saved,
                                     workspace, stream=None):
    """As mhlmoe_train_step_host; host outputs are complete after mhl_host_drain + a stream sync."""
    ws = weights_struct(W) if isinstance(W, dict) else W
    gs = grads_struct(grads) if isinstance(grads, dict) else grads
    _check(_lib.mhlmoe_train_step_host_pipelined(plan.handle, _ptr(x_host), _ptr(dout_host), ctypes.byref(ws),
                                                 _ptr(out_host), _ptr(dx_host), ctypes.byref(gs), _ptr(io),
                                                 _ptr(saved), _ptr(workspace),
                                                 workspace.numel() * workspace.element_size(), _stream(stream)),
           "mhlmoe_train_step_host_pipelined")


def mhl_host_drain(plan: Plan, stream=None):
    _check(_lib.mhl_host_drain(plan.handle, _stream(stream)), "mhl_host_drain")


def mhlmoe_update_bias(plan: Plan, saved, bias, gamma: float, stream=None):
    """Aux-free load-balancing step on the router bias (in place, device fp32 [H_loc][N_e])."""
    _check(_lib.mhlmoe_update_bias(plan.handle, _ptr(saved), _ptr(bias), ctypes.c_float(gamma), _stream(stream)),
           "mhlmoe_update_bias")


def mhl_check_device_status(plan: Plan):
    _check(_lib.mhl_check_device_status(plan.handle), "mhl_check_device_status")


def mhl_launch_count(plan: Plan) -> int:
    return int(_lib.mhl_launch_count(plan.handle))


def mhl_a2a_bytes_posted(plan: Plan) -> int:
    return int(_lib.mhl_a2a_bytes_posted(plan.handle))


def mhl_set_step_timing(plan: Plan, enable: bool):
    _check(_lib.mhl_set_step_timing(plan.handle, int(bool(enable))), "mhl_set_step_timing")


def mhl_step_times(plan: Plan) -> dict:
    """{step name: (total ms, calls)} accumulated since the last call (CUDA events)."""
    names = ctypes.create_string_buffer(4096)
    ms = (ctypes.c_double * 64)()
    calls = (ctypes.c_int32 * 64)()
    n = _lib.mhl_step_times(plan.handle, names, 4096, ms, calls, 64)
    if n < 0:
        raise MhlError(1, "mhl_step_times", "NULL plan")
    keys = [k for k in names.value.decode().split(",") if k]
    return {k: (ms[i], calls[i]) for i, k in enumerate(keys)}


def mhl_dp_reduce(plan: Plan, dW_in, dW_out, workspace, stream=None):
    _check(_lib.mhl_dp_reduce(plan.handle, _ptr(dW_in), _ptr(dW_out), _ptr(workspace), workspace.numel(),
                              _stream(stream)), "mhl_dp_reduce")


def mhl_kernel_paths(plan: Plan, reset: bool = False) -> set:
    """Names (PATHS keys) of the kernel implementations launched since the plan was created or
    last reset."""
    bits = int(_lib.mhl_kernel_paths(plan.handle, int(bool(reset))))
    return {k for k, b in PATHS.items() if bits & b}


def mhl_status_string(s: int) -> str:
    return _lib.mhl_status_string(s).decode()


def mhl_last_error() -> str:
    return _lib.mhl_last_error().decode()


def library():
    """The loaded ctypes CDLL (for export checks)."""
    return _lib
