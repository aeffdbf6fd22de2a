"""Torch-memory convenience around the C ABI: owns the plan, the `saved` and
`workspace` buffers, and exposes forward/backward.  Marshalling only — the
computation is entirely in libmhlmoe.so (see mhlmoe.py)."""
from __future__ import annotations

import torch

from . import mhlmoe as C


def torch_dtype(dtype: str):
    return torch.bfloat16 if dtype == "bf16" else torch.float32


class MHLatentMoE:
    """One rank's view of the HP layer.

    cfg fields: T_loc, d, N_h, d_h, N_e, k, d_e, dtype ('bf16'|'fp32').
    With ``loopback=True`` the plan runs G virtual ranks on this device and every
    call takes the global batch ([G*T_loc, d]) and all N_h heads' weights.
    """

    def __init__(self, T_loc, d, N_h, d_h, N_e, k, d_e, dtype="bf16", world_size=1, rank=0, loopback=False,
                 simt=False, nccl_id=None, device="cuda", pair=False, routing_tokens=False, windowed=False,
                 det_dp=False, bwd_fused=False):
        flags = ((C.MHL_FLAG_LOOPBACK if loopback else 0) | (C.MHL_FLAG_SIMT if simt else 0)
                 | (C.MHL_FLAG_PAIR if pair else 0) | (C.MHL_FLAG_ROUTING_TOKENS if routing_tokens else 0)
                 | (C.MHL_FLAG_WINDOWED_COMBINE if windowed else 0) | (C.MHL_FLAG_DET_DP if det_dp else 0)
                 | (C.MHL_FLAG_BWD_FUSED if bwd_fused else 0))
        self.routing_tokens = routing_tokens
        self.cfg = C.make_config(T_loc, d, N_h, d_h, N_e, k, d_e, dtype, world_size, rank, flags)
        self.plan = C.hp_plan(self.cfg, nccl_id)
        self.info = self.plan.info
        self.dtype = dtype
        self.T_loc, self.d, self.N_h, self.d_h, self.N_e, self.k, self.d_e = T_loc, d, N_h, d_h, N_e, k, d_e
        self.G = world_size
        self.loopback = loopback
        self.device = device
        self.saved = torch.empty(max(1, self.info["saved_bytes"]), dtype=torch.uint8, device=device)
        self.workspace = torch.empty(max(1, self.info["workspace_bytes"]), dtype=torch.uint8, device=device)
        self.H_loc = N_h if loopback else N_h // world_size
        self.T_glob = T_loc * world_size
        self.T_call = self.T_glob if loopback else T_loc

    def alloc_grads(self):
        f32 = dict(dtype=torch.float32, device=self.device)
        D = self.N_h * self.d_h
        D_in = D * (2 if self.routing_tokens else 1)   # [2D, d] with separate routing sub-tokens
        return dict(dW_in=torch.empty(D_in, self.d, **f32), dW_out=torch.empty(self.d, D, **f32),
                    dW_r=torch.empty(self.H_loc, self.d_h, self.N_e, **f32),
                    dW1=torch.empty(self.H_loc, self.N_e, self.d_e, self.d_h, **f32),
                    dW2=torch.empty(self.H_loc, self.N_e, self.d_e, self.d_h, **f32))

    def forward(self, x, W, out=None, want_routing=False, stream=None):
        if out is None:
            out = torch.empty(self.T_call, self.d, dtype=torch_dtype(self.dtype), device=self.device)
        idx = gates = None
        if want_routing:
            idx = torch.empty(self.H_loc, self.T_glob, self.k, dtype=torch.int32, device=self.device)
            gates = torch.empty(self.H_loc, self.T_glob, self.k, dtype=torch.float32, device=self.device)
        C.mhlmoe_forward(self.plan, x, W, out, self.saved, self.workspace, idx, gates, stream)
        return out, idx, gates

    def backward(self, x, W, d_out, grads, dx=None, stream=None):
        if dx is None:
            dx = torch.empty(self.T_call, self.d, dtype=torch_dtype(self.dtype), device=self.device)
        C.mhlmoe_backward(self.plan, x, W, d_out, self.saved, dx, grads, self.workspace, stream)
        return dx

    def saved_xs(self):
        """The forward's sub-tokens as the GPU stored them: `saved` begins with Xs [T_glob][XW] E
        (the all-to-all #1 receive buffer, include/mhlmoe.h), XW = H_loc*d_h (x2 with routing
        sub-tokens).  Test access, G = 1 or one rank."""
        XW = self.H_loc * self.d_h * (2 if self.routing_tokens else 1)
        td = torch_dtype(self.dtype)
        n = self.T_glob * XW
        return self.saved[: n * torch.tensor([], dtype=td).element_size()].view(td).view(self.T_glob, XW)

    def check_status(self):
        C.mhl_check_device_status(self.plan)

    def launches(self):
        return C.mhl_launch_count(self.plan)

    def paths(self, reset=False):
        """Kernel implementations that ran (mhl_kernel_paths)."""
        return C.mhl_kernel_paths(self.plan, reset)


def weights_to_device(W: dict, dtype: str, device="cuda", heads=None) -> dict:
    """numpy weights (float32 arrays, bf16-exact for bf16) -> device tensors in the ABI dtypes.
    ``heads`` = (begin, end) slices the per-head tensors to a rank's local heads."""
    td = torch_dtype(dtype)
    out = {}
    for n, a in W.items():
        t = torch.from_numpy(a)
        if heads is not None and n in ("W_r", "b", "W1", "W2"):
            t = t[heads[0]:heads[1]]
        out[n] = t.to(device=device, dtype=(torch.float32 if n in ("W_r", "b") else td)).contiguous()
    return out
