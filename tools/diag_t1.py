"""Diagnostic (under gpurun): per-row error of dW_in vs the oracle at tiny T, showing the worst row is
the one whose dXs cancels (bf16 replica rows), while the tensor-wide error stays ~3e-3."""
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import torch
import oracle as O
from workloads import LayerConfig, make_problem
from test_gpu_parity import _run_gpu
from parity_util import check_routing
for T in (1, 2, 8, 64):
    cfg = LayerConfig("edge", T=T, d=256, N_h=2, d_h=128, N_e=64, k=8, d_e=64, dtype="bf16")
    W, x, dout = make_problem(cfg, 60 + T, "exact")
    g = _run_gpu(cfg, W, x, dout)
    P = {k: v.astype(np.float64) for k, v in W.items()}
    xs = x.astype(np.float64)
    C0 = O.layer_forward(P, xs, cfg.k, mode="bf16")
    rt = check_routing(P, C0, g["idx"], cfg.k, x=xs, exact=True)
    C = O.layer_forward(P, xs, cfg.k, mode="bf16", forced_idx=rt.forced)
    gr = O.layer_backward(P, xs, dout.astype(np.float64), C)
    # dXs from the GPU: recover from dx? use dW_in rows / x  (T=1: row i = dXs_i * x)
    ref = gr["dW_in"]; gp = g["dW_in"]
    row_err = np.max(np.abs(gp - ref), 1) / np.maximum(np.max(np.abs(ref), 1), 1e-30)
    worst = int(np.argmax(row_err))
    glob = np.max(np.abs(gp - ref)) / np.max(np.abs(ref))
    print(f"T={T}: dW_in worst row {worst} rel {row_err[worst]:.3e}  |ref row max| {np.max(np.abs(ref[worst])):.3e} vs tensor max {np.max(np.abs(ref)):.3e}; global rel {glob:.3e}; dXs_ref[:,worst] {gr['dXs'][:, worst][:4]}")
