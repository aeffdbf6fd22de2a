"""bench.py host logic on CPU: the --gpus N launch path (re-exec under torch.distributed.run, one
process per GPU; rank 0 alone prints the line) through the reference arm, which needs no GPU, and
the algorithmic-work model's units."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from workloads import PRESETS  # noqa: E402


def test_gpus_2_reexecs_under_torchrun_and_rank0_prints_one_line():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "2", "--warmup", "3", "--config", "tiny", "--cpu-sample", "16"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 2
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert "2 steps" in d["cpu_baseline"]["sample"]


def test_torchrun_argv_is_the_driver_launch_form():
    a = bench.torchrun_argv(["--gpus", "8", "--steps", "5"], 8)
    assert a[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=8" in a and "127.0.0.1" in a
    assert a[-4:] == ["--gpus", "8", "--steps", "5"]


def test_expert_spans_are_tensor_bound_and_intermediates_are_not_algorithmic():
    cfg = PRESETS["paper"]
    w = bench.step_work(cfg, cfg.T, 1)
    unit = 2 * cfg.T * cfg.N_h * cfg.k * cfg.d_h * cfg.d_e           # 275 GFLOP at paper scale
    assert w["F5_expert_fwd"]["flops"] == 2 * unit
    assert w["B5_expert_bwd_dx"]["flops"] + w["B5_expert_dx_gemm"]["flops"] + w["B5_expert_bwd_dw"]["flops"] == 5 * unit
    for k in ("F5_expert_fwd", "B5_expert_bwd_dx", "B5_expert_dx_gemm", "B5_expert_bwd_dw"):
        bound = bench.span_roofline(w[k], 1e-3, 1631.7, 6549.1)[0]
        assert bound == "tensor", k
        assert w[k]["impl_bytes"] > w[k]["bytes"]          # Yrep / dH / gA / dXrep counted apart
    # §8(d): expert_bwd 1.37 TFLOP implemented
    assert abs(5 * unit / 1e12 - 1.374) < 0.01


def test_expert_data_movement_bytes_and_fused_accounting():
    """`sm_bytes` (L2 <-> SM bytes of each expert kernel, the ring probe's unit): per replica row F5
    moves X in and Yrep out, K1 X and dY in and dH, gA out, K2 dH in and dXrep out, dW X, dY, dH, gA
    in; the fused input side replaces K1 + K2 (3 units, no dH re-read) and B6 gains the router
    term's inputs."""
    cfg = PRESETS["paper"]
    rep = cfg.T * cfg.N_h * cfg.k
    row, erow = cfg.d_h * 2, cfg.d_e * 2
    w = bench.step_work(cfg, cfg.T, 1)
    assert w["F5_expert_fwd"]["sm_bytes"] == 2 * rep * row
    assert w["B5_expert_bwd_dx"]["sm_bytes"] == 2 * rep * (row + erow)
    assert w["B5_expert_dx_gemm"]["sm_bytes"] == rep * (row + erow)
    assert w["B5_expert_bwd_dw"]["sm_bytes"] == 2 * rep * (row + erow)
    total = sum(w[k]["sm_bytes"] for k in ("F5_expert_fwd", "B5_expert_bwd_dx", "B5_expert_dx_gemm", "B5_expert_bwd_dw"))
    assert abs(total / 1e9 - 20.4) < 0.1                       # 608 KB per 128-row tile
    f = bench.step_work(cfg, cfg.T, 1, fused_bwd=True)
    assert "B5_expert_dx_gemm" not in f
    unit = 2 * rep * cfg.d_h * cfg.d_e
    assert f["B5_expert_bwd_dx"]["flops"] == 3 * unit
    assert f["B5_expert_bwd_dx"]["sm_bytes"] == 3 * rep * row + 2 * rep * erow
    assert f["B6_combine_bwd"]["bytes"] > w["B6_combine_bwd"]["bytes"]
    probe = bench.load_probe_ceiling()
    assert probe is not None and 5.0 < probe["gather_store_TBps"] < 10.0
