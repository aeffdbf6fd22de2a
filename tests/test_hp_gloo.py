"""Multi-process (world_size 2, gloo, CPU) tests of the Head Parallel host logic.

Each rank queries its plan from the C library (pure host: hp_plan_query), the ranks
exchange the plans over torch.distributed and check that heads are partitioned in
contiguous blocks (R12) and that every rank sends/receives the same, k-independent byte
count (P:811-P:812).  Then the HP data movement is run for real over gloo: each rank
projects its own tokens with the oracle, all-to-alls the sub-token blocks using the split
sizes from its plan, runs its local heads, all-to-alls the head outputs back and projects
(Eq. 5-6); the result must equal the unsharded oracle bitwise (HP only moves data).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from paper_2602_04870_b200 import mhlmoe as C
        from workloads import LayerConfig, make_problem

        cfg = LayerConfig("gloo", T=64, d=32, N_h=4, d_h=8, N_e=6, k=2, d_e=8, dtype="bf16")
        T_loc = cfg.T // world
        # ---- plans from the library, gathered
        infos = {}
        for k in (1, 2, 4, 6):
            info = C.hp_plan_query(C.make_config(T_loc, cfg.d, cfg.N_h, cfg.d_h, cfg.N_e, k, cfg.d_e, "bf16",
                                                 world, rank))
            infos[k] = info
        mine = [infos[2]["head_begin"], infos[2]["head_end"], infos[2]["a2a_bytes_per_rank"]]
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        assert [p[:2] for p in allp] == [[r * cfg.N_h // world, (r + 1) * cfg.N_h // world] for r in range(world)]
        assert len({p[2] for p in allp}) == 1
        assert len({infos[k]["a2a_bytes_per_rank"] for k in infos}) == 1
        # ---- HP data movement over gloo with the oracle's per-rank arithmetic
        W, x, _ = make_problem(cfg, 3, "conf")
        P = {kk: v.astype(np.float64) for kk, v in W.items()}
        H_loc, d_h = cfg.N_h // world, cfg.d_h
        hb, he = infos[2]["head_begin"], infos[2]["head_end"]
        x_r = x[rank * T_loc:(rank + 1) * T_loc].astype(np.float64)
        Xs_r = O.round_storage(x_r @ P["W_in"].T, "bf16")                       # Eq. 5 on my tokens
        send = torch.from_numpy(np.ascontiguousarray(
            np.stack([Xs_r[:, p * H_loc * d_h:(p + 1) * H_loc * d_h] for p in range(world)])))
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send)                                       # a2a #1
        # bytes one rank sends to each peer in bf16 storage = the plan's closed form
        assert (send.numel() // world) * 2 == infos[2]["a2a_bytes_per_peer"]
        Xh = recv.numpy().reshape(world * T_loc, H_loc * d_h)                    # all tokens, my heads
        ys = []
        for hl in range(H_loc):
            h = hb + hl
            X_h = Xh[:, hl * d_h:(hl + 1) * d_h]
            I, S_sel, *_ = O.route_topk(X_h, P["W_r"][h], P["b"][h], cfg.k)
            ys.append(O.experts_dense(X_h, P["W1"][h], P["W2"][h], I, O.gates_from_scores(S_sel)))
        y = O.round_storage(np.concatenate(ys, 1), "bf16")
        send2 = torch.from_numpy(np.ascontiguousarray(y.reshape(world, T_loc, H_loc * d_h)))
        recv2 = torch.empty_like(send2)
        dist.all_to_all_single(recv2, send2)                                     # a2a #2
        cat_r = np.concatenate([recv2.numpy()[p] for p in range(world)], 1)
        out_r = O.round_storage(cat_r @ P["W_out"].T, "bf16")                    # Eq. 6
        ref = O.layer_forward(P, x.astype(np.float64), cfg.k, mode="bf16").out[rank * T_loc:(rank + 1) * T_loc]
        assert np.array_equal(out_r, ref)
        assert he - hb == H_loc
        result_q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        result_q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_hp_two_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_bench_reference_arm_json():
    """bench.py --impl reference prints one valid JSON line (oracle on a bounded sample)."""
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "tiny",
                          "--cpu-sample", "32", "--steps", "1"], capture_output=True, text=True, timeout=600)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"


def _sched_worker(rank, world, port, result_q):
    """The pipelined exchange schedule of hp_exchange (capi.cpp): at step i rank r sends the block
    addressed to q = (r+i) mod G and receives the block of src = (r-i) mod G.  Over gloo it must
    deliver exactly what an all-to-all delivers (block s of rank r = rank s's block for r), and
    the block sizes come from the plan (x2 for the scatter with separate routing sub-tokens).
    A step's send and receive are posted together (NCCL group there, isend + recv here)."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_04870_b200 import mhlmoe as C
        ok = True
        for flags in (0, C.MHL_FLAG_ROUTING_TOKENS):
            cfg = C.make_config(64, 32, 4, 8, 8, 2, 8, "bf16", world, rank, flags)
            info = C.hp_plan_query(cfg)
            n = info["a2a_bytes_per_peer"] // 2                     # bf16 elements per block
            base = 64 * 8 * (4 // world)                            # T_loc * H_loc * d_h
            ok &= n == (2 if flags else 1) * base
            send = [torch.full((n,), float(100 * rank + q)) for q in range(world)]
            recv = [torch.empty(n) for _ in range(world)]
            recv[rank].copy_(send[rank])                            # step 0: the self block
            for i in range(1, world):                               # one grouped send/recv pair per step
                q, src = (rank + i) % world, (rank - i) % world
                w = dist.isend(send[q], q)
                dist.recv(recv[src], src)
                w.wait()
            ok &= all(torch.equal(recv[s], torch.full((n,), float(100 * s + rank))) for s in range(world))
        result_q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_pipelined_exchange_schedule_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sched_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res
