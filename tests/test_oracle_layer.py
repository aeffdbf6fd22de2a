"""Pins for the oracle's layer forward/backward and Head Parallel emulation.

* Special cases that reduce to textbook forms: N_h = 1 is LatentMoE routed on x
  with the composed router (P:529, P:319-P:321); W_in = W_out = I, N_h = 1 is the
  plain Mixtral MoE of Eq. 1-4 (P:501-P:511).
* Invariants: per-head decomposition and head independence (Eq. 6, "sharing no
  parameters"); FLOP parity; HP bitwise equal to the unsharded
  layer, HP bytes constant in k, equal per rank, zero at P = 1 (P:810-P:813);
  HP/EP volume = 25% at k = 4 (printed).
* Backward: fp64 central finite differences along random directions for every
  parameter group and x (catches a dropped term, wrong sign or transposed operand).
"""
import os

import numpy as np
import pytest

import oracle as O
from workloads import LayerConfig, make_problem

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _prob(cfg, seed=0, dist="conf", T=None):
    W, x, dout = make_problem(cfg, seed, dist, T)
    P = {k: v.astype(np.float64) for k, v in W.items()}
    return P, x.astype(np.float64), dout.astype(np.float64)


TINY64 = LayerConfig("t", T=48, d=12, N_h=3, d_h=4, N_e=5, k=2, d_e=3, dtype="fp32")


# ---------------------------------------------------------------- textbook reductions
def _mixtral_moe_token(x_t, Wr, b, W1, W2, k):
    """Eq. 1-4 for one token, written independently: s = r(x), top-k over s+b,
    g = exp(s_sel)/sum exp(s_sel), o = sum_j g_j E_j(x)."""
    s = x_t @ Wr
    keyed = sorted(range(len(s)), key=lambda e: (-(s[e] + b[e]), e))[:k]
    ex = np.exp(np.array([s[e] for e in keyed]) - max(s[e] for e in keyed))
    g = ex / ex.sum()
    o = np.zeros(W2.shape[2])
    for gj, e in zip(g, keyed):
        o += gj * (O.gelu(W1[e] @ x_t) @ W2[e])
    return o


def test_identity_projections_single_head_is_textbook_moe():
    cfg = LayerConfig("m", T=20, d=6, N_h=1, d_h=6, N_e=5, k=2, d_e=4, dtype="fp32")
    P, x, _ = _prob(cfg, 1)
    P["W_in"] = np.eye(6); P["W_out"] = np.eye(6)
    out = O.layer_forward(P, x, cfg.k, mode="fp64").out
    ref = np.stack([_mixtral_moe_token(x[t], P["W_r"][0], P["b"][0], P["W1"][0], P["W2"][0], 2) for t in range(20)])
    np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-13)


def test_single_head_is_latentmoe_with_composed_router():
    """LatentMoE: route on x with R (d x N_e), then down-project W_down,
    experts, up-project W_up.  N_h = 1 MH-LatentMoE == LatentMoE with
    R = W_in^T W_r[0], W_down = W_in, W_up = W_out (selection identical where
    margins are not tiny)."""
    cfg = LayerConfig("l", T=40, d=10, N_h=1, d_h=6, N_e=7, k=3, d_e=4, dtype="fp32")
    P, x, _ = _prob(cfg, 2)
    C = O.layer_forward(P, x, cfg.k, mode="fp64")
    R = P["W_in"].T @ P["W_r"][0]                        # [d, N_e], composed router
    for t in range(cfg.T):
        if C.margin[0][t] < 1e-9:
            continue
        s = x[t] @ R
        sel = sorted(range(cfg.N_e), key=lambda e: (-(s[e] + P["b"][0][e]), e))[:cfg.k]
        g = np.exp(s[sel] - s[sel].max()); g /= g.sum()
        z = P["W_in"] @ x[t]                               # down-projection
        y = sum(gj * (O.gelu(P["W1"][0][e] @ z) @ P["W2"][0][e]) for gj, e in zip(g, sel))
        np.testing.assert_allclose(C.out[t], P["W_out"] @ y, rtol=1e-11, atol=1e-12)


# ---------------------------------------------------------------- multi-head invariants
def test_per_head_decomposition_and_head_independence():
    P, x, _ = _prob(TINY64, 3)
    C = O.layer_forward(P, x, TINY64.k, mode="fp64")
    d_h = TINY64.d_h
    ys = []
    for h in range(TINY64.N_h):
        Ph = dict(W_in=P["W_in"][h * d_h:(h + 1) * d_h], W_out=np.eye(d_h), W_r=P["W_r"][h:h + 1],
                  b=P["b"][h:h + 1], W1=P["W1"][h:h + 1], W2=P["W2"][h:h + 1])
        ys.append(O.layer_forward(Ph, x, TINY64.k, mode="fp64").out)
    np.testing.assert_array_equal(np.concatenate(ys, 1), C.cat)
    # perturbing head 1's experts leaves heads 0 and 2 bitwise unchanged
    P2 = {k: v.copy() for k, v in P.items()}
    P2["W1"][1] += 0.5
    C2 = O.layer_forward(P2, x, TINY64.k, mode="fp64")
    for h in (0, 2):
        np.testing.assert_array_equal(C2.cat[:, h * d_h:(h + 1) * d_h], C.cat[:, h * d_h:(h + 1) * d_h])
    assert not np.array_equal(C2.cat[:, d_h:2 * d_h], C.cat[:, d_h:2 * d_h])


def _counted_scalar_forward(P, x, k):
    """An independent scalar-loop forward of the layer (Eq. 1-6, fp64, no storage rounding) that
    counts every multiply-add it performs: the pin of layer_flops / moe_flops_equivalent."""
    import math
    N_h, d_h, N_e = P["W_r"].shape
    d_e = P["W1"].shape[2]
    T, d = x.shape
    D = N_h * d_h
    macs = dict(w_in=0, router=0, experts=0, w_out=0)
    out = np.zeros((T, P["W_out"].shape[0]))
    for t in range(T):
        xs = [sum(P["W_in"][i][c] * x[t][c] for c in range(d)) for i in range(D)]
        macs["w_in"] += D * d
        cat = []
        for h in range(N_h):
            sub = xs[h * d_h:(h + 1) * d_h]
            s = [sum(sub[i] * P["W_r"][h][i][e] for i in range(d_h)) for e in range(N_e)]
            macs["router"] += d_h * N_e
            order = sorted(range(N_e), key=lambda e: (-(s[e] + P["b"][h][e]), e))[:k]
            m = max(s[e] for e in order)
            z = sum(math.exp(s[e] - m) for e in order)
            y = [0.0] * d_h
            for e in order:
                g = math.exp(s[e] - m) / z
                hid = [sum(sub[i] * P["W1"][h][e][j][i] for i in range(d_h)) for j in range(d_e)]
                a = [v * 0.5 * (1.0 + math.erf(v / math.sqrt(2.0))) for v in hid]
                for c in range(d_h):
                    y[c] += g * sum(a[j] * P["W2"][h][e][j][c] for j in range(d_e))
                macs["experts"] += 2 * d_h * d_e
            cat.extend(y)
        for o in range(out.shape[1]):
            out[t][o] = sum(cat[c] * P["W_out"][o][c] for c in range(D))
        macs["w_out"] += out.shape[1] * D
    return out, macs


def test_flop_parity_p777():
    """layer_flops / moe_flops_equivalent against the multiply-adds an independent scalar-loop forward
    actually performs (its output checked against the oracle's), and P:777's parity: router +
    experts of the layer = one MoE over N_h*T sub-tokens."""
    cfg = TINY64.replace(T=6, d=16, N_h=2, d_h=8, N_e=6, k=2, d_e=5, dtype="fp64")
    P, x, _ = _prob(cfg, 9)
    out, macs = _counted_scalar_forward(P, x, cfg.k)
    C = O.layer_forward(P, x, cfg.k, mode="fp64")
    np.testing.assert_allclose(out, C.out, rtol=1e-10, atol=1e-12)
    f = O.layer_flops(cfg.T, cfg.d, cfg.N_h, cfg.d_h, cfg.N_e, cfg.k, cfg.d_e)
    assert f == {kk: 2 * v for kk, v in macs.items()}
    assert f["router"] + f["experts"] == O.moe_flops_equivalent(cfg.T, cfg.N_h, cfg.d_h, cfg.N_e, cfg.k, cfg.d_e)


def test_bf16_rounding_points():
    cfg = TINY64.replace(dtype="bf16")
    P, x, _ = _prob(cfg, 4)
    C = O.layer_forward(P, x, cfg.k, mode="bf16")
    for arr in (C.Xs, C.cat, C.out):
        np.testing.assert_array_equal(arr, O.round_storage(arr, "bf16"))
    C64 = O.layer_forward(P, x, cfg.k, mode="fp64")
    assert not np.array_equal(C64.Xs, C.Xs)


# ---------------------------------------------------------------- backward: finite differences
def _loss(P, x, dout, k, forced):
    return float(np.sum(O.layer_forward(P, x, k, mode="fp64", forced_idx=forced).out * dout))


@pytest.mark.parametrize("seed", [0, 1])
def test_backward_directional_finite_differences(seed):
    cfg = LayerConfig("fd", T=16, d=8, N_h=2, d_h=4, N_e=5, k=2, d_e=3, dtype="fp32")
    P, x, dout = _prob(cfg, 10 + seed)
    C = O.layer_forward(P, x, cfg.k, mode="fp64")
    forced = {h: C.I[h] for h in range(cfg.N_h)}   # hold the (piecewise-constant) selection fixed (R13)
    grads = O.layer_backward(P, x, dout, C)
    rng = np.random.default_rng(seed)
    eps = 1e-6
    for name, gname in [("W_in", "dW_in"), ("W_out", "dW_out"), ("W_r", "dW_r"), ("W1", "dW1"), ("W2", "dW2"), ("x", "dx")]:
        for _ in range(3):
            v = rng.standard_normal(x.shape if name == "x" else P[name].shape)
            def f(s):
                Pp = dict(P)
                xx = x
                if name == "x":
                    xx = x + s * v
                else:
                    Pp[name] = P[name] + s * v
                return _loss(Pp, xx, dout, cfg.k, forced)
            fd = (f(eps) - f(-eps)) / (2 * eps)
            an = float(np.sum(grads[gname] * v))
            assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)), (name, fd, an)
    # selections must be stable under the perturbation for the forced-idx FD to be the true derivative
    assert min(float(np.min(m)) for m in C.margin) > 1e-5


def test_backward_structural_zeros():
    cfg = LayerConfig("z", T=12, d=8, N_h=2, d_h=4, N_e=9, k=2, d_e=3, dtype="fp32")
    P, x, dout = _prob(cfg, 20)
    C = O.layer_forward(P, x, cfg.k, mode="fp64")
    g = O.layer_backward(P, x, dout, C)
    for h in range(cfg.N_h):
        used = set(C.I[h].reshape(-1).tolist())
        for e in range(cfg.N_e):
            if e not in used:
                assert np.all(g["dW_r"][h][:, e] == 0)          # unselected router columns exactly 0
                assert np.all(g["dW1"][h, e] == 0) and np.all(g["dW2"][h, e] == 0)
    z = O.layer_backward(P, x, np.zeros_like(dout), C)
    for key in ("dx", "dW_in", "dW_out", "dW_r", "dW1", "dW2"):
        assert np.all(z[key] == 0)


# ---------------------------------------------------------------- Head Parallel (P:796-P:813)
@pytest.mark.parametrize("G", [1, 2, 4])
def test_hp_forward_bitwise_equals_unsharded(G):
    cfg = LayerConfig("hp", T=64, d=16, N_h=4, d_h=4, N_e=6, k=2, d_e=3, dtype="bf16")
    P, x, _ = _prob(cfg, 30)
    ref = O.layer_forward(P, x, cfg.k, mode="bf16").out
    out, _ranks, nbytes = O.hp_layer_forward(P, x, cfg.k, G, mode="bf16")
    np.testing.assert_array_equal(out, ref)
    T_loc = cfg.T // G
    per_pair = T_loc * (cfg.N_h // G) * cfg.d_h * 2
    expect = 2 * per_pair * (G - 1)                       # two forward all-to-alls
    assert np.all(nbytes.sum(1) == expect) and np.all(nbytes.sum(0) == expect)
    np.testing.assert_array_equal(nbytes, 2 * O.hp_a2a_bytes(T_loc, cfg.N_h, cfg.d_h, G, 2))
    if G == 1:
        assert nbytes.sum() == 0


def test_hp_bytes_constant_in_k_and_routing():
    cfg = LayerConfig("hp", T=32, d=8, N_h=4, d_h=2, N_e=16, k=2, d_e=2, dtype="bf16")
    seen = set()
    for k in (2, 4, 8, 16):
        for seed in range(3):
            P, x, _ = _prob(cfg.replace(k=k), seed)
            _o, _r, nb = O.hp_layer_forward(P, x, k, 4, mode="bf16")
            seen.add(nb.tobytes())
            assert nb.max(initial=0) == nb[~np.eye(4, dtype=bool)].min()   # max = min over pairs
    assert len(seen) == 1


def test_hp_backward_equals_unsharded():
    cfg = LayerConfig("hpb", T=32, d=8, N_h=4, d_h=2, N_e=5, k=2, d_e=3, dtype="bf16")
    P, x, dout = _prob(cfg, 40)
    C = O.layer_forward(P, x, cfg.k, mode="bf16")
    ref = O.layer_backward(P, x, dout, C)
    for G in (2, 4):
        hp = O.hp_layer_backward(P, x, dout, cfg.k, G, mode="bf16")
        np.testing.assert_array_equal(hp["dx"], ref["dx"])
        for key in ("dW_r", "dW1", "dW2"):
            np.testing.assert_allclose(hp[key], ref[key], rtol=1e-12, atol=1e-14)
        for key in ("dW_in", "dW_out"):                   # rank-partial sums (R19)
            np.testing.assert_allclose(hp[key], ref[key], rtol=1e-12, atol=1e-14)
        np.testing.assert_array_equal(hp["bytes_bwd"], hp["bytes_fwd"])


def test_hp_volume_vs_ep_printed_25pct():
    rows = {l.split()[0]: float(l.split()[1]) for l in open(os.path.join(GOLDEN, "paper_printed.txt"))
            if l.strip() and not l.startswith("#")}
    T, N_h, d_h, G = 4096, 8, 128, 4
    hp = O.hp_a2a_bytes(T // G, N_h, d_h, G, 2).sum()
    # EP with the same sub-token rows, each dispatched k times (G-1)/G of them cross GPUs
    ep = O.ep_dispatch_rows(T * N_h, 4) * d_h * 2 * (G - 1) // G
    assert hp / ep == rows["hp_over_ep_volume_k4"]


def test_hp_rejects_bad_degree():
    P, x, _ = _prob(TINY64, 0)
    with pytest.raises(ValueError):
        O.hp_layer_forward(P, x, 2, 2, mode="fp32")    # N_h = 3 not divisible by 2


# ---------------------------------------------------------------- separate routing sub-tokens (P:1565-P:1570)
RT = LayerConfig("rt", T=40, d=10, N_h=2, d_h=4, N_e=6, k=2, d_e=3, dtype="fp32", routing_tokens=True)


def test_routing_tokens_with_duplicated_rows_is_the_base_layer():
    """W_in = [W; W] makes r_t = x_t: forward, routing and every gradient reduce to the base layer
    (dW_in's two halves summing to the base dW_in), in fp64 storage mode."""
    cfg = RT.replace(routing_tokens=False)
    P, x, dout = _prob(cfg, 50)
    P2 = dict(P, W_in=np.concatenate([P["W_in"], P["W_in"]], axis=0))
    C = O.layer_forward(P, x, cfg.k, mode="fp64")
    C2 = O.layer_forward(P2, x, cfg.k, mode="fp64")
    for h in range(cfg.N_h):
        np.testing.assert_array_equal(C2.I[h], C.I[h])
    np.testing.assert_allclose(C2.out, C.out, rtol=1e-12, atol=1e-14)
    g = O.layer_backward(P, x, dout, C)
    g2 = O.layer_backward(P2, x, dout, C2)
    D = cfg.D
    np.testing.assert_allclose(g2["dW_in"][:D] + g2["dW_in"][D:], g["dW_in"], rtol=1e-12, atol=1e-13)
    for key in ("dx", "dW_out", "dW_r", "dW1", "dW2"):
        np.testing.assert_allclose(g2[key], g[key], rtol=1e-12, atol=1e-13)
    assert g2["dW_in"].shape == (2 * D, cfg.d)


def test_routing_tokens_route_on_r_and_compute_on_x():
    """The selection depends only on the routing rows of W_in, the expert output only (given the
    selection) on the sub-token rows: perturbing the sub-token half leaves every I unchanged, and
    perturbing the routing half leaves the selected experts' inputs unchanged."""
    P, x, _ = _prob(RT, 51)
    D = RT.D
    C = O.layer_forward(P, x, RT.k, mode="fp64")
    Px = dict(P, W_in=P["W_in"].copy())
    Px["W_in"][:D] *= 1.7
    Cx = O.layer_forward(Px, x, RT.k, mode="fp64")
    for h in range(RT.N_h):
        np.testing.assert_array_equal(Cx.I[h], C.I[h])
    assert not np.allclose(Cx.out, C.out)
    Pr = dict(P, W_in=P["W_in"].copy())
    Pr["W_in"][D:] = np.random.default_rng(3).standard_normal(Pr["W_in"][D:].shape)
    Cr = O.layer_forward(Pr, x, RT.k, mode="fp64")
    assert any(not np.array_equal(Cr.I[h], C.I[h]) for h in range(RT.N_h))
    np.testing.assert_array_equal(Cr.Xs[:, :D], C.Xs[:, :D])


@pytest.mark.parametrize("seed", [52, 53])
def test_routing_tokens_backward_finite_differences(seed):
    P, x, dout = _prob(RT, seed)
    C = O.layer_forward(P, x, RT.k, mode="fp64")
    forced = {h: C.I[h] for h in range(RT.N_h)}
    grads = O.layer_backward(P, x, dout, C)
    rng = np.random.default_rng(seed)
    eps = 1e-6
    for name, gname in [("W_in", "dW_in"), ("W_r", "dW_r"), ("W1", "dW1"), ("x", "dx")]:
        for _ in range(3):
            v = rng.standard_normal(x.shape if name == "x" else P[name].shape)
            def f(s):
                Pp = dict(P)
                xx = x
                if name == "x":
                    xx = x + s * v
                else:
                    Pp[name] = P[name] + s * v
                return _loss(Pp, xx, dout, RT.k, forced)
            fd = (f(eps) - f(-eps)) / (2 * eps)
            an = float(np.sum(grads[gname] * v))
            assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)), (name, fd, an)
    # the routing half of dW_in is the router's alone: zero when every dS vanishes (dout = 0 on gates)
    assert np.any(grads["dW_in"][RT.D:] != 0)
    assert min(float(np.min(m)) for m in C.margin) > 1e-5


@pytest.mark.parametrize("G", [1, 2])
def test_routing_tokens_hp_equals_unsharded_and_doubles_scatter_bytes(G):
    cfg = RT.replace(T=48, N_h=2, dtype="bf16")
    P, x, dout = _prob(cfg, 54)
    C = O.layer_forward(P, x, cfg.k, mode="bf16")
    ref = O.layer_backward(P, x, dout, C)
    hp = O.hp_layer_backward(P, x, dout, cfg.k, G, mode="bf16")
    np.testing.assert_array_equal(hp["out"], C.out)
    np.testing.assert_array_equal(hp["dx"], ref["dx"])
    for key in ("dW_in", "dW_out", "dW_r", "dW1", "dW2"):
        np.testing.assert_allclose(hp[key], ref[key], rtol=1e-12, atol=1e-14)
    per_pair = (cfg.T // G) * (cfg.N_h // G) * cfg.d_h * 2
    # forward: the scatter carries x and r (2 blocks), the gather the head outputs (1 block)
    assert np.all(hp["bytes_fwd"][~np.eye(G, dtype=bool)] == 3 * per_pair)
    assert np.all(hp["bytes_bwd"] == hp["bytes_fwd"])
