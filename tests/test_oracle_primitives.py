"""Pins for the oracle's primitives: rounding, GELU, softmax/gates, routing, clustering.

Each test checks the oracle against something other than itself: textbook
values (tests/golden/), a library routine on a special case, an independent
algorithm from the paper (Alg. 1's online merge vs the full sort), brute force
over all k-subsets, or an invariant the paper states.
"""
import itertools
import math
import os

import numpy as np
import pytest
import torch

import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- rounding (R9)
def test_round_bf16_matches_torch_on_fp32_values():
    rng = np.random.default_rng(0)
    a = (rng.standard_normal(200000) * np.exp(rng.uniform(-20, 20, 200000))).astype(np.float32)
    ref = torch.from_numpy(a).to(torch.bfloat16).to(torch.float64).numpy()
    got = O.round_storage(a.astype(np.float64), "bf16")
    assert np.array_equal(got, ref)


def test_round_bf16_ties_to_even():
    # bf16 has 8 significant bits: neighbours of 1 are 1 and 1 + 2^-7
    assert O.round_storage(np.array([1 + 2.0 ** -8]), "bf16")[0] == 1.0
    assert O.round_storage(np.array([1 + 3 * 2.0 ** -8]), "bf16")[0] == 1 + 2.0 ** -6
    assert O.round_storage(np.array([1 + 2.0 ** -8 + 2.0 ** -30]), "bf16")[0] == 1 + 2.0 ** -7
    assert O.round_storage(np.array([-(1 + 2.0 ** -8)]), "bf16")[0] == -1.0


def test_round_fp32_and_fp64():
    a = np.array([1 / 3, math.pi, -1e-3])
    assert np.array_equal(O.round_storage(a, "fp32"), a.astype(np.float32).astype(np.float64))
    assert np.array_equal(O.round_storage(a, "fp64"), a)


# ---------------------------------------------------------------- GELU (R1)
def test_gelu_textbook_phi_values():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "gelu_phi_values.txt")) if l.strip() and not l.startswith("#")]
    x = np.array([float(r[0]) for r in rows])
    phi = np.array([float(r[1]) for r in rows])
    np.testing.assert_allclose(O.gelu(x), x * phi, rtol=1e-14, atol=1e-16)


def test_gelu_properties():
    assert O.gelu(np.array([0.0]))[0] == 0.0
    assert abs(O.gelu(np.array([10.0]))[0] - 10.0) < 1e-6
    xs = np.arange(-10, 10, 1e-4)
    g = O.gelu(xs)
    assert g.min() >= -0.17 and g.min() < -0.169      # exact-erf GELU minimum ~ -0.16997
    assert np.all(g + 1.0 > 0)                         # needed by Eq. 8's log
    # tanh-approximate GELU differs measurably: the oracle is NOT the tanh form (R1)
    tanh_form = 0.5 * xs * (1 + np.tanh(math.sqrt(2 / math.pi) * (xs + 0.044715 * xs ** 3)))
    assert np.max(np.abs(tanh_form - g)) > 1e-4


def test_gelu_grad_against_central_differences():
    xs = np.linspace(-6, 6, 1201)
    eps = 1e-6
    fd = (O.gelu(xs + eps) - O.gelu(xs - eps)) / (2 * eps)
    np.testing.assert_allclose(O.gelu_grad(xs), fd, atol=1e-8)
    assert O.gelu_grad(np.array([0.0]))[0] == 0.5


def test_gelu_matches_torch_exact_gelu():
    xs = np.linspace(-8, 8, 4001)
    ref = torch.nn.functional.gelu(torch.from_numpy(xs), approximate="none").numpy()
    np.testing.assert_allclose(O.gelu(xs), ref, rtol=1e-14, atol=1e-15)


# ---------------------------------------------------------------- gates (Eq. 2-3)
def test_gates_sum_to_one_and_special_cases():
    rng = np.random.default_rng(1)
    S = rng.standard_normal((100, 5)) * 3
    g = O.gates_from_scores(S)
    np.testing.assert_allclose(g.sum(1), 1.0, atol=1e-15)
    assert np.all(O.gates_from_scores(rng.standard_normal((10, 1))) == 1.0)   # k = 1 -> exactly 1
    np.testing.assert_allclose(O.gates_from_scores(np.full((3, 4), 0.7)), 0.25, atol=1e-16)
    # softmax([-inf, 0]) = [0, 1]  (SPEC softmax example; Eq. 3 masking)
    np.testing.assert_array_equal(O.softmax_lastaxis(np.array([[-np.inf, 0.0]])), [[0.0, 1.0]])


def test_gates_equal_literal_eq2_masked_softmax():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((64, 16)); W = rng.standard_normal((16, 32)); b = rng.standard_normal(32)
    for k in (1, 2, 5, 32):
        I, S_sel, _m, S, _K = O.route_topk(X, W, b, k)
        np.testing.assert_allclose(O.gates_from_scores(S_sel), O.gates_eq2_masked(S, I), rtol=1e-14, atol=1e-300)


# ---------------------------------------------------------------- routing (Eq. 3, Alg. 1)
def test_route_topk_brute_force_subsets():
    """Top-k set = the unique k-subset maximising the sum of keys (continuous inputs,
    no ties); slot order = descending key."""
    rng = np.random.default_rng(3)
    N_e = 7
    X = rng.standard_normal((40, 6)); W = rng.standard_normal((6, N_e)); b = rng.standard_normal(N_e)
    for k in (1, 2, 3, 7):
        I, S_sel, margin, S, K = O.route_topk(X, W, b, k)
        for t in range(X.shape[0]):
            best = max(itertools.combinations(range(N_e), k), key=lambda c: sum(K[t, list(c)]))
            assert set(I[t].tolist()) == set(best)
            assert np.all(np.diff(K[t, I[t]]) <= 0)
            np.testing.assert_array_equal(S_sel[t], S[t, I[t]])
            # scores returned are the UNBIASED ones (P:837, P:885-P:886)
            np.testing.assert_allclose(S_sel[t], X[t] @ W[:, I[t]], rtol=1e-13, atol=1e-13)
        if k < N_e:
            srt = np.sort(K, axis=1)[:, ::-1]
            np.testing.assert_allclose(margin, srt[:, k - 1] - srt[:, k])
        else:
            assert np.all(np.isinf(margin))


def test_route_topk_ties_lower_index_and_degenerate():
    X = np.ones((3, 2)); W = np.zeros((2, 6)); b = np.zeros(6)
    I, *_ = O.route_topk(X, W, b, 4)
    np.testing.assert_array_equal(I, [[0, 1, 2, 3]] * 3)            # all tie -> lower index first
    # -0.0 and +0.0 tie (R6)
    b2 = np.array([0.0, -0.0, -1.0])
    I2, *_ = O.route_topk(np.ones((1, 1)), np.zeros((1, 3)), b2, 1)
    assert I2[0, 0] == 0
    # N_e == k returns all experts (SPEC degenerate case)
    rng = np.random.default_rng(4)
    X = rng.standard_normal((20, 4)); W = rng.standard_normal((4, 5)); b = rng.standard_normal(5)
    I3, *_ = O.route_topk(X, W, b, 5)
    assert all(sorted(r) == list(range(5)) for r in I3.tolist())


def test_route_bias_steers_selection_not_scores():
    rng = np.random.default_rng(5)
    X = rng.standard_normal((50, 8)); W = rng.standard_normal((8, 16)); b = np.zeros(16)
    b[7] = 1e3
    I, S_sel, *_ = O.route_topk(X, W, b, 3)
    assert np.all(I[:, 0] == 7)
    np.testing.assert_allclose(S_sel[:, 0], X @ W[:, 7], rtol=1e-14)
    # shift invariance: adding a constant to every key leaves the selection unchanged
    b3 = rng.standard_normal(16)
    Ia, *_ = O.route_topk(X, W, b3, 4)
    Ib, *_ = O.route_topk(X, W, b3 + 0.5, 4)
    np.testing.assert_array_equal(Ia, Ib)


def test_route_rejects_nonfinite():
    X = np.ones((2, 2)); W = np.ones((2, 3)); W[0, 1] = np.nan
    with pytest.raises(O.NonFiniteScore):
        O.route_topk(X, W, np.zeros(3), 1)


def test_pack_key_order_preserving():
    vals = np.array([-np.inf, -3.5, -1e-30, -0.0, 0.0, 1e-30, 2.0, np.inf], np.float32)
    o = O.ord32(vals)
    assert np.all(np.diff(o[[0, 1, 2, 4, 5, 6, 7]].astype(np.int64)) > 0)
    assert o[3] == o[4]                                         # -0.0 canonicalised
    keys = O.pack_key(np.array([1.0, 1.0, 2.0], np.float32), np.array([5, 3, 9]))
    assert keys[1] > keys[0] > 0                                 # tie -> lower index is the larger key
    v, i = O.unpack_key(keys)
    np.testing.assert_array_equal(v, [1.0, 1.0, 2.0]); np.testing.assert_array_equal(i, [5, 3, 9])
    # every real key is > 0 = Alg. 1's accumulator init (R17)
    assert O.pack_key(np.array([-np.inf], np.float32), np.array([0xFFFFFFFE]))[0] > 0


@pytest.mark.parametrize("M", [1, 2, 16, 64, 100])
def test_alg1_online_merge_equals_full_sort(M):
    """Alg. 1 (paper's online block top-k with packed keys) == full sort, for
    integer-valued scores (exact in fp32 and fp64, many ties)."""
    rng = np.random.default_rng(10 + M)
    N_e, k = 100, 6
    X = rng.integers(-3, 4, (300, 5)).astype(np.float64)
    W = rng.integers(-3, 4, (5, N_e)).astype(np.float64)
    b = rng.integers(-2, 3, N_e).astype(np.float64)
    I_ref, S_ref, *_ = O.route_topk(X, W, b, k)
    I, S_top = O.route_online_alg1(X, W, b, k, M)
    np.testing.assert_array_equal(I, I_ref)
    np.testing.assert_array_equal(S_top, S_ref)


# ---------------------------------------------------------------- experts (Eq. 1, Eq. 8)
def _expert_problem(seed, T=30, d_h=8, N_e=6, d_e=5, k=2):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((T, d_h)); W1 = rng.standard_normal((N_e, d_e, d_h)) / 3
    W2 = rng.standard_normal((N_e, d_e, d_h)) / 3; Wr = rng.standard_normal((d_h, N_e))
    I, S_sel, *_ = O.route_topk(X, Wr, np.zeros(N_e), k)
    return X, W1, W2, I, O.gates_from_scores(S_sel)


def test_experts_dense_equals_sparse_loop_and_flex_form():
    X, W1, W2, I, g = _expert_problem(20)
    y_dense = O.experts_dense(X, W1, W2, I, g)
    np.testing.assert_allclose(y_dense, O.experts_sparse_loop(X, W1, W2, I, g), rtol=1e-12, atol=1e-13)
    # the paper's FlexAttention identity (P:953-P:968), per expert over its clustered rows
    y_flex = np.zeros_like(y_dense)
    for e in range(W1.shape[0]):
        tt, jj = np.nonzero(I == e)
        if tt.size:
            y_flex[tt] += g[tt, jj][:, None] * O.expert_flex_form(X[tt], W1[e], W2[e])
    np.testing.assert_allclose(y_dense, y_flex, rtol=1e-10, atol=1e-11)


def test_experts_special_cases():
    X, W1, W2, I, g = _expert_problem(21)
    assert np.all(O.experts_dense(np.zeros_like(X), W1, W2, I, g) == 0)       # zero in -> zero out
    rng = np.random.default_rng(22)
    Xi = rng.standard_normal((12, 4))
    eye = np.eye(4)[None]                                                     # d_e = d_h, W1 = W2 = I
    y = O.experts_dense(Xi, eye, eye, np.zeros((12, 1), np.int64), np.ones((12, 1)))
    np.testing.assert_allclose(y, O.gelu(Xi), rtol=1e-15)


# ---------------------------------------------------------------- clustering (Fig. 2)
def test_cluster_plan_brute_force():
    rng = np.random.default_rng(30)
    T, k, N_e = 50, 3, 7
    I = np.stack([rng.choice(N_e, k, replace=False) for _ in range(T)])
    perm, pos, off = O.cluster_plan(I, N_e)
    ref = sorted(range(T * k), key=lambda r: (I[r // k, r % k], r))      # stable by expert
    np.testing.assert_array_equal(perm, ref)
    for t in range(T):
        for j in range(k):
            assert perm[pos[t, j]] == t * k + j
    assert off[0] == 0 and off[-1] == T * k and np.all(np.diff(off) >= 0)
    for e in range(N_e):
        assert np.all(I.reshape(-1)[perm[off[e]:off[e + 1]]] == e)
    # everything to expert 0 (degenerate)
    p0, q0, o0 = O.cluster_plan(np.zeros((5, 1), np.int64), 4)
    np.testing.assert_array_equal(p0, np.arange(5)); np.testing.assert_array_equal(o0, [0, 5, 5, 5, 5])


def test_expert_loads_brute_force():
    rng = np.random.default_rng(3)
    T, k, N_e = 50, 3, 7
    I = np.stack([rng.choice(N_e, size=k, replace=False) for _ in range(T)])
    count = {}
    for t in range(T):
        for j in range(k):
            count[int(I[t, j])] = count.get(int(I[t, j]), 0) + 1
    load = O.expert_loads(I, N_e)
    assert [count.get(e, 0) for e in range(N_e)] == load.tolist()
    assert load.sum() == T * k and load.max() <= T


def test_update_bias_sign_rule_cases():
    """S:248-S:251 examples: balanced -> unchanged; one overloaded expert -> exactly -gamma;
    underloaded experts move up by gamma; the update is fp32."""
    b = np.array([0.5, -0.25, 0.125, 0.0], np.float32)
    assert np.array_equal(O.update_bias(b, np.array([5, 5, 5, 5]), 1e-3), b)
    nb = O.update_bias(b, np.array([8, 4, 4, 4]), 1e-3)          # mean 5
    assert nb.dtype == np.float32
    assert nb[0] == np.float32(b[0] - np.float32(1e-3))
    assert np.all(nb[1:] == (b[1:] + np.float32(1e-3)).astype(np.float32))
    # mean need not be an integer: load == mean never happens, every expert moves
    nb = O.update_bias(b, np.array([3, 2, 2, 2]), 0.5)            # mean 2.25
    assert np.array_equal(nb, (b + np.float32(0.5) * np.array([-1, 1, 1, 1], np.float32)).astype(np.float32))


def test_update_bias_closed_loop_reduces_imbalance():
    """closed loop on skewed synthetic tokens -> max/mean expert load decreases
    (router = the oracle's full-sort top-k, bias only steers selection)."""
    rng = np.random.default_rng(11)
    T, d_h, N_e, k = 512, 16, 8, 2
    X = rng.standard_normal((T, d_h))
    W = rng.standard_normal((d_h, N_e)) * 0.1
    W[:, 0] += 0.3                                                # expert 0 preferred
    X[:, :] += 0.5
    b = np.zeros(N_e, np.float32)
    ratios = []
    for _ in range(200):
        I, *_ = O.route_topk(X, W, b.astype(np.float64), k)
        load = O.expert_loads(I, N_e)
        ratios.append(load.max() / load.mean())
        b = O.update_bias(b, load, 2e-2)
    assert ratios[0] > 1.5
    assert np.mean(ratios[-20:]) < 0.75 * ratios[0]
