"""Plain, slow, obviously-correct fp64 oracle of the Multi-Head LatentMoE layer.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``): the product path never
imports this module.

Citations are ``P:n`` = line n of the paper's LaTeX (PAPER.md, arxiv
2602.04870) and ``R#`` = a reading listed in DESIGN.md ("Readings of the
paper").  Every function writes out the plain definition; library primitives
used as steps are numpy matmul/argsort and ``scipy.special.erf``.  There is no
blocking, fusion or reordering beyond what the cited definition states.

Shapes (global problem, independent of the number of GPUs G):
    x      [T, d]                tokens (B*T flattened b-major, R20)
    W_in   [D, d]   D = N_h*d_h  Eq. 5, P:765  (x_t -> W_in x_t)
           or [2D, d] with separate routing sub-tokens (ablation, P:1565-P:1570):
           [x_t1..x_tNh, r_t1..r_tNh] = split(W_in x_t); head i routes on r_ti and
           computes its experts on x_ti
    W_out  [d, D]                Eq. 6
    W_r    [N_h, d_h, N_e]       router, fp32 values (Alg. 1 REQUIRE)
    b      [N_h, N_e]            aux-free load-balancing bias
    W1, W2 [N_h, N_e, d_e, d_h]  expert e of head h computes gelu(x W1_e^T) W2_e (R2)

``mode`` selects the storage rounding applied at the boundaries where the
GPU path stores a tensor (R9): 'bf16' (round-to-nearest-even to bfloat16),
'fp32' (round to float32) or 'fp64' (no rounding).  All arithmetic is fp64.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.special import erf as _erf

__all__ = [
    "NonFiniteScore", "round_storage", "gelu", "gelu_grad", "softmax_lastaxis",
    "router_scores", "route_topk", "gates_from_scores", "gates_eq2_masked",
    "ord32", "pack_key", "unpack_key", "route_online_alg1",
    "experts_dense", "experts_sparse_loop", "expert_flex_form",
    "cluster_plan", "layer_forward", "layer_backward", "hp_layer_forward",
    "hp_layer_backward", "hp_a2a_bytes", "layer_flops", "moe_flops_equivalent",
    "ep_dispatch_rows", "ForwardCache", "expert_loads", "update_bias", "has_routing_tokens",
]


class NonFiniteScore(ValueError):
    """A router score or biased key is NaN/Inf (R7)."""


# ---------------------------------------------------------------------------
# Storage rounding (R9).  Oracle-private: fp64 -> bf16 RNE through frexp.
# ---------------------------------------------------------------------------
def _round_bf16_from_f64(a: np.ndarray) -> np.ndarray:
    """Round fp64 values to the nearest bfloat16 (8 significant bits), ties to even.

    Direct fp64 -> bf16 rounding (no intermediate fp32 step, so no double
    rounding).  m in [0.5, 1) times 2**8 is rounded with np.rint, which is
    round-half-to-even.  Normal bf16 range only (|a| >= 2**-126); smaller
    magnitudes are flushed through the same formula (never reached by our
    workloads, whose magnitudes are O(1e-3..1e2)).
    """
    a = np.asarray(a, dtype=np.float64)
    m, e = np.frexp(a)
    return np.ldexp(np.rint(m * 256.0), e - 8)


def round_storage(a: np.ndarray, mode: str) -> np.ndarray:
    """rnd(.) of R9: the value the GPU path holds after storing ``a`` in ``mode``."""
    a = np.asarray(a, dtype=np.float64)
    if mode == "bf16":
        return _round_bf16_from_f64(a)
    if mode == "fp32":
        return a.astype(np.float32).astype(np.float64)
    if mode == "fp64":
        return a.copy()
    raise ValueError(f"unknown mode {mode!r}")


# ---------------------------------------------------------------------------
# Activation (R1: exact erf GELU; P:936 sigma, P:953-P:955 gelu)
# ---------------------------------------------------------------------------
_SQRT1_2 = 1.0 / math.sqrt(2.0)
_INV_SQRT_2PI = 1.0 / math.sqrt(2.0 * math.pi)


def gelu(x: np.ndarray) -> np.ndarray:
    """gelu(x) = x * Phi(x), Phi(x) = (1 + erf(x / sqrt 2)) / 2   (R1)."""
    x = np.asarray(x, dtype=np.float64)
    return x * 0.5 * (1.0 + _erf(x * _SQRT1_2))


def gelu_grad(x: np.ndarray) -> np.ndarray:
    """d gelu / dx = Phi(x) + x * phi(x), phi the standard normal pdf."""
    x = np.asarray(x, dtype=np.float64)
    return 0.5 * (1.0 + _erf(x * _SQRT1_2)) + x * _INV_SQRT_2PI * np.exp(-0.5 * x * x)


def softmax_lastaxis(z: np.ndarray) -> np.ndarray:
    """Max-subtracted softmax along the last axis (Eq. 2).  -inf entries give 0."""
    z = np.asarray(z, dtype=np.float64)
    m = np.max(z, axis=-1, keepdims=True)
    e = np.exp(z - m)
    return e / np.sum(e, axis=-1, keepdims=True)


# ---------------------------------------------------------------------------
# Routing (Eq. 2-4, P:509-P:511; Alg. 1, P:819-P:841; bias trick P:885-P:886)
# ---------------------------------------------------------------------------
def router_scores(X_h: np.ndarray, W_r_h: np.ndarray) -> np.ndarray:
    """s_{i,t} = r(x_t)_i with a linear router (Eq. 4): S = X_h W_r[h]  [T, N_e]."""
    return np.asarray(X_h, np.float64) @ np.asarray(W_r_h, np.float64)


def route_topk(X_h, W_r_h, b_h, k):
    """Top-k selection by a FULL SORT of the biased keys (Eq. 3; P:885-P:886).

    keys K = S + b select the experts; the returned scores are the raw, unbiased
    S at the selected experts (R5).  Slot order: descending K, ties to the lower
    expert index (R5, R6) - a stable argsort of -K keeps ascending index order
    among equal keys (and -0.0 == +0.0 ties by index, R6).

    Returns (I [T,k] int64, S_sel [T,k], margin [T], S [T,N_e], K [T,N_e]);
    margin = K_(k) - K_(k+1), +inf when k == N_e (R8).
    """
    S = router_scores(X_h, W_r_h)
    K = S + np.asarray(b_h, np.float64)[None, :]
    if not np.all(np.isfinite(K)):
        raise NonFiniteScore("non-finite router score/key (R7)")
    T, N_e = K.shape
    if not (1 <= k <= N_e):
        raise ValueError("k must satisfy 1 <= k <= N_e")
    order = np.argsort(-K, axis=1, kind="stable")
    I = order[:, :k]
    rows = np.arange(T)[:, None]
    S_sel = S[rows, I]
    if k < N_e:
        margin = K[np.arange(T), order[:, k - 1]] - K[np.arange(T), order[:, k]]
    else:
        margin = np.full(T, np.inf)
    return I.astype(np.int64), S_sel, margin, S, K


def gates_from_scores(S_sel: np.ndarray) -> np.ndarray:
    """g = softmax over the k selected unbiased scores (Eq. 2-3 with -inf elsewhere, R4)."""
    return softmax_lastaxis(S_sel)


def gates_eq2_masked(S: np.ndarray, I: np.ndarray) -> np.ndarray:
    """Literal Eq. 2-3 (P:509-P:510): N_e-wide softmax of g' (s if selected, -inf
    otherwise), gathered at I.  Independent form used to pin gates_from_scores."""
    T, N_e = S.shape
    gp = np.full((T, N_e), -np.inf)
    rows = np.arange(T)[:, None]
    gp[rows, I] = S[rows, I]
    g_full = softmax_lastaxis(gp)
    return g_full[rows, I]


# --- Alg. 1 (online block top-k with packed 64-bit keys), used as a pin -----
def ord32(v: np.ndarray) -> np.ndarray:
    """Order-preserving map float32 -> uint32 (R6): flip the sign bit of
    non-negative values, all bits of negative ones; -0.0 is canonicalised to +0.0."""
    f = np.asarray(v, dtype=np.float32).copy()
    f[f == 0] = 0.0  # canonicalise -0.0 (R6)
    u = f.view(np.uint32).astype(np.uint64)
    neg = (u >> np.uint64(31)) == 1
    return np.where(neg, (~u) & np.uint64(0xFFFFFFFF), u | np.uint64(0x80000000)).astype(np.uint64)


def pack_key(v_f32: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """64-bit key = ord32(score) << 32 | (~idx & 0xffffffff)  (R6).
    The maximum key is the highest score, ties going to the LOWER index."""
    idx = np.asarray(idx, dtype=np.uint64)
    return (ord32(v_f32) << np.uint64(32)) | ((~idx) & np.uint64(0xFFFFFFFF))


def unpack_key(key: np.ndarray):
    """Inverse of pack_key: (float32 score, int64 index)."""
    key = np.asarray(key, dtype=np.uint64)
    hi = (key >> np.uint64(32)) & np.uint64(0xFFFFFFFF)
    lo = key & np.uint64(0xFFFFFFFF)
    idx = ((~lo) & np.uint64(0xFFFFFFFF)).astype(np.int64)
    pos = (hi >> np.uint64(31)) == 1
    bits = np.where(pos, hi & np.uint64(0x7FFFFFFF), (~hi) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    return bits.view(np.float32), idx


def route_online_alg1(X_h, W_r_h, b_h, k, M):
    """Algorithm 1 (P:819-P:841) for one head, step by step, keys held as float32.

    For each expert block of M: S_block = X W_r,block + b_block (line 7), pack
    (line 8), block top-k (line 9), merge with the accumulator A (init 0, line 4;
    line 10).  Then unpack (line 12) and remove the bias (line 13).  Returns
    (I_top [T,k], S_top [T,k]) with S_top = S' - b[I] exactly as line 13 states.
    """
    X_h = np.asarray(X_h, np.float64)
    T = X_h.shape[0]
    N_e = W_r_h.shape[1]
    A = np.zeros((T, k), dtype=np.uint64)                      # line 4
    for e0 in range(0, N_e, M):                                # line 5
        e1 = min(N_e, e0 + M)
        S_block = (X_h @ np.asarray(W_r_h, np.float64)[:, e0:e1]
                   + np.asarray(b_h, np.float64)[None, e0:e1])  # line 7
        keys = pack_key(S_block.astype(np.float32),
                        np.broadcast_to(np.arange(e0, e1), S_block.shape))  # line 8
        kk = min(k, e1 - e0)
        blk = np.sort(keys, axis=1)[:, ::-1][:, :kk]            # line 9 (uint64 sort)
        merged = np.concatenate([A, blk], axis=1)
        A = np.sort(merged, axis=1)[:, ::-1][:, :k]            # line 10
    S_prime, I = unpack_key(A)                                  # line 12
    S_top = S_prime.astype(np.float64) - np.asarray(b_h, np.float64)[I]  # line 13
    return I, S_top


# ---------------------------------------------------------------------------
# Experts (Eq. 1; single expert sigma(X W_in^T) W_out; R2)
# ---------------------------------------------------------------------------
def _selection_weights(I: np.ndarray, g: np.ndarray, N_e: int) -> np.ndarray:
    """w[t, e] = g[t, j] if I[t, j] == e else 0 (Eq. 3's -inf => weight 0)."""
    T = I.shape[0]
    w = np.zeros((T, N_e))
    w[np.arange(T)[:, None], I] = g
    return w


def experts_dense(X_h, W1_h, W2_h, I, g):
    """y_t = sum_i g_{i,t} E_i(x_t) (Eq. 1) computed DENSELY over all N_e experts
    with a selection mask; E_e(x) = gelu(x W1_e^T) W2_e (R2)."""
    X_h = np.asarray(X_h, np.float64)
    N_e = W1_h.shape[0]
    w = _selection_weights(I, g, N_e)
    y = np.zeros((X_h.shape[0], W2_h.shape[2]))
    for e in range(N_e):
        H = X_h @ np.asarray(W1_h[e], np.float64).T
        Y = gelu(H) @ np.asarray(W2_h[e], np.float64)
        y += w[:, e:e + 1] * Y
    return y


def experts_sparse_loop(X_h, W1_h, W2_h, I, g):
    """Per-token loop over only the k selected experts (Eq. 1 read literally);
    an independent path pinning experts_dense."""
    X_h = np.asarray(X_h, np.float64)
    T, k = I.shape
    y = np.zeros((T, W2_h.shape[2]))
    for t in range(T):
        for j in range(k):
            e = int(I[t, j])
            h = gelu(np.asarray(W1_h[e], np.float64) @ X_h[t])
            y[t] += g[t, j] * (h @ np.asarray(W2_h[e], np.float64))
    return y


def expert_flex_form(X_rows, W1_e, W2_e):
    """The paper's FlexAttention formulation of one expert (P:953-P:968):
    score_mod(s) = log(gelu(s) + 1); O' = softmax(score_mod(X K^T)) V with
    K = W1_e, V = W2_e; l = sum_j (gelu(s_j) + 1); result O' * l - sum_j V_j.
    Equals gelu(X W1_e^T) W2_e exactly in real arithmetic (pin for experts_*)."""
    s = np.asarray(X_rows, np.float64) @ np.asarray(W1_e, np.float64).T
    z = np.log(gelu(s) + 1.0)                     # Eq. 8 score_mod
    O_prime = softmax_lastaxis(z) @ np.asarray(W2_e, np.float64)
    ell = np.sum(np.exp(z), axis=-1, keepdims=True)
    return O_prime * ell - np.sum(np.asarray(W2_e, np.float64), axis=0)[None, :]


def cluster_plan(I: np.ndarray, N_e: int):
    """Token clustering (Fig. 2, P:941-P:949): replicas r = t*k + j stably
    sorted by expert.  Returns perm [T*k] (sorted position -> r), pos [T,k]
    (r -> sorted position), off [N_e+1] (segment offsets).  Dropless:
    every replica appears exactly once."""
    T, k = I.shape
    flat = np.asarray(I, np.int64).reshape(-1)
    perm = np.argsort(flat, kind="stable")
    pos = np.empty_like(perm)
    pos[perm] = np.arange(flat.size)
    counts = np.bincount(flat, minlength=N_e)
    off = np.concatenate([[0], np.cumsum(counts)])
    return perm.astype(np.int64), pos.reshape(T, k).astype(np.int64), off.astype(np.int64)


# ---------------------------------------------------------------------------
# The layer (Eq. 5-6, P:763-P:775) forward and hand-derived backward
# ---------------------------------------------------------------------------
@dataclass
class ForwardCache:
    mode: str
    Xs: np.ndarray                    # rnd(x W_in^T)           [T, D]
    Xs_pre: np.ndarray | None = None  # x W_in^T before the storage rounding (fp64)
    I: list = field(default_factory=list)       # per head [T,k]
    g: list = field(default_factory=list)       # per head [T,k]
    S_sel: list = field(default_factory=list)   # per head [T,k]
    margin: list = field(default_factory=list)  # per head [T]
    y: list = field(default_factory=list)       # per head [T,d_h] (unrounded)
    cat: np.ndarray | None = None     # rnd(concat y_h)         [T, D]
    out: np.ndarray | None = None     # rnd(cat W_out^T)        [T, d]


def _heads(P):
    N_h, d_h = P["W_r"].shape[0], P["W_r"].shape[1]
    return N_h, d_h


def has_routing_tokens(P) -> bool:
    """W_in [2D, d]: the separate-routing-token variant of P:1565-P:1570."""
    N_h, d_h = _heads(P)
    D = N_h * d_h
    rows = np.asarray(P["W_in"]).shape[0]
    if rows not in (D, 2 * D):
        raise ValueError("W_in must have N_h*d_h rows (or 2*N_h*d_h with routing tokens)")
    return rows == 2 * D


def layer_forward(P: dict, x: np.ndarray, k: int, mode: str = "bf16",
                  forced_idx: dict | None = None) -> ForwardCache:
    """o_t = W_out concat(f_1(x_t1), ..., f_Nh(x_tNh)), [x_t1..x_tNh] = split(W_in x_t).

    Steps O1-O8 of DESIGN.md: Eq. 5 split, per head the MoE of
    Eq. 1-4 (P:508-P:511) with the biased top-k of P:885, Eq. 6.
    ``forced_idx`` {h: I [T,k]} overrides the selection (R11) for gradient
    comparisons across near-ties; gates are then the softmax of the raw
    scores at the forced experts.
    """
    N_h, d_h = _heads(P)
    D = N_h * d_h
    rtok = has_routing_tokens(P)
    x = np.asarray(x, np.float64)
    Xs_pre = x @ np.asarray(P["W_in"], np.float64).T
    Xs = round_storage(Xs_pre, mode)                                          # O1
    C = ForwardCache(mode=mode, Xs=Xs, Xs_pre=Xs_pre)
    ys = []
    for h in range(N_h):
        X_h = Xs[:, h * d_h:(h + 1) * d_h]                                   # O2
        # routing sub-token: x_th itself, or r_th = columns D + h*d_h.. (P:1568-P:1569)
        R_h = Xs[:, D + h * d_h:D + (h + 1) * d_h] if rtok else X_h
        I, S_sel, margin, S, _K = route_topk(R_h, P["W_r"][h], P["b"][h], k)  # O3-O4
        if forced_idx is not None and h in forced_idx:
            I = np.asarray(forced_idx[h], np.int64)
            S_sel = S[np.arange(S.shape[0])[:, None], I]
        g = gates_from_scores(S_sel)                                          # O5
        y = experts_dense(X_h, P["W1"][h], P["W2"][h], I, g)                  # O6
        C.I.append(I); C.g.append(g); C.S_sel.append(S_sel); C.margin.append(margin); C.y.append(y)
        ys.append(y)
    C.cat = round_storage(np.concatenate(ys, axis=1), mode)                   # O7
    C.out = round_storage(C.cat @ np.asarray(P["W_out"], np.float64).T, mode)  # O8
    return C


def layer_backward(P: dict, x: np.ndarray, dout: np.ndarray, C: ForwardCache) -> dict:
    """Hand-derived dense-masked backward (O9-O12; Alg. 2 P:846-P:866 for the router).

    dW_r gets gradient only through the selected scores (R13); no bias gradient.
    Returns dict(dx, dW_in, dW_out, dW_r, dW1, dW2, dXs, dcat, dg, dS).
    """
    mode = C.mode
    N_h, d_h = _heads(P)
    D = N_h * d_h
    rtok = has_routing_tokens(P)
    x = np.asarray(x, np.float64)
    dout = np.asarray(dout, np.float64)
    W_out = np.asarray(P["W_out"], np.float64)
    dW_out = dout.T @ C.cat                                                   # O9
    dcat = round_storage(dout @ W_out, mode)
    dW_r = np.zeros(P["W_r"].shape)
    dW1 = np.zeros(P["W1"].shape)
    dW2 = np.zeros(P["W2"].shape)
    dXs_heads, dR_heads, dgs, dSs = [], [], [], []
    for h in range(N_h):
        X_h = C.Xs[:, h * d_h:(h + 1) * d_h]
        R_h = C.Xs[:, D + h * d_h:D + (h + 1) * d_h] if rtok else None
        dY = dcat[:, h * d_h:(h + 1) * d_h]                                   # O10
        gh = _head_backward(_head_params(P, h), X_h, dY, C.I[h], C.g[h], R_h)  # O10-O11
        dW_r[h], dW1[h], dW2[h] = gh["dW_r"], gh["dW1"], gh["dW2"]
        dXs_heads.append(gh["dXs_h"]); dgs.append(gh["dg"]); dSs.append(gh["dS"])
        if rtok:
            dR_heads.append(gh["dR_h"])
    dXs = round_storage(np.concatenate(dXs_heads + dR_heads, axis=1), mode)  # O12
    dx = round_storage(dXs @ np.asarray(P["W_in"], np.float64), mode)
    dW_in = dXs.T @ x
    return dict(dx=dx, dW_in=dW_in, dW_out=dW_out, dW_r=dW_r, dW1=dW1, dW2=dW2,
                dXs=dXs, dcat=dcat, dg=dgs, dS=dSs)


# ---------------------------------------------------------------------------
# Head Parallel, emulated by literal sharding (P:796-P:813; R12)
# ---------------------------------------------------------------------------
def _check_hp(N_h, G):
    if not (1 <= G <= N_h and N_h % G == 0):
        raise ValueError("Head Parallel needs P <= N_h and N_h % P == 0 (P:803)")


def hp_a2a_bytes(T_loc: int, N_h: int, d_h: int, G: int, el: int) -> np.ndarray:
    """Byte matrix B[src, dst] of one HP all-to-all: each rank sends each peer
    its T_loc tokens x (N_h/G) heads x d_h (P:804-P:805), self-sends excluded.
    Independent of k and of the routing (P:811-P:812)."""
    _check_hp(N_h, G)
    B = np.full((G, G), T_loc * (N_h // G) * d_h * el, dtype=np.int64)
    np.fill_diagonal(B, 0)
    return B


def hp_layer_forward(P: dict, x: np.ndarray, k: int, G: int, mode: str = "bf16"):
    """HP forward on G emulated ranks.  Rank r owns tokens [r*T_loc, (r+1)*T_loc)
    and heads [r*N_h/G, (r+1)*N_h/G) (R12).  Every send buffer is built
    literally; bytes crossing ranks are counted.  Returns (out [T,d], per-rank
    state list, byte matrix [G,G] summed over both forward all-to-alls)."""
    N_h, d_h = _heads(P)
    _check_hp(N_h, G)
    D = N_h * d_h
    rtok = has_routing_tokens(P)
    x = np.asarray(x, np.float64)
    T = x.shape[0]
    if T % G:
        raise ValueError("T must be divisible by G")
    T_loc, H_loc = T // G, N_h // G
    HD = H_loc * d_h
    el = {"bf16": 2, "fp32": 4, "fp64": 8}[mode]
    nbytes = np.zeros((G, G), np.int64)
    # rank r: projection of its own tokens (Eq. 5), split into destination blocks; with routing
    # sub-tokens the block also carries r_t of the destination's heads (twice the bytes)
    send1 = {}
    for r in range(G):
        Xs_r = round_storage(x[r * T_loc:(r + 1) * T_loc] @ np.asarray(P["W_in"], np.float64).T, mode)
        for p in range(G):
            blk = Xs_r[:, p * HD:(p + 1) * HD].copy()
            if rtok:
                blk = np.concatenate([blk, Xs_r[:, D + p * HD:D + (p + 1) * HD]], axis=1)
            send1[(r, p)] = blk
            if p != r:
                nbytes[r, p] += blk.size * el
    ranks = []
    for p in range(G):
        # all-to-all #1: rank p receives all tokens of its heads, sources in rank order
        recv1 = np.concatenate([send1[(r, p)] for r in range(G)], axis=0)   # [T, H_loc*d_h]
        st = {"I": [], "g": [], "y": [], "Xs": recv1}
        for hl in range(H_loc):
            h = p * H_loc + hl
            X_h = recv1[:, hl * d_h:(hl + 1) * d_h]
            R_h = recv1[:, HD + hl * d_h:HD + (hl + 1) * d_h] if rtok else X_h
            I, S_sel, _m, _S, _K = route_topk(R_h, P["W_r"][h], P["b"][h], k)
            g = gates_from_scores(S_sel)
            st["I"].append(I); st["g"].append(g)
            st["y"].append(experts_dense(X_h, P["W1"][h], P["W2"][h], I, g))
        ranks.append(st)
    out = np.zeros((T, P["W_out"].shape[0]))
    for r in range(G):
        # all-to-all #2: rank r gathers its tokens' outputs of every head
        blocks = []
        for p in range(G):
            y_p = np.concatenate(ranks[p]["y"], axis=1)[r * T_loc:(r + 1) * T_loc]
            blk = round_storage(y_p, mode)
            if p != r:
                nbytes[p, r] += blk.size * el
            blocks.append(blk)
        cat_r = np.concatenate(blocks, axis=1)
        ranks[r]["cat"] = cat_r
        out[r * T_loc:(r + 1) * T_loc] = round_storage(cat_r @ np.asarray(P["W_out"], np.float64).T, mode)
    return out, ranks, nbytes


def hp_layer_backward(P, x, dout, k, G, mode="bf16"):
    """HP backward on G emulated ranks (mirror of hp_layer_forward; all-to-alls
    #3 and #4).  dW_in / dW_out are returned summed over ranks (R19)."""
    out, ranks, nb_f = hp_layer_forward(P, x, k, G, mode)
    N_h, d_h = _heads(P)
    rtok = has_routing_tokens(P)
    T = x.shape[0]
    T_loc, H_loc = T // G, N_h // G
    HD = H_loc * d_h
    el = {"bf16": 2, "fp32": 4, "fp64": 8}[mode]
    nbytes = np.zeros((G, G), np.int64)
    x = np.asarray(x, np.float64)
    dout = np.asarray(dout, np.float64)
    W_out = np.asarray(P["W_out"], np.float64)
    N_e = P["W1"].shape[1]
    dW_out = np.zeros(W_out.shape)
    dcat = {}
    for r in range(G):
        do_r = dout[r * T_loc:(r + 1) * T_loc]
        dW_out += do_r.T @ ranks[r]["cat"]
        dc = round_storage(do_r @ W_out, mode)
        for p in range(G):
            dcat[(r, p)] = dc[:, p * H_loc * d_h:(p + 1) * H_loc * d_h]
            if p != r:
                nbytes[r, p] += dcat[(r, p)].size * el
    dW_r = np.zeros(P["W_r"].shape); dW1 = np.zeros(P["W1"].shape); dW2 = np.zeros(P["W2"].shape)
    dXs_blocks = {}
    for p in range(G):
        recv3 = np.concatenate([dcat[(r, p)] for r in range(G)], axis=0)
        dX_loc, dR_loc = [], []
        for hl in range(H_loc):
            h = p * H_loc + hl
            X_h = ranks[p]["Xs"][:, hl * d_h:(hl + 1) * d_h]
            R_h = ranks[p]["Xs"][:, HD + hl * d_h:HD + (hl + 1) * d_h] if rtok else None
            gh = _head_backward(_head_params(P, h), X_h, recv3[:, hl * d_h:(hl + 1) * d_h],
                                ranks[p]["I"][hl], ranks[p]["g"][hl], R_h)
            dW_r[h] = gh["dW_r"]; dW1[h] = gh["dW1"]; dW2[h] = gh["dW2"]
            dX_loc.append(gh["dXs_h"])
            if rtok:
                dR_loc.append(gh["dR_h"])
        dXl = np.concatenate(dX_loc + dR_loc, axis=1)   # [T, HD] or [T, 2HD] (dX | dR of local heads)
        for r in range(G):
            blk = round_storage(dXl[r * T_loc:(r + 1) * T_loc], mode)
            dXs_blocks[(p, r)] = blk
            if p != r:
                nbytes[p, r] += blk.size * el
    dx = np.zeros(x.shape); dW_in = np.zeros(P["W_in"].shape)
    for r in range(G):
        dXs_r = np.concatenate([dXs_blocks[(p, r)][:, :HD] for p in range(G)]
                               + ([dXs_blocks[(p, r)][:, HD:] for p in range(G)] if rtok else []), axis=1)
        dx[r * T_loc:(r + 1) * T_loc] = round_storage(dXs_r @ np.asarray(P["W_in"], np.float64), mode)
        dW_in += dXs_r.T @ x[r * T_loc:(r + 1) * T_loc]
    return dict(out=out, dx=dx, dW_in=dW_in, dW_out=dW_out, dW_r=dW_r, dW1=dW1, dW2=dW2,
                bytes_fwd=nb_f, bytes_bwd=nbytes)


def _head_params(P, h):
    return dict(W_r=P["W_r"][h:h + 1], b=P["b"][h:h + 1], W1=P["W1"][h:h + 1], W2=P["W2"][h:h + 1])


def _head_backward(Ph, X_h, dY, I, g, R_h=None):
    """Per-head part of O10-O11: chain rule of Eq. 1 through the dense-masked
    experts (dW2 = A^T (w dY), dH = (w dY W2^T) * gelu'(H), dW1 = dH^T X,
    dX += dH W1, dg_j = <dY, E_{I_j}(x)>), the softmax Jacobian of Eq. 2 over the
    k selected scores (dS = g (dg - sum g dg)), and Alg. 2 (P:846-P:866) in its
    dense-masked form: dW_r = X^T dS_full, dX += dS_full W_r^T (R13).  With a
    separate routing sub-token R_h (P:1565-P:1570) the router terms use R_h:
    dW_r = R^T dS_full and dR = dS_full W_r^T is returned apart from dX."""
    N_e = Ph["W1"].shape[1]
    T, k = I.shape
    w = _selection_weights(I, g, N_e)
    dXs_h = np.zeros_like(X_h)
    dg = np.zeros((T, k))
    dW1 = np.zeros(Ph["W1"].shape[1:]); dW2 = np.zeros(Ph["W2"].shape[1:])
    for e in range(N_e):
        W1e = np.asarray(Ph["W1"][0, e], np.float64); W2e = np.asarray(Ph["W2"][0, e], np.float64)
        H = X_h @ W1e.T
        A = gelu(H)
        Y = A @ W2e
        dYe = w[:, e:e + 1] * dY
        dW2[e] = A.T @ dYe
        dH = (dYe @ W2e.T) * gelu_grad(H)
        dW1[e] = dH.T @ X_h
        dXs_h += dH @ W1e
        tt, jj = np.nonzero(I == e)
        if tt.size:
            dg[tt, jj] = np.sum(dY[tt] * Y[tt], axis=1)
    dS = g * (dg - np.sum(g * dg, axis=1, keepdims=True))
    dS_full = np.zeros((T, N_e))
    dS_full[np.arange(T)[:, None], I] = dS
    W_r_h = np.asarray(Ph["W_r"][0], np.float64)
    if R_h is None:
        dW_r = X_h.T @ dS_full
        dXs_h = dXs_h + dS_full @ W_r_h.T
        return dict(dXs_h=dXs_h, dW_r=dW_r, dW1=dW1, dW2=dW2, dg=dg, dS=dS)
    dW_r = R_h.T @ dS_full
    return dict(dXs_h=dXs_h, dR_h=dS_full @ W_r_h.T, dW_r=dW_r, dW1=dW1, dW2=dW2, dg=dg, dS=dS)


# ---------------------------------------------------------------------------
# Aux-free, global load balancing (rule per S:245-S:253, R24)
# ---------------------------------------------------------------------------
def expert_loads(I: np.ndarray, N_e: int) -> np.ndarray:
    """Expert loads of one head over the step's tokens: load[e] = #{(t, j): I[t, j] = e}.
    Under HP the head's whole token set is on one rank, so this count is already the
    *global* load the paper balances on."""
    return np.bincount(np.asarray(I, np.int64).reshape(-1), minlength=N_e).astype(np.int64)


def update_bias(b_h: np.ndarray, load: np.ndarray, gamma: float) -> np.ndarray:
    """Aux-free bias update of one head: b[e] -= gamma * sign(load[e] - mean(load)) (R24; the
    paper cites the aux-free method and only states that the bias enters selection,
    not the scores; the sign rule and gamma come from SPEC S:248).  The bias is
    fp32 (P:1992 'routers compute in FP32'), so the update is evaluated in fp32."""
    load = np.asarray(load, np.float64)
    mean = load.sum() / load.size
    step = np.float32(gamma) * np.sign(load - mean).astype(np.float32)
    return (np.asarray(b_h, np.float32) - step).astype(np.float32)


# ---------------------------------------------------------------------------
# Closed-form counters (P:777 FLOP parity; P:343 / P:1193 EP vs HP volume)
# ---------------------------------------------------------------------------
def layer_flops(T, d, N_h, d_h, N_e, k, d_e):
    """Forward FLOPs (multiply-add = 2) of the layer, split by part."""
    D = N_h * d_h
    return dict(w_in=2 * T * d * D, router=2 * T * N_h * d_h * N_e,
                experts=4 * T * N_h * k * d_h * d_e, w_out=2 * T * D * d)


def moe_flops_equivalent(T, N_h, d_h, N_e, k, d_e):
    """FLOPs of N_h independent MoEs (one per sub-token) = router + experts of a
    single MoE over N_h*T sub-tokens; P:777 says this equals the layer's FLOPs
    'discounting the linear projections'."""
    return 2 * (N_h * T) * d_h * N_e + 4 * (N_h * T) * k * d_h * d_e


def ep_dispatch_rows(T, k):
    """Rows an Expert-Parallel dispatch moves: every token duplicated k times
    (P:539-P:541, "first duplicates tokens").  HP moves each token once
    (P:811), so HP/EP volume = 1/k (25% at k=4)."""
    return T * k
