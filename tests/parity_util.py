"""Comparison rules of the conformance check (R8, R10, R11, R22).

Test infrastructure: runs the oracle on the same seeded inputs as the CUDA path
and compares element by element.
"""
from __future__ import annotations

import numpy as np

import oracle as O

MARGIN = 1e-3          # north_star: exclude sub-tokens whose oracle margin at the k-th expert is < 1e-3
TOL = {"bf16": 2e-2, "fp32": 1e-4}
GATE_TOL = 1e-5
FP32_ACC_REL = 2.0 ** -16   # generous bound on |fp32-accumulated GEMM - exact| / |value| (R22)


def rel_err(gpu, ref) -> float:
    """R10: max|gpu - ref| / max|ref| (infinity-norm relative)."""
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(gpu - ref)) / den) if den > 0 else float(np.max(np.abs(gpu)))


def boundary_flip_budget(Xs_pre: np.ndarray, W_r_h: np.ndarray, mode: str) -> np.ndarray:
    """R22: the bf16 storage of Xs (a boundary tensor, R9) is computed with fp64
    accumulation by the oracle and fp32 accumulation on the GPU; an element whose exact
    value lies within FP32_ACC_REL*|v| of a bf16 rounding midpoint may round to the
    neighbouring bf16 value on the GPU.  Returns, per token, the largest change of any
    router key such 1-ulp flips can cause: max_e sum_{i ambiguous} ulp_i |W_r[i, e]|."""
    if mode != "bf16":
        return np.zeros(Xs_pre.shape[0])
    m, e = np.frexp(Xs_pre)
    ulp = np.ldexp(1.0, e - 8)
    q = m * 256.0
    dist = np.abs((q - np.floor(q)) - 0.5) * ulp          # distance to the nearest rounding midpoint
    amb = dist <= FP32_ACC_REL * np.abs(Xs_pre)
    return np.max((amb * ulp) @ np.abs(W_r_h), axis=1)


def routing_slice(P, h):
    """Columns of Xs that head h routes on: its sub-token, or with separate routing sub-tokens
    (W_in [2D, d], P:1565-P:1570) the r part at column D + h*d_h."""
    N_h, d_h = P["W_r"].shape[0], P["W_r"].shape[1]
    off = N_h * d_h if O.has_routing_tokens(P) else 0
    return slice(off + h * d_h, off + (h + 1) * d_h)


def check_routing(P, C, gpu_idx, k, margin_thr=MARGIN):
    """R8 (+R22): a sub-token is *clean* if its oracle margin minus twice its Xs
    boundary-flip budget is >= 1e-3.  On clean sub-tokens the GPU's index SET must equal
    the oracle's, and the slot order must match on slots separated from both
    neighbours by >= 1e-3 + 2*budget.  Every GPU selection must lie in the oracle's
    near-tie set {e : K_e >= K_(k) - 1e-3 - 2*budget}.  Returns (forced_idx, n_clean,
    n_excluded)."""
    N_h, d_h = P["W_r"].shape[0], P["W_r"].shape[1]
    forced = {}
    n_clean = n_excl = 0
    for h in range(N_h):
        sl = routing_slice(P, h)
        X_h = C.Xs[:, sl]
        I, _S_sel, margin, _S, K = O.route_topk(X_h, P["W_r"][h], P["b"][h], k)
        budget = boundary_flip_budget(C.Xs_pre[:, sl], P["W_r"][h], C.mode)
        gi = np.asarray(gpu_idx[h], np.int64)
        thr = margin_thr + 2 * budget
        clean = margin >= thr
        n_clean += int(clean.sum()); n_excl += int((~clean).sum())
        bad = np.nonzero(clean & np.any(np.sort(gi, 1) != np.sort(I, 1), axis=1))[0]
        assert bad.size == 0, (f"head {h}: {bad.size} clean sub-tokens select different experts, e.g. t={bad[:5]} "
                               f"gpu={gi[bad[:2]]} oracle={I[bad[:2]]}")
        rows = np.arange(I.shape[0])[:, None]
        keys_sel = K[rows, I]
        gap = -np.diff(keys_sel, axis=1)                       # K_(j) - K_(j+1) >= 0
        sep = gap >= thr[:, None]
        sep_prev = np.concatenate([np.ones((I.shape[0], 1), bool), sep], 1)
        sep_next = np.concatenate([sep, np.ones((I.shape[0], 1), bool)], 1)
        must = sep_prev & sep_next & clean[:, None]            # slot j is unambiguous
        if not np.all(gi[must] == I[must]):
            t = np.nonzero(np.any(must & (gi != I), axis=1))[0][:3]
            raise AssertionError(f"head {h}: slot order differs on clean separated slots, t={t}, gpu={gi[t]}, "
                                 f"oracle={I[t]}, keys={K[t[:1]][0][I[t[0]]]}, budget={budget[t]}")
        kth = keys_sel[:, -1]
        in_tie = K[rows, gi] >= (kth - max(margin_thr, MARGIN) - 2 * budget)[:, None]
        assert np.all(in_tie), f"head {h}: a GPU selection is outside the oracle's near-tie set"
        forced[h] = gi
    return forced, n_clean, n_excl
