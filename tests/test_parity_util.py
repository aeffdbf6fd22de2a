"""The comparison helpers themselves (tests/parity_util.py), on CPU."""
import numpy as np

import oracle as O
from parity_util import dW_r_scale, rel_err_slices, xs_band_ratio
from workloads import LayerConfig, make_problem


def test_dW_r_scale_bounds_the_reference_componentwise():
    cfg = LayerConfig("p", T=64, d=64, N_h=2, d_h=32, N_e=16, k=4, d_e=16, dtype="bf16")
    W, x, dout = make_problem(cfg, 0, "conf")
    P = {k: v.astype(np.float64) for k, v in W.items()}
    C = O.layer_forward(P, x.astype(np.float64), cfg.k, mode="bf16")
    gr = O.layer_backward(P, x.astype(np.float64), dout.astype(np.float64), C)
    sc = dW_r_scale(P, C, gr)
    assert np.all(np.abs(gr["dW_r"]) <= sc * (1 + 1e-12) + 1e-300)
    assert np.all((sc > 0) == (np.abs(gr["dW_r"]) > 0) | (sc > 0))


def test_rel_err_slices_flags_a_single_bad_slice_and_zero_slices():
    ref = np.ones((4, 3, 5))
    ref[2] *= 1e-3                      # a small slice: its error must be judged against itself
    gpu = ref.copy()
    gpu[2, 0, 0] += 1e-4                # 10 % of that slice, 1e-4 of the global max
    assert rel_err_slices(gpu, ref, (0,)) > 0.05
    z = np.zeros((2, 3))
    assert rel_err_slices(z + np.array([[0, 0, 0], [0, 1e-9, 0]]), z, (0,)) == float("inf")


def test_xs_band_ratio_is_distance_to_midpoint_in_units():
    x = np.ones((1, 4))
    W = np.ones((1, 4)) * 0.25
    # exact value 1 + 2^-8 = a bf16 rounding midpoint (between 1 and 1 + 2^-7) -> distance 0
    Xs = np.array([[1.0 + 2.0 ** -8]])
    assert xs_band_ratio(x, W, Xs)[0, 0] == 0.0
    Xs = np.array([[1.0]])              # on a representable value: half an ulp (2^-8) from a midpoint
    unit = 2.0 ** -24 * 2.0 * 0.5
    assert np.isclose(xs_band_ratio(x, W, Xs)[0, 0], 2.0 ** -8 / unit)
