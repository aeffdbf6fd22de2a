"""The seeded input recipes (workloads/, no method arithmetic): the `exact` recipe's premise that
every sub-token is exact in fp32 whatever the summation order (so the GPU and the oracle round it
to the same bf16 value and north_star's margin rule applies without the R22 budget)."""
import numpy as np

from workloads import EXACT_NNZ, PRESETS, LayerConfig, make_problem


def _fp32_sum_in_order(prod, order):
    acc = np.zeros(prod.shape[:-1], np.float32)
    for i in order:
        acc = acc + prod[..., i]
    return acc


def test_exact_recipe_subtokens_are_exact_in_fp32_for_any_order():
    rng = np.random.default_rng(0)
    for cfg in (PRESETS["paper"].replace(T=8, d=2048), LayerConfig("s", T=32, d=512, N_h=2, d_h=256, N_e=64,
                                                                      k=8, d_e=128, dtype="bf16")):
        W, x, _ = make_problem(cfg, 3, "exact")
        assert np.all((W["W_in"] != 0).sum(1) == EXACT_NNZ)
        exact = x.astype(np.float64) @ W["W_in"].astype(np.float64).T
        prod = x[:, None, :].astype(np.float32) * W["W_in"][None].astype(np.float32)   # exact products
        assert np.array_equal(prod.astype(np.float64), x[:, None, :].astype(np.float64) * W["W_in"][None])
        for _ in range(3):
            got = _fp32_sum_in_order(prod, rng.permutation(cfg.d))
            np.testing.assert_array_equal(got.astype(np.float64), exact)
        # blocked accumulation (tensor-core style: 16-term blocks summed then added) is exact too
        blk = prod.reshape(*prod.shape[:-1], -1, 16).sum(-1, dtype=np.float32)
        np.testing.assert_array_equal(_fp32_sum_in_order(blk, range(blk.shape[-1])).astype(np.float64), exact)
        # the sub-tokens are O(1), like the variance-preserving recipe's
        assert 0.5 < exact.std() < 1.5


def test_exact_recipe_tokens_are_bf16_above_two_to_minus_six():
    cfg = PRESETS["paper"].replace(T=256, d=2048)
    _, x, _ = make_problem(cfg, 1, "exact")
    nz = x[x != 0]
    assert np.all(np.abs(nz) >= 2.0 ** -6)
    u = nz.astype(np.float32).view(np.uint32)
    assert np.all((u & 0xFFFF) == 0)             # bf16-representable
    assert (x == 0).mean() < 0.02
