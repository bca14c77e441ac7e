"""Pin the CPU oracle against golden vectors produced by the reference itself.

The vectors come from tests/golden/make_golden.py, which imports the
reference `mvkernels` package. These tests run on CPU only.
"""

import numpy as np
import pytest

import oracle as O


def g_of(key):
    return tuple(int(v) for v in key.split("_"))


def test_all_36_signatures(golden):
    sigs = [g_of(s) for s in golden["sig_list"]]
    assert len(sigs) == 36
    assert sigs == O.all_signatures(3)


def test_product_tables_bit_exact(golden):
    for s in golden["sig_list"]:
        tgt, cof = O.product_table(g_of(str(s)))
        np.testing.assert_array_equal(tgt, golden[f"table_target_{s}"])
        np.testing.assert_array_equal(cof, golden[f"table_coeff_{s}"])


def test_schedules_match(golden):
    for s in golden["sig_list"]:
        terms = np.array([[t, a, b, int(n)] for t, a, b, n in O.schedule_terms(g_of(str(s)))],
                         dtype=np.int64).reshape(-1, 4)
        np.testing.assert_array_equal(terms, golden[f"sched_{s}"])


def test_schedule_term_counts():
    # tests/test_specialize.py:28-43 known answers
    assert len(O.schedule_terms((1,))) == 4
    assert len(O.schedule_terms((1, 1))) == 16
    assert len(O.schedule_terms((0, 1))) == 12
    assert len(O.schedule_terms((1, 1, 1))) == 64
    assert len(O.schedule_terms((1, -1, 0))) == 48
    assert (2, 3, 1, True) in O.schedule_terms((1, 1))


def test_blade_product_known_answers():
    # tests/test_algebra.py:76-91
    assert O.blade_product(1, 1, (1, 1)) == (0, 1)
    assert O.blade_product(1, 1, (-1, 1)) == (0, -1)
    assert O.blade_product(1, 1, (0, 1)) == (0, 0)
    for g in [(1, 1), (-1, -1), (0, 1)]:
        assert O.blade_product(2, 1, g) == (3, -1)
    assert O.blade_product(3, 3, (1, 1)) == (0, -1)


@pytest.mark.parametrize("n", range(10))
def test_expanded_kernel_bit_exact(golden, n):
    g = tuple(golden[f"conv{n}_g"])
    W = O.expanded_kernel(golden[f"conv{n}_f"], g)
    ref = golden[f"conv{n}_W"]
    assert W.shape == ref.shape
    assert np.array_equal(W, ref)  # +-0 compare equal


@pytest.mark.parametrize("n", range(10))
def test_conv_oracle_matches_reference(golden, n):
    g = tuple(golden[f"conv{n}_g"])
    B, ci, co, di, df, k = golden[f"conv{n}_dims"]
    y = O.conv_ref(golden[f"conv{n}_x"], golden[f"conv{n}_f"], golden[f"conv{n}_b"], g, di, df)
    ref = golden[f"conv{n}_y"]
    assert y.shape == ref.shape
    # both accumulate in fp64 and round once; allow one fp32 ulp for reassociation
    np.testing.assert_allclose(y, ref, rtol=2e-7, atol=1e-9)
    assert O.max_rel_error(y, ref) <= 1e-6
    assert O.conv_flops(B, ci, co, di - df + 1, df, g) == int(golden[f"conv{n}_flops"])
    np.testing.assert_array_equal(O.gather_index_table(di, df, k), golden[f"conv{n}_in_index"])


def test_act_oracle_matches_reference(golden):
    for n in range(int(golden["act_count"])):
        k, mode, K = golden[f"act{n}_meta"]
        ki = tuple(golden[f"act{n}_ki"])
        w = golden[f"act{n}_w"] if mode == 0 else None
        b = golden[f"act{n}_bias"] if mode == 0 else None
        y = O.activation_ref(golden[f"act{n}_x"], int(mode), ki, w, b)
        assert O.max_abs_error(y, golden[f"act{n}_y"]) <= 1e-6, n
        assert O.max_abs_error(y, golden[f"act{n}_y_specialized"]) <= 1e-5, n


def test_spatial_act_matches_server_fold(golden):
    for mode in (0, 1, 2):
        x = golden[f"sact{mode}_x"]
        w = golden[f"sact{mode}_w"] if mode == 0 else None
        b = golden[f"sact{mode}_bias"] if mode == 0 else None
        y = O.activation_ref(x, mode, tuple(range(8)), w, b)
        assert O.max_abs_error(y, golden[f"sact{mode}_y"]) <= 1e-6


@pytest.mark.parametrize("name", ["blk2v", "blk2s", "blk3s", "blk3v"])
def test_block_oracle(golden, name):
    meta = golden[f"{name}_meta"]
    k = int(meta[3])
    g = tuple(int(v) for v in meta[:k])
    pad, residual, mode, B, C, d = (int(v) for v in meta[4:10])
    aw = golden[f"{name}_aw"] if mode == 0 else None
    ab = golden[f"{name}_ab"] if mode == 0 else None
    nb = 1 << k
    y = O.block_ref(golden[f"{name}_x"], g, d, golden[f"{name}_f1"], golden[f"{name}_b1"],
                    mode, tuple(range(nb)), aw, ab, golden[f"{name}_f2"], golden[f"{name}_b2"],
                    padding="same" if pad else "valid", residual=bool(residual))
    assert O.max_rel_error(y, golden[f"{name}_y"]) <= 1e-5


def test_metrics_known_answers(golden):
    a, b = golden["mre_a"], golden["mre_b"]
    assert O.max_rel_error(a, b) == float(golden["mre_default"])
    assert O.max_rel_error(a, b, floor=1.0) == float(golden["mre_floor1"])
    assert O.max_abs_error(a, b) == float(golden["mae"])


def test_activation_flops(golden):
    got = [O.activation_flops(5, 7, nb, K, m) for nb, K in ((4, 4), (8, 8), (8, 3)) for m in (0, 1, 2)]
    np.testing.assert_array_equal(got, golden["act_flops"])
    assert O.activation_flops(1, 1, 4, 4, 1) == 37  # tests/test_activation.py:241-243
    assert O.conv_flops(1, 1, 1, 1, 1, (1, 1)) == 36  # tests/test_conv.py:213-215


def test_mvtf_bytes(golden):
    raw = O.mvtf_encode(golden["mvtf_arr"], tag=1, k=2)
    assert raw == golden["mvtf_bytes"].tobytes()
    data, tag, k = O.mvtf_decode(raw)
    np.testing.assert_array_equal(data, golden["mvtf_arr"])
    assert (tag, k) == (1, 2)


def test_linear_oracle_matches_reference(golden):
    for n in range(int(golden["lin_count"])):
        g = tuple(int(v) for v in golden[f"lin{n}_g"])
        x, w, b = golden[f"lin{n}_x"], golden[f"lin{n}_w"], golden[f"lin{n}_b"]
        y = O.linear_ref(x, w, b, g)
        np.testing.assert_allclose(y, golden[f"lin{n}_y"], rtol=2e-7, atol=1e-9)
        assert O.max_rel_error(y, golden[f"lin{n}_y_gemm"]) <= 1e-4
        assert O.linear_flops(x.shape[0], x.shape[1], w.shape[1], g) == int(golden[f"lin{n}_flops"])
