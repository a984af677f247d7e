"""Pins for oracle/tensor_ops.py (O1) against closed forms, brute force and library routines."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import tensor_ops as T

RNG = np.random.default_rng(11)


@pytest.mark.parametrize("cin,cout,h,w,kh,kw,sh,sw,ph,pw", [
    (3, 4, 7, 6, 3, 3, 1, 1, 1, 1),
    (2, 3, 9, 9, 3, 3, 2, 2, 0, 0),
    (4, 2, 8, 8, 1, 7, 1, 1, 0, 3),
    (4, 2, 8, 8, 7, 1, 1, 1, 3, 0),
    (2, 2, 7, 7, 5, 5, 1, 1, 2, 2),
    (3, 5, 6, 6, 1, 1, 2, 2, 0, 0),
    (2, 3, 9, 8, 3, 3, 2, 2, 1, 1),
])
def test_conv_tapshift_equals_literal_loops(cin, cout, h, w, kh, kw, sh, sw, ph, pw):
    x = RNG.standard_normal((2, cin, h, w))
    wt = RNG.standard_normal((cout, cin, kh, kw))
    b = RNG.standard_normal(cout)
    y1 = T.conv2d(x, wt, b, sh, sw, ph, pw)
    y2 = T.conv2d_loops(x, wt, b, sh, sw, ph, pw)
    np.testing.assert_allclose(y1, y2, rtol=1e-12, atol=1e-12)


def test_conv_matches_torch_f64():
    for (k, s, p) in [((3, 3), 2, (0, 0)), ((1, 7), 1, (0, 3)), ((5, 5), 1, (2, 2)), ((7, 7), 2, (0, 0))]:
        x = RNG.standard_normal((1, 5, 17, 15))
        wt = RNG.standard_normal((6, 5) + k)
        b = RNG.standard_normal(6)
        y = T.conv2d(x, wt, b, s, s, p[0], p[1])
        ref = F.conv2d(torch.from_numpy(x), torch.from_numpy(wt), torch.from_numpy(b), stride=s, padding=p).numpy()
        np.testing.assert_allclose(y, ref, rtol=1e-11, atol=1e-11)


def test_conv_1x1_is_matmul():
    x = RNG.standard_normal((1, 9, 5, 4))
    wt = RNG.standard_normal((7, 9, 1, 1))
    y = T.conv2d(x, wt, None, 1, 1, 0, 0)
    ref = (wt[:, :, 0, 0] @ x[0].reshape(9, -1)).reshape(7, 5, 4)
    np.testing.assert_allclose(y[0], ref, rtol=1e-12, atol=1e-12)


def test_conv_delta_kernel_is_shift():
    x = RNG.standard_normal((1, 1, 6, 6))
    wt = np.zeros((1, 1, 3, 3))
    wt[0, 0, 2, 0] = 1.0                       # y[oh, ow] = x[oh - 1 + 2, ow - 1 + 0]
    y = T.conv2d(x, wt, None, 1, 1, 1, 1)[0, 0]
    ref = np.zeros((6, 6))
    ref[:5, 1:] = x[0, 0, 1:, :5]
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("h,k,s,p,ceil", [(109, 3, 2, 0, True), (54, 3, 2, 0, True), (27, 3, 2, 0, True),
                                          (35, 3, 2, 0, False), (42, 3, 2, 1, False), (21, 3, 2, 1, False),
                                          (10, 3, 2, 1, True), (8, 2, 2, 1, True)])
def test_out_size_matches_torch(h, k, s, p, ceil):
    ref = F.max_pool2d(torch.zeros(1, 1, h, h), k, s, p, ceil_mode=ceil).shape[-1]
    assert T.out_size(h, k, s, p, ceil) == ref


@pytest.mark.parametrize("k,s,p,ceil", [(3, 2, 0, True), (3, 2, 0, False), (3, 1, 1, False), (3, 2, 1, False),
                                        (2, 2, 1, True)])
def test_maxpool_matches_torch(k, s, p, ceil):
    x = RNG.standard_normal((1, 3, 11, 10))
    y = T.maxpool2d(x, k, s, p, ceil)
    ref = F.max_pool2d(torch.from_numpy(x), k, s, p, ceil_mode=ceil).numpy()
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("k,s,p,inc,ceil", [(3, 1, 1, True, False), (3, 1, 1, False, False), (3, 2, 1, False, False),
                                            (3, 2, 1, True, False), (3, 2, 1, True, True), (3, 2, 1, False, True)])
def test_avgpool_matches_torch(k, s, p, inc, ceil):
    x = RNG.standard_normal((1, 3, 11, 10))
    y = T.avgpool2d(x, k, s, p, inc, ceil)
    ref = F.avg_pool2d(torch.from_numpy(x), k, s, p, ceil_mode=ceil, count_include_pad=inc).numpy()
    np.testing.assert_allclose(y, ref, rtol=1e-13, atol=1e-13)


def test_avgpool_constant_closed_forms():
    x = np.full((1, 2, 5, 5), 3.0)
    ex = T.avgpool2d(x, 3, 1, 1, count_include_pad=False)
    assert np.all(ex == 3.0)                                    # exclude-pad mean of a constant
    inc = T.avgpool2d(x, 3, 1, 1, count_include_pad=True)
    assert inc[0, 0, 0, 0] == pytest.approx(3.0 * 4 / 9)       # corner: 4 of 9 taps inside
    assert inc[0, 0, 0, 2] == pytest.approx(3.0 * 6 / 9)       # edge: 6 of 9
    assert inc[0, 0, 2, 2] == 3.0


def test_sepconv_matches_torch_depthwise_pointwise():
    c, cout, k, s = 6, 5, 5, 2
    xs = [RNG.standard_normal((1, c, 9, 9)) for _ in range(2)]
    aw = np.array([0.25, 0.75])
    wd = RNG.standard_normal((c, k, k))
    wp = RNG.standard_normal((cout, c))
    b = RNG.standard_normal(cout)
    y = T.sepconv(xs, np.concatenate([wd.ravel(), wp.ravel()]), b, cout, k, s, k // 2, aw)
    agg = torch.relu(torch.from_numpy(0.25 * xs[0] + 0.75 * xs[1]))
    d = F.conv2d(agg, torch.from_numpy(wd[:, None]), stride=s, padding=k // 2, groups=c)
    ref = F.conv2d(d, torch.from_numpy(wp[:, :, None, None]), torch.from_numpy(b)).numpy()
    np.testing.assert_allclose(y, ref, rtol=1e-11, atol=1e-11)


def test_add_concat_linear_gap_closed_forms():
    a, b = RNG.standard_normal((1, 4, 3, 3)), RNG.standard_normal((1, 4, 3, 3))
    assert np.array_equal(T.add([a, b]), a + b)
    np.testing.assert_allclose(T.add([a, b], np.array([2.0, -1.0])), 2 * a - b, rtol=0, atol=1e-15)
    c = T.concat([a, b])
    assert c.shape == (1, 8, 3, 3) and np.array_equal(c[:, 4:], b)
    g = T.global_avgpool(np.arange(18.0).reshape(1, 2, 3, 3))
    assert g[0, 0, 0, 0] == 4.0 and g[0, 1, 0, 0] == 13.0
    w = RNG.standard_normal((3, 8))
    bb = RNG.standard_normal(3)
    y = T.linear(c[:, :, :1, :1], w, bb)
    np.testing.assert_allclose(y[0, :, 0, 0], w @ c[0, :, 0, 0] + bb, rtol=1e-12)
