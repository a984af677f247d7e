"""O1: tensor semantics of the schedule units, float64, NCHW (TEST INFRASTRUCTURE ONLY).

The paper's units are "Conv-Relu" and "Relu-SepConv" plus Concat/pool/add; BN is
folded into the bias (Z9/Z12). Each function writes the textbook definition out.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np


def out_size(h: int, k: int, s: int, p: int, ceil_mode: bool = False) -> int:
    """Ho = floor((H + 2p - k)/s) + 1; with ceil_mode, ceil(...) + 1, minus one when the last
    window would start in the right padding (the torch rule, Z11)."""
    if not ceil_mode:
        return (h + 2 * p - k) // s + 1
    o = -(-(h + 2 * p - k) // s) + 1
    if (o - 1) * s >= h + p:
        o -= 1
    return o


def relu(x: np.ndarray) -> np.ndarray:
    return np.maximum(x, 0.0)


def conv2d_loops(x, w, b, sh, sw, ph, pw):
    """Literal 7-loop definition; tiny shapes only. Used to pin ``conv2d``.
    y[n,co,oh,ow] = b[co] + sum_{ci,i,j} W[co,ci,i,j] * x[n,ci,oh*sh-ph+i, ow*sw-pw+j], x=0 outside."""
    n_, cin, h, wd = x.shape
    cout, _, kh, kw = w.shape
    ho, wo = out_size(h, kh, sh, ph), out_size(wd, kw, sw, pw)
    y = np.zeros((n_, cout, ho, wo))
    for n in range(n_):
        for co in range(cout):
            for oh in range(ho):
                for ow in range(wo):
                    acc = float(b[co]) if b is not None else 0.0
                    for ci in range(cin):
                        for i in range(kh):
                            for j in range(kw):
                                ih, iw = oh * sh - ph + i, ow * sw - pw + j
                                if 0 <= ih < h and 0 <= iw < wd:
                                    acc += float(w[co, ci, i, j]) * float(x[n, ci, ih, iw])
                    y[n, co, oh, ow] = acc
    return y


def conv2d(x: np.ndarray, w: np.ndarray, b: Optional[np.ndarray], sh: int, sw: int, ph: int, pw: int,
           ho: Optional[int] = None, wo: Optional[int] = None, ph_hi: Optional[int] = None,
           pw_hi: Optional[int] = None) -> np.ndarray:
    """Tap-shift form of the same sum: y += W[:,:,i,j] @ shifted(x) for every tap (i, j).
    The per-tap product is an un-optimised ``einsum`` whose reduction over ci runs in a fixed order
    for every output channel, so a row's value does not depend on how many rows are computed
    together (this is what makes merged == unmerged exact, tests/test_oracle_graph.py).
    Optional (ho, wo, ph_hi, pw_hi) give an explicit output size / right padding, which the merged
    convolution's bounding-box kernel needs (Z4)."""
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    n, cin, h, wd = x.shape
    cout, cin_w, kh, kw = w.shape
    assert cin == cin_w, (cin, cin_w)
    if ho is None:
        ho = out_size(h, kh, sh, ph)
    if wo is None:
        wo = out_size(wd, kw, sw, pw)
    ph_hi = ph + kh if ph_hi is None else ph_hi
    pw_hi = pw + kw if pw_hi is None else pw_hi
    xp = np.zeros((n, cin, h + ph + ph_hi, wd + pw + pw_hi))
    xp[:, :, ph:ph + h, pw:pw + wd] = x
    y = np.zeros((n, cout, ho * wo))
    for i in range(kh):
        for j in range(kw):
            xs = xp[:, :, i:i + sh * (ho - 1) + 1:sh, j:j + sw * (wo - 1) + 1:sw].reshape(n, cin, ho * wo)
            y += np.einsum('oc,ncp->nop', w[:, :, i, j], xs)
    y = y.reshape(n, cout, ho, wo)
    if b is not None:
        y = y + np.asarray(b, dtype=np.float64)[None, :, None, None]
    return y


def depthwise2d(x: np.ndarray, wd: np.ndarray, s: int, p: int) -> np.ndarray:
    """d[n,c,oh,ow] = sum_{i,j} Wd[c,i,j] * x[n,c,oh*s-p+i, ow*s-p+j] (x = 0 outside)."""
    n, c, h, w = x.shape
    k = wd.shape[1]
    ho, wo = out_size(h, k, s, p), out_size(w, k, s, p)
    xp = np.zeros((n, c, h + 2 * p + k, w + 2 * p + k))
    xp[:, :, p:p + h, p:p + w] = x
    y = np.zeros((n, c, ho, wo))
    for i in range(k):
        for j in range(k):
            y += wd[None, :, i, j, None, None] * xp[:, :, i:i + s * (ho - 1) + 1:s, j:j + s * (wo - 1) + 1:s]
    return y


def sepconv(xs: Sequence[np.ndarray], weight: np.ndarray, bias: np.ndarray, cout: int, k: int, s: int, p: int,
            add_weights: Optional[np.ndarray] = None, relu_post: bool = False) -> np.ndarray:
    """Relu-SepConv: x' = ReLU(sum_i w_i x_i); d = depthwise_kxk(x'); y = Wp d + b."""
    agg = _weighted_sum(xs, add_weights)
    c = agg.shape[1]
    weight = np.asarray(weight, dtype=np.float64)
    wd = weight[:c * k * k].reshape(c, k, k)
    wp = weight[c * k * k:].reshape(cout, c)
    d = depthwise2d(relu(agg), wd, s, p)
    n, _, ho, wo = d.shape
    y = np.matmul(wp, d.reshape(n, c, ho * wo)).reshape(n, cout, ho, wo)
    y = y + np.asarray(bias, dtype=np.float64)[None, :, None, None]
    return relu(y) if relu_post else y


def maxpool2d(x: np.ndarray, k: int, s: int, p: int, ceil_mode: bool = False) -> np.ndarray:
    """Max over the window intersected with the input (padding = -inf)."""
    n, c, h, w = x.shape
    ho, wo = out_size(h, k, s, p, ceil_mode), out_size(w, k, s, p, ceil_mode)
    xp = np.full((n, c, h + 2 * p + k + s, w + 2 * p + k + s), -np.inf)
    xp[:, :, p:p + h, p:p + w] = x
    y = np.full((n, c, ho, wo), -np.inf)
    for i in range(k):
        for j in range(k):
            y = np.maximum(y, xp[:, :, i:i + s * (ho - 1) + 1:s, j:j + s * (wo - 1) + 1:s])
    return y


def avgpool2d(x: np.ndarray, k: int, s: int, p: int, count_include_pad: bool = True,
              ceil_mode: bool = False) -> np.ndarray:
    """Window sum / divisor; divisor = window size clipped to the padded input (include_pad) or to
    the input itself (exclude_pad), per output position (the torch definition, Z11)."""
    n, c, h, w = x.shape
    ho, wo = out_size(h, k, s, p, ceil_mode), out_size(w, k, s, p, ceil_mode)
    y = np.zeros((n, c, ho, wo))
    for oh in range(ho):
        hs = oh * s - p
        he = min(hs + k, h + p)
        hsz = he - hs
        h0, h1 = max(hs, 0), min(he, h)
        for ow in range(wo):
            ws = ow * s - p
            we = min(ws + k, w + p)
            wsz = we - ws
            w0, w1 = max(ws, 0), min(we, w)
            div = hsz * wsz if count_include_pad else (h1 - h0) * (w1 - w0)
            y[:, :, oh, ow] = x[:, :, h0:h1, w0:w1].sum(axis=(2, 3)) / div
    return y


def global_avgpool(x: np.ndarray, relu_pre: bool = False) -> np.ndarray:
    x = relu(x) if relu_pre else x
    return x.mean(axis=(2, 3), keepdims=True)


def _weighted_sum(xs: Sequence[np.ndarray], weights: Optional[np.ndarray]) -> np.ndarray:
    if weights is None:
        weights = np.ones(len(xs))
    acc = np.zeros(np.asarray(xs[0]).shape)
    for wi, xi in zip(weights, xs):
        acc = acc + float(wi) * np.asarray(xi, dtype=np.float64)
    return acc


def add(xs: Sequence[np.ndarray], weights: Optional[np.ndarray] = None) -> np.ndarray:
    """sum_i w_i x_i (NASNet combinations; RandWire sigma(w)-weighted aggregation)."""
    return _weighted_sum(xs, weights)


def concat(xs: Sequence[np.ndarray]) -> np.ndarray:
    """Concatenation along C, in input order."""
    return np.concatenate([np.asarray(v, dtype=np.float64) for v in xs], axis=1)


def linear(x: np.ndarray, w: np.ndarray, b: np.ndarray, relu_post: bool = False) -> np.ndarray:
    """FC head as a 1x1 conv on the flattened input: y = W x + b."""
    n = x.shape[0]
    xf = np.asarray(x, dtype=np.float64).reshape(n, -1)
    y = xf @ np.asarray(w, dtype=np.float64).T + np.asarray(b, dtype=np.float64)[None, :]
    y = y.reshape(n, -1, 1, 1)
    return relu(y) if relu_post else y
