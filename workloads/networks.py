"""Network builders for BASELINE.json's configs (Table 2; Fig. 2).

The paper names the networks only. Topologies follow the public definitions, with the readings
listed in DESIGN.md (Z9 schedule units, Z10 blocks, Z11 pooling conventions, Z17 Fig. 2 shapes):

* ``fig2_block``   Z17: x[1,64,28,28]; a 3x3 64->128, b 3x3 128->64 on a, c 1x1 64->64, d 3x3 64->96.
* ``inception_v3`` torchvision topology, Mixed_5b..Mixed_7c = 11 blocks (+ stem and head blocks).
* ``squeezenet``   v1.0, one block per fire module, max pools with ceil_mode.
* ``nasnet_a_large`` 331x331, F=168, 6 normal cells per stage, one block per cell.
* ``randwire_ws_small`` WS(K=4, P=0.75), N=32 nodes per random stage, C=78.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Sequence

import numpy as np

from .netspec import NetBuilder, NetSpec


# --------------------------------------------------------------------------------------------
# Fig. 2 / Fig. 5 / small test graphs
# --------------------------------------------------------------------------------------------

def fig2_block(seed: int = 2, batch: int = 1, math: str = "tf32") -> NetSpec:
    """Fig. 2 4-conv block; shapes per DESIGN.md Z17. Block 0 = {a, b, c, d}; block 1 = concat."""
    nb = NetBuilder("fig2", (batch, 64, 28, 28), seed, math)
    a = nb.conv(0, 128, 3, 1, 1, name="a")
    nb.conv(a, 64, 3, 1, 1, name="b")
    nb.conv(0, 64, 1, 1, 0, name="c")
    nb.conv(0, 96, 3, 1, 1, name="d")
    nb.new_block()
    nb.concat([2, 3, 4], name="concat")
    return nb.net


def fig5_graph(seed: int = 5, batch: int = 1, math: str = "tf32") -> NetSpec:
    """Fig. 5 graph: a -> b, c independent; then a concat block."""
    nb = NetBuilder("fig5", (batch, 16, 8, 8), seed, math)
    a = nb.conv(0, 16, 3, 1, 1, name="a")
    nb.conv(a, 16, 1, 1, 0, name="b")
    nb.conv(0, 16, 1, 1, 0, name="c")
    nb.new_block()
    nb.concat([2, 3], name="concat")
    return nb.net


def tiny_mixed_net(seed: int = 7, batch: int = 1, math: str = "tf32", hw: int = 19) -> NetSpec:
    """Small graph exercising every op kind (parity tests; not a paper workload)."""
    nb = NetBuilder("tiny_mixed", (batch, 3, hw, hw), seed, math)
    s = nb.conv(0, 24, 3, 2, 1, name="stem")                     # Cin 3 -> padded channels
    nb.new_block()
    b1 = nb.conv(s, 16, 1, name="b1")
    b5 = nb.conv(s, 8, 1, name="b5_1")
    b5 = nb.conv(b5, 16, (1, 5), 1, (0, 2), name="b5_2")
    bp = nb.avgpool(s, 3, 1, 1, count_include_pad=True, name="pool")
    bp = nb.conv(bp, 8, 1, name="pool_proj")
    mp = nb.maxpool(s, 3, 1, 1, name="maxpool")
    cat = nb.concat([b1, b5, bp, mp], name="concat")          # 16+16+8+24 = 64
    nb.new_block()
    x1 = nb.conv(cat, 32, 1, relu=False, relu_pre=True, name="sq")
    sp = nb.sepconv(x1, 32, 3, 1, name="sep3")
    sp2 = nb.sepconv([x1, sp], 32, 5, 1, add_weights=[0.3, 0.7], name="sep5agg")
    ap = nb.avgpool(x1, 3, 1, 1, count_include_pad=False, name="avg_excl")
    ad = nb.add([sp2, ap, x1], name="add3")
    idn = nb.identity(ad, name="id")
    nb.new_block()
    r = nb.maxpool(idn, 3, 2, 0, ceil_mode=True, name="maxpool_ceil")
    g = nb.gavgpool(r, name="gap")
    nb.linear(g, 10, name="fc")
    return nb.net


def conv_zoo_net(seed: int = 11, batch: int = 1, math: str = "tf32", hw: int = 37, cin: int = 48) -> NetSpec:
    """Conv shape zoo (parity tests of the im2col paths; not a paper workload): square / asymmetric
    kernels, strides 1-3, zero and non-zero padding, chained convs and one mergeable group."""
    nb = NetBuilder("conv_zoo", (batch, cin, hw, hw), seed, math)
    nb.new_block()
    a = nb.conv(0, 48, 3, 1, 1, name="k3s1p1")
    nb.conv(0, 40, 3, 2, 0, name="k3s2p0")
    nb.conv(0, 32, 5, 1, 2, name="k5s1p2")
    d = nb.conv(0, 48, (1, 7), 1, (0, 3), name="k1x7")
    nb.conv(d, 40, (7, 1), 1, (3, 0), name="k7x1")
    nb.conv(0, 64, 3, 2, 1, name="k3s2p1")
    nb.conv(0, 24, 3, 3, 1, name="k3s3p1")
    nb.conv(0, 16, 7, 2, 3, name="k7s2p3")
    nb.conv(a, 56, 3, 1, 1, relu=False, name="chain")
    nb.conv(a, 24, 1, 1, 0, name="k1")
    nb.conv(0, 40, 2, 1, 0, name="k2s1p0")
    nb.new_block()
    m1 = nb.conv(a, 32, 3, 1, 1, name="m3")
    m2 = nb.conv(a, 32, 1, 1, 0, name="m1")
    m3 = nb.conv(a, 16, 5, 1, 2, name="m5")
    nb.concat([m1, m2, m3], name="cat")
    return nb.net


def sepconv_zoo_net(seed: int = 13, batch: int = 1, math: str = "tf32", hw: int = 37, cin: int = 40) -> NetSpec:
    """Relu-SepConv shape zoo (parity tests of the fused depthwise->pointwise GEMM; not
    a paper workload): k in {3, 5, 7} x stride {1, 2}, a channel count that leaves a partial K chunk,
    weighted multi-input aggregation (negative weights: the ReLU follows the sum), Cout > 256 (two
    N tiles), a sepconv chain and a post-ReLU unit."""
    nb = NetBuilder("sepconv_zoo", (batch, cin, hw, hw), seed, math)
    nb.new_block()
    x1 = nb.conv(0, cin, 1, relu=False, name="pre")
    nb.sepconv(0, 48, 3, 1, name="k3s1")
    nb.sepconv(0, 40, 3, 2, name="k3s2")
    s5 = nb.sepconv(0, 56, 5, 1, name="k5s1")
    nb.sepconv(0, 24, 5, 2, name="k5s2")
    nb.sepconv(0, 32, 7, 1, name="k7s1")
    nb.sepconv(0, 40, 7, 2, name="k7s2")
    nb.sepconv([0, x1], 40, 3, 1, add_weights=[0.5, -0.8], name="agg2")
    nb.sepconv([x1, 0, x1], 32, 5, 2, add_weights=[1.3, 0.4, -0.2], name="agg3s2")
    nb.sepconv(s5, 48, 3, 1, relu_post=True, name="chain")
    nb.sepconv(0, 300, 3, 1, name="wide")
    return nb.net


# --------------------------------------------------------------------------------------------
# Inception V3 (torchvision topology; Conv-Relu units, BN folded into bias)
# --------------------------------------------------------------------------------------------

def _inception_a(nb: NetBuilder, x: int, pool_features: int, tag: str) -> int:
    nb.new_block()
    b1 = nb.conv(x, 64, 1, name=f"{tag}.b1x1")
    b5 = nb.conv(x, 48, 1, name=f"{tag}.b5x5_1")
    b5 = nb.conv(b5, 64, 5, 1, 2, name=f"{tag}.b5x5_2")
    bd = nb.conv(x, 64, 1, name=f"{tag}.b3x3dbl_1")
    bd = nb.conv(bd, 96, 3, 1, 1, name=f"{tag}.b3x3dbl_2")
    bd = nb.conv(bd, 96, 3, 1, 1, name=f"{tag}.b3x3dbl_3")
    bp = nb.avgpool(x, 3, 1, 1, count_include_pad=True, name=f"{tag}.pool")
    bp = nb.conv(bp, pool_features, 1, name=f"{tag}.bpool")
    return nb.concat([b1, b5, bd, bp], name=f"{tag}.concat")


def _inception_b(nb: NetBuilder, x: int, tag: str) -> int:
    nb.new_block()
    b3 = nb.conv(x, 384, 3, 2, 0, name=f"{tag}.b3x3")
    bd = nb.conv(x, 64, 1, name=f"{tag}.b3x3dbl_1")
    bd = nb.conv(bd, 96, 3, 1, 1, name=f"{tag}.b3x3dbl_2")
    bd = nb.conv(bd, 96, 3, 2, 0, name=f"{tag}.b3x3dbl_3")
    bp = nb.maxpool(x, 3, 2, 0, name=f"{tag}.pool")
    return nb.concat([b3, bd, bp], name=f"{tag}.concat")


def _inception_c(nb: NetBuilder, x: int, c7: int, tag: str) -> int:
    nb.new_block()
    b1 = nb.conv(x, 192, 1, name=f"{tag}.b1x1")
    b7 = nb.conv(x, c7, 1, name=f"{tag}.b7x7_1")
    b7 = nb.conv(b7, c7, (1, 7), 1, (0, 3), name=f"{tag}.b7x7_2")
    b7 = nb.conv(b7, 192, (7, 1), 1, (3, 0), name=f"{tag}.b7x7_3")
    bd = nb.conv(x, c7, 1, name=f"{tag}.b7x7dbl_1")
    bd = nb.conv(bd, c7, (7, 1), 1, (3, 0), name=f"{tag}.b7x7dbl_2")
    bd = nb.conv(bd, c7, (1, 7), 1, (0, 3), name=f"{tag}.b7x7dbl_3")
    bd = nb.conv(bd, c7, (7, 1), 1, (3, 0), name=f"{tag}.b7x7dbl_4")
    bd = nb.conv(bd, 192, (1, 7), 1, (0, 3), name=f"{tag}.b7x7dbl_5")
    bp = nb.avgpool(x, 3, 1, 1, count_include_pad=True, name=f"{tag}.pool")
    bp = nb.conv(bp, 192, 1, name=f"{tag}.bpool")
    return nb.concat([b1, b7, bd, bp], name=f"{tag}.concat")


def _inception_d(nb: NetBuilder, x: int, tag: str) -> int:
    nb.new_block()
    b3 = nb.conv(x, 192, 1, name=f"{tag}.b3x3_1")
    b3 = nb.conv(b3, 320, 3, 2, 0, name=f"{tag}.b3x3_2")
    b7 = nb.conv(x, 192, 1, name=f"{tag}.b7x7x3_1")
    b7 = nb.conv(b7, 192, (1, 7), 1, (0, 3), name=f"{tag}.b7x7x3_2")
    b7 = nb.conv(b7, 192, (7, 1), 1, (3, 0), name=f"{tag}.b7x7x3_3")
    b7 = nb.conv(b7, 192, 3, 2, 0, name=f"{tag}.b7x7x3_4")
    bp = nb.maxpool(x, 3, 2, 0, name=f"{tag}.pool")
    return nb.concat([b3, b7, bp], name=f"{tag}.concat")


def _inception_e(nb: NetBuilder, x: int, tag: str) -> int:
    """Inception-E: 9 convs + pool + one concat = 11 ops, width 6 (Table 1 row 1: n=11, d=6)."""
    nb.new_block()
    b1 = nb.conv(x, 320, 1, name=f"{tag}.b1x1")
    b3 = nb.conv(x, 384, 1, name=f"{tag}.b3x3_1")
    b3a = nb.conv(b3, 384, (1, 3), 1, (0, 1), name=f"{tag}.b3x3_2a")
    b3b = nb.conv(b3, 384, (3, 1), 1, (1, 0), name=f"{tag}.b3x3_2b")
    bd = nb.conv(x, 448, 1, name=f"{tag}.b3x3dbl_1")
    bd = nb.conv(bd, 384, 3, 1, 1, name=f"{tag}.b3x3dbl_2")
    bda = nb.conv(bd, 384, (1, 3), 1, (0, 1), name=f"{tag}.b3x3dbl_3a")
    bdb = nb.conv(bd, 384, (3, 1), 1, (1, 0), name=f"{tag}.b3x3dbl_3b")
    bp = nb.avgpool(x, 3, 1, 1, count_include_pad=True, name=f"{tag}.pool")
    bp = nb.conv(bp, 192, 1, name=f"{tag}.bpool")
    return nb.concat([b1, b3a, b3b, bda, bdb, bp], name=f"{tag}.concat")


def inception_v3(seed: int = 3, batch: int = 1, math: str = "tf32", image: int = 299) -> NetSpec:
    nb = NetBuilder("inception_v3", (batch, 3, image, image), seed, math)
    x = nb.conv(0, 32, 3, 2, 0, name="Conv2d_1a_3x3")
    x = nb.conv(x, 32, 3, 1, 0, name="Conv2d_2a_3x3")
    x = nb.conv(x, 64, 3, 1, 1, name="Conv2d_2b_3x3")
    x = nb.maxpool(x, 3, 2, 0, name="maxpool1")
    x = nb.conv(x, 80, 1, name="Conv2d_3b_1x1")
    x = nb.conv(x, 192, 3, 1, 0, name="Conv2d_4a_3x3")
    x = nb.maxpool(x, 3, 2, 0, name="maxpool2")
    x = _inception_a(nb, x, 32, "Mixed_5b")
    x = _inception_a(nb, x, 64, "Mixed_5c")
    x = _inception_a(nb, x, 64, "Mixed_5d")
    x = _inception_b(nb, x, "Mixed_6a")
    x = _inception_c(nb, x, 128, "Mixed_6b")
    x = _inception_c(nb, x, 160, "Mixed_6c")
    x = _inception_c(nb, x, 160, "Mixed_6d")
    x = _inception_c(nb, x, 192, "Mixed_6e")
    x = _inception_d(nb, x, "Mixed_7a")
    x = _inception_e(nb, x, "Mixed_7b")
    x = _inception_e(nb, x, "Mixed_7c")
    nb.new_block()
    x = nb.gavgpool(x, name="avgpool")
    nb.linear(x, 1000, name="fc")
    return nb.net


# --------------------------------------------------------------------------------------------
# SqueezeNet 1.0
# --------------------------------------------------------------------------------------------

def _fire(nb: NetBuilder, x: int, sq: int, e1: int, e3: int, tag: str) -> int:
    nb.new_block()
    s = nb.conv(x, sq, 1, name=f"{tag}.squeeze")
    a = nb.conv(s, e1, 1, name=f"{tag}.expand1x1")
    b = nb.conv(s, e3, 3, 1, 1, name=f"{tag}.expand3x3")
    return nb.concat([a, b], name=f"{tag}.concat")


def squeezenet(seed: int = 4, batch: int = 1, math: str = "tf32", image: int = 224) -> NetSpec:
    nb = NetBuilder("squeezenet", (batch, 3, image, image), seed, math)
    x = nb.conv(0, 96, 7, 2, 0, name="conv1")
    x = nb.maxpool(x, 3, 2, 0, ceil_mode=True, name="pool1")
    x = _fire(nb, x, 16, 64, 64, "fire2")
    x = _fire(nb, x, 16, 64, 64, "fire3")
    x = _fire(nb, x, 32, 128, 128, "fire4")
    nb.new_block()
    x = nb.maxpool(x, 3, 2, 0, ceil_mode=True, name="pool4")
    x = _fire(nb, x, 32, 128, 128, "fire5")
    x = _fire(nb, x, 48, 192, 192, "fire6")
    x = _fire(nb, x, 48, 192, 192, "fire7")
    x = _fire(nb, x, 64, 256, 256, "fire8")
    nb.new_block()
    x = nb.maxpool(x, 3, 2, 0, ceil_mode=True, name="pool8")
    x = _fire(nb, x, 64, 256, 256, "fire9")
    nb.new_block()
    x = nb.conv(x, 1000, 1, name="conv10")
    nb.gavgpool(x, name="avgpool")
    return nb.net


# --------------------------------------------------------------------------------------------
# NASNet-A Large (Zoph et al. 2018; public "nasnetalarge" layout), Relu-SepConv units
# --------------------------------------------------------------------------------------------

def _sep_pair(nb: NetBuilder, x: int, cout: int, k: int, s: int, tag: str) -> int:
    """NASNet "separable x2" = two Relu-SepConv units (Z9)."""
    y = nb.sepconv(x, cout, k, s, k // 2, name=f"{tag}.sep1")
    return nb.sepconv(y, cout, k, 1, k // 2, name=f"{tag}.sep2")


def _adjust(nb: NetBuilder, x_prev: int, prev_hw: int, hw: int, f: int, tag: str) -> int:
    """ReLU -> 1x1 conv (-> BN) on h_{i-1}; factorized reduction when its resolution is 2x (two
    stride-2 1x1 paths, the second shifted by one pixel, expressed as a 3x3 s2 p1 conv whose only
    non-zero tap is (2, 2))."""
    if prev_hw == hw:
        return nb.conv(x_prev, f, 1, relu=False, relu_pre=True, name=f"{tag}.conv_prev_1x1")
    p1 = nb.conv(x_prev, f // 2, 1, 2, 0, relu=False, relu_pre=True, name=f"{tag}.fr_path1")
    p2 = nb.conv(x_prev, f - f // 2, 3, 2, 1, relu=False, relu_pre=True, name=f"{tag}.fr_path2")
    w = nb.net.ops[p2 - 1].weight
    w[:, :, :2, :] = 0.0
    w[:, :, :, :2] = 0.0
    return nb.concat([p1, p2], name=f"{tag}.fr_concat")


def _normal_cell(nb: NetBuilder, x: int, x_prev: int, hw: int, prev_hw: int, f: int, tag: str) -> int:
    nb.new_block()
    h = _adjust(nb, x_prev, prev_hw, hw, f, tag)
    xx = nb.conv(x, f, 1, relu=False, relu_pre=True, name=f"{tag}.conv_1x1")
    c0 = nb.add([_sep_pair(nb, xx, f, 5, 1, f"{tag}.c0l"), _sep_pair(nb, h, f, 3, 1, f"{tag}.c0r")], name=f"{tag}.c0")
    c1 = nb.add([_sep_pair(nb, h, f, 5, 1, f"{tag}.c1l"), _sep_pair(nb, h, f, 3, 1, f"{tag}.c1r")], name=f"{tag}.c1")
    c2 = nb.add([nb.avgpool(xx, 3, 1, 1, count_include_pad=False, name=f"{tag}.c2l"), h], name=f"{tag}.c2")
    c3 = nb.add([nb.avgpool(h, 3, 1, 1, count_include_pad=False, name=f"{tag}.c3l"),
                 nb.avgpool(h, 3, 1, 1, count_include_pad=False, name=f"{tag}.c3r")], name=f"{tag}.c3")
    c4 = nb.add([_sep_pair(nb, xx, f, 3, 1, f"{tag}.c4l"), xx], name=f"{tag}.c4")
    return nb.concat([h, c0, c1, c2, c3, c4], name=f"{tag}.concat")


def _reduction_cell(nb: NetBuilder, x: int, x_prev: int, hw: int, prev_hw: int, f: int, tag: str) -> int:
    nb.new_block()
    h = _adjust(nb, x_prev, prev_hw, hw, f, tag)
    xx = nb.conv(x, f, 1, relu=False, relu_pre=True, name=f"{tag}.conv_1x1")
    c0 = nb.add([_sep_pair(nb, xx, f, 5, 2, f"{tag}.c0l"), _sep_pair(nb, h, f, 7, 2, f"{tag}.c0r")], name=f"{tag}.c0")
    c1 = nb.add([nb.maxpool(xx, 3, 2, 1, name=f"{tag}.c1l"), _sep_pair(nb, h, f, 7, 2, f"{tag}.c1r")], name=f"{tag}.c1")
    c2 = nb.add([nb.avgpool(xx, 3, 2, 1, count_include_pad=False, name=f"{tag}.c2l"),
                 _sep_pair(nb, h, f, 5, 2, f"{tag}.c2r")], name=f"{tag}.c2")
    c3 = nb.add([nb.avgpool(c0, 3, 1, 1, count_include_pad=False, name=f"{tag}.c3l"), c1], name=f"{tag}.c3")
    c4 = nb.add([nb.sepconv(c0, f, 3, 1, 1, name=f"{tag}.c4l"), nb.maxpool(xx, 3, 2, 1, name=f"{tag}.c4r")],
                name=f"{tag}.c4")
    return nb.concat([c1, c2, c3, c4], name=f"{tag}.concat")


def nasnet_a_large(seed: int = 6, batch: int = 1, math: str = "tf32", image: int = 331,
                   penultimate_filters: int = 4032, cells_per_stage: int = 6) -> NetSpec:
    """22 cells: 2 stem cells (read as reduction cells, Z10), 3 x 6 normal cells and 2
    reduction cells; F = 4032 / 24 = 168; one DP block per cell."""
    nb = NetBuilder("nasnet_a_large", (batch, 3, image, image), seed, math)
    f = penultimate_filters // 24                   # 168
    stem = nb.conv(0, 96, 3, 2, 0, relu=False, name="conv0")
    hw0 = (image - 3) // 2 + 1                      # 165
    hw1 = (hw0 - 1) // 2 + 1                        # 83
    hw2 = (hw1 - 1) // 2 + 1                        # 42
    nb.new_block()                                  # cell_stem_0: both inputs are the stem output
    xx0 = nb.conv(stem, f // 4, 1, relu=False, relu_pre=True, name="cell_stem_0.conv_1x1")
    s0 = _reduction_body(nb, xx0, stem, f // 4, "cell_stem_0")
    nb.new_block()                                  # cell_stem_1: h_{i-1} = stem (2x resolution)
    h1 = _adjust(nb, stem, hw0, hw1, f // 2, "cell_stem_1")
    xx1 = nb.conv(s0, f // 2, 1, relu=False, relu_pre=True, name="cell_stem_1.conv_1x1")
    s1 = _reduction_body(nb, xx1, h1, f // 2, "cell_stem_1")
    prev, cur, prev_hw, cur_hw = s0, s1, hw1, hw2
    filters = f
    for stage in range(3):
        if stage > 0:
            filters *= 2
            nxt_hw = (cur_hw - 1) // 2 + 1
            red = _reduction_cell(nb, cur, prev, cur_hw, prev_hw, filters, f"reduction_cell_{stage - 1}")
            prev, cur, prev_hw, cur_hw = cur, red, cur_hw, nxt_hw
        for i in range(cells_per_stage):
            nc = _normal_cell(nb, cur, prev, cur_hw, prev_hw, filters, f"cell_{stage * cells_per_stage + i}")
            prev, cur, prev_hw = cur, nc, cur_hw
    nb.new_block()
    g = nb.gavgpool(cur, relu_pre=True, name="avgpool")
    nb.linear(g, 1000, name="last_linear")
    return nb.net


def _reduction_body(nb: NetBuilder, xx: int, h_src: int, f: int, tag: str) -> int:
    """Stem-cell body: the reduction-cell combinations over (xx, h) where h = xx for cell_stem_0."""
    h = h_src
    if nb.ch[h] != f:
        h = nb.conv(h, f, 1, relu=False, relu_pre=True, name=f"{tag}.h_1x1")
    c0 = nb.add([_sep_pair(nb, xx, f, 5, 2, f"{tag}.c0l"), _sep_pair(nb, h, f, 7, 2, f"{tag}.c0r")], name=f"{tag}.c0")
    c1 = nb.add([nb.maxpool(xx, 3, 2, 1, name=f"{tag}.c1l"), _sep_pair(nb, h, f, 7, 2, f"{tag}.c1r")], name=f"{tag}.c1")
    c2 = nb.add([nb.avgpool(xx, 3, 2, 1, count_include_pad=False, name=f"{tag}.c2l"),
                 _sep_pair(nb, h, f, 5, 2, f"{tag}.c2r")], name=f"{tag}.c2")
    c3 = nb.add([nb.avgpool(c0, 3, 1, 1, count_include_pad=False, name=f"{tag}.c3l"), c1], name=f"{tag}.c3")
    c4 = nb.add([nb.sepconv(c0, f, 3, 1, 1, name=f"{tag}.c4l"), nb.maxpool(xx, 3, 2, 1, name=f"{tag}.c4r")],
                name=f"{tag}.c4")
    return nb.concat([c1, c2, c3, c4], name=f"{tag}.concat")


# --------------------------------------------------------------------------------------------
# RandWire-WS, small regime (Xie et al. 2019), Relu-SepConv nodes with weighted aggregation
# --------------------------------------------------------------------------------------------

def _ws_dag(n: int, k: int, p: float, rng: np.random.Generator) -> List[List[int]]:
    """Watts-Strogatz ring lattice (k neighbours) with rewiring probability p, oriented low -> high
    index. Returns predecessor lists. (Input generation: topology only.)"""
    adj = [set() for _ in range(n)]
    for i in range(n):
        for j in range(1, k // 2 + 1):
            a, b = i, (i + j) % n
            adj[a].add(b)
            adj[b].add(a)
    for j in range(1, k // 2 + 1):
        for i in range(n):
            b = (i + j) % n
            if rng.random() < p and b in adj[i]:
                choices = [c for c in range(n) if c != i and c not in adj[i]]
                if choices:
                    c = choices[int(rng.integers(len(choices)))]
                    adj[i].discard(b)
                    adj[b].discard(i)
                    adj[i].add(c)
                    adj[c].add(i)
    return [sorted(u for u in adj[v] if u < v) for v in range(n)]


def _random_stage(nb: NetBuilder, x: int, cout: int, n: int, rng: np.random.Generator, tag: str) -> int:
    preds = _ws_dag(n, 4, 0.75, rng)
    succ_count = [0] * n
    for v in range(n):
        for u in preds[v]:
            succ_count[u] += 1
    nb.new_block()
    node_out: Dict[int, int] = {}
    for v in range(n):
        if not preds[v]:
            node_out[v] = nb.sepconv(x, cout, 3, 2, 1, name=f"{tag}.node{v}")
        else:
            ins = [node_out[u] for u in preds[v]]
            w = 1.0 / (1.0 + np.exp(-rng.standard_normal(len(ins))))       # sigma(w) aggregation weights
            node_out[v] = nb.sepconv(ins, cout, 3, 1, 1, add_weights=w if len(ins) > 1 else None,
                                     name=f"{tag}.node{v}")
    outs = [node_out[v] for v in range(n) if succ_count[v] == 0]
    if len(outs) == 1:
        return outs[0]
    return nb.add(outs, weights=[1.0 / len(outs)] * len(outs), name=f"{tag}.output_avg")


def randwire_ws_small(seed: int = 8, batch: int = 1, math: str = "bf16", image: int = 224,
                      channels: int = 78, nodes: int = 32) -> NetSpec:
    nb = NetBuilder("randwire_ws_small", (batch, 3, image, image), seed, math)
    rng = np.random.default_rng([seed, 0xD46])
    c = channels
    x = nb.conv(0, c // 2, 3, 2, 1, name="conv1")               # 112
    nb.new_block()
    x = nb.sepconv(x, c, 3, 2, 1, name="conv2")                  # 56
    x = _random_stage(nb, x, c, nodes, rng, "conv3")             # 28
    x = _random_stage(nb, x, 2 * c, nodes, rng, "conv4")         # 14
    x = _random_stage(nb, x, 4 * c, nodes, rng, "conv5")         # 7
    nb.new_block()
    x = nb.conv(x, 1280, 1, relu=True, relu_pre=True, name="classifier_conv")
    g = nb.gavgpool(x, name="avgpool")
    nb.linear(g, 1000, name="fc")
    return nb.net


NETWORKS: Dict[str, Callable[..., NetSpec]] = {
    "fig2": fig2_block,
    "fig5": fig5_graph,
    "tiny_mixed": tiny_mixed_net,
    "conv_zoo": conv_zoo_net,
    "sepconv_zoo": sepconv_zoo_net,
    "inception_v3": inception_v3,
    "squeezenet": squeezenet,
    "nasnet_a_large": nasnet_a_large,
    "randwire_ws_small": randwire_ws_small,
}


def build(name: str, **kw) -> NetSpec:
    return NETWORKS[name](**kw)
