"""Network driver parity on the GPU (BASELINE configs 2-4 graphs on small synthetic scenes).

Layer-wise with teacher forcing: every CONV op's GPU input tensor is fed to
the CPU oracle (same coordinates; features and weights rounded to the GPU operand type);
output coordinates must be bit-exact and features within 2e-6 of max|out| (only the
accumulation order differs); against the unrounded fp32 oracle the north_star tolerance
(max <= 1e-2, mean <= 1e-3) must hold per layer. ADD / CONCAT are checked exactly. The
end-to-end error through the whole graph is reported and bounded loosely.
"""
import numpy as np
import pytest

import paper_2401_06145_b200 as sc
from paper_2401_06145_b200 import datasets as D
from paper_2401_06145_b200 import network as N
from oracle_lib import load_oracle

pytestmark = pytest.mark.gpu


def f16(a):
    return a.astype(np.float16).astype(np.float32)


def rel(g, r):
    d = np.abs(g.astype(np.float64) - r.astype(np.float64))
    s = max(np.abs(r).max(), 1e-30)
    return d.max() / s, d.mean() / max(np.abs(r).mean(), 1e-30)


def teacher_forced(ctx, g, weights, coords, feats, max_convs=None):
    """fp32 partials (strict same-operand parity); the default f16-partial network is checked
    end to end in test_minkunet42_small_scan."""
    ora = load_oracle()
    net = N.Network(ctx, g, weights, sc.exec_cfg(partial_f16=0))
    net.forward(coords, feats, True)
    checked = 0
    worst = (0.0, 0.0)
    for o in g.ops:
        xin, fin = net.read(o.a)
        xout, fout = net.read(o.out)
        if o.kind == N.CONV:
            if max_convs is not None and checked >= max_convs:
                continue
            W = weights[o.weight]
            tgt = net.read(o.b)[0] if o.transposed else None
            oq, of, _ = ora.layer_forward(xin, True, f16(fin), f16(W), o.K, o.offset_scale, o.out_stride,
                                          bool(o.transposed), tgt, workers=8)
            if o.relu:
                of = np.maximum(of, 0)
            np.testing.assert_array_equal(xout, oq)
            mx, _ = rel(fout, of)
            assert mx <= 2e-6, (o, mx)
            _, of32, _ = ora.layer_forward(xin, True, fin, W, o.K, o.offset_scale, o.out_stride, bool(o.transposed),
                                           tgt, workers=8)
            if o.relu:
                of32 = np.maximum(of32, 0)
            mx, mean = rel(fout, of32)
            worst = (max(worst[0], mx), max(worst[1], mean))
            assert mx <= 1e-2 and mean <= 1e-3, (o, mx, mean)
            checked += 1
        elif o.kind == N.ADD:
            xb, fb = net.read(o.b)
            ref = fin + fb
            np.testing.assert_array_equal(fout, np.maximum(ref, 0) if o.relu else ref)
        else:
            xb, fb = net.read(o.b)
            np.testing.assert_array_equal(fout, np.concatenate([fin, fb], 1))
    return net, checked, worst


def oracle_graph(g, weights, coords, feats):
    """Whole graph on the CPU oracle (fp32 features, fp64 accumulation)."""
    ora = load_oracle()
    T = {g.input: (coords, feats)}
    for o in g.ops:
        xin, fin = T[o.a]
        if o.kind == N.CONV:
            tgt = T[o.b][0] if o.transposed else None
            q, f, _ = ora.layer_forward(xin, True, fin, weights[o.weight], o.K, o.offset_scale, o.out_stride,
                                        bool(o.transposed), tgt, workers=8)
            T[o.out] = (q, np.maximum(f, 0) if o.relu else f)
        elif o.kind == N.ADD:
            s = fin + T[o.b][1]
            T[o.out] = (xin, np.maximum(s, 0) if o.relu else s)
        else:
            T[o.out] = (xin, np.concatenate([fin, T[o.b][1]], 1))
    return T[g.output]


def test_minkunet42_small_scan(ctx):
    coords, feats = D.kitti_scan(3, n_azimuth=400)
    g = N.minkunet42()
    w = N.init_weights(g, 7)
    net, checked, worst = teacher_forced(ctx, g, w, coords, feats)
    assert checked == 49
    st = net.stats()
    # 5 submanifold (ts 1..16) + 4 down + 4 transposed + 4 1x1 identity maps (ts 2..16 ... ts 1)
    assert st["convs"] == 49 and st["maps_built"] <= 18
    q, ref = oracle_graph(g, w, coords, feats)
    for pf in (0, 1):
        net = N.Network(ctx, g, w, sc.exec_cfg(partial_f16=pf))
        net.forward(coords, feats)
        xo, fo = net.read(g.output)
        np.testing.assert_array_equal(xo, q)
        mx, mean = rel(fo, ref)
        print(f"MinkUNet42 end-to-end (partial_f16={pf}): |P|={len(coords)} max_rel={mx:.2e} mean_rel={mean:.2e};"
              f" per-layer worst {worst}")
        assert mx <= 1e-2 and mean <= 1e-3


def test_sparse_resnet21d_small_room(ctx):
    coords, feats = D.s3dis_room(2, n_points=60000, resolution=0.05)
    g = N.sparse_resnet21d()
    w = N.init_weights(g, 3)
    net, checked, _ = teacher_forced(ctx, g, w, coords, feats)
    assert checked == 21


def test_unet_pair_object(ctx):
    coords, feats = D.shapenet_object(5, n_points=40000)
    g = N.unet_pair()
    w = N.init_weights(g, 5)
    net, checked, _ = teacher_forced(ctx, g, w, coords, feats)
    assert checked == 2
    xo, fo = net.read(g.output)
    np.testing.assert_array_equal(xo, coords)  # transposed conv lands on the input coordinates


def test_network_repeatable(ctx):
    coords, feats = D.kitti_scan(4, n_azimuth=300)
    g = N.minkunet42()
    w = N.init_weights(g, 1)
    net = N.Network(ctx, g, w)
    net.forward(coords, feats)
    a = net.read(g.output)[1]
    net.forward(coords, feats)
    b = net.read(g.output)[1]
    np.testing.assert_array_equal(a, b)
