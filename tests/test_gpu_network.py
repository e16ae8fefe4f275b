"""Network driver parity on the GPU (BASELINE configs 2-4 graphs on small synthetic scenes).

Layer-wise with teacher forcing: every CONV op's GPU input tensor (16-bit
activations, read back exactly) is fed to the CPU oracle with the same coordinates and the
weights rounded to the GPU operand type; output coordinates must be bit-exact and the
features must equal the oracle's output rounded to f16 up to one f16 ulp (only the fp32
accumulation order differs before the final rounding), and SURVEY §8(c)'s per-element
metric (max rel_e <= 1e-2, mean <= 1e-3, tests/parity.py) must hold per layer; the effect
of rounding the weights to 16 bits is bounded against the unrounded fp32 oracle (Frobenius-
relative <= 1e-3). ADD / CONCAT are
checked exactly (fp32 sum of the 16-bit operands, rounded once). Both dataflows (Minuet
GMaS and the fused output-stationary kernel) are teacher-forced; the default network
(AUTO dataflow, residual ADDs folded into conv epilogues) is checked end to end.
"""
import numpy as np
import pytest

import paper_2401_06145_b200 as sc
from paper_2401_06145_b200 import datasets as D
from paper_2401_06145_b200 import network as N
from oracle_lib import load_oracle
from oracle_net import oracle_graph  # noqa: F401  (the oracle graph runner, shared with bench.py)
from parity import assert_north_star, elementwise_errors

pytestmark = pytest.mark.gpu


def f16(a):
    return a.astype(np.float16).astype(np.float32)


def assert_f16_rounded(g, r):
    """g = r rounded to f16, allowing one f16 ulp (2^-10 relative) for accumulation-order ties."""
    r64, g64 = r.astype(np.float64), g.astype(np.float64)
    tol = np.abs(r64) * 2.0 ** -10 + 4e-6 * max(np.abs(r64).max(), 1e-30)
    bad = np.abs(g64 - r64) > tol
    assert not bad.any(), (int(bad.sum()), float(np.abs(g64 - r64).max()))


def teacher_forced(ctx, g, weights, coords, feats, dataflow=sc.DATAFLOW_GMAS, max_convs=None):
    """fp32 partials for GMaS (strict same-operand parity); residual folding off so every
    tensor is materialised. The default network is checked end to end in the tests below."""
    ora = load_oracle()
    net = N.Network(ctx, g, weights, sc.exec_cfg(partial_f16=0, dataflow=dataflow, fuse_residual=0))
    net.forward(coords, feats, True)
    checked = 0
    worst = (0.0, 0.0)
    for o in g.ops:
        xin, fin = net.read(o.a)
        xout, fout = net.read(o.out)
        if o.kind == N.CONV:
            if max_convs is not None and checked >= max_convs:
                continue
            np.testing.assert_array_equal(fin, f16(fin))  # activations are 16-bit
            W = weights[o.weight]
            tgt = net.read(o.b)[0] if o.transposed else None
            oq, of, _ = ora.layer_forward(xin, True, fin, f16(W), o.K, o.offset_scale, o.out_stride,
                                          bool(o.transposed), tgt, workers=8)
            if o.relu:
                of = np.maximum(of, 0)
            np.testing.assert_array_equal(xout, oq)
            assert_f16_rounded(fout, of)
            mx, mean, _ = assert_north_star(fout, of, str(o))  # SURVEY §8(c) per-element metric
            _, of32, _ = ora.layer_forward(xin, True, fin, W, o.K, o.offset_scale, o.out_stride, bool(o.transposed),
                                           tgt, workers=8)
            if o.relu:
                of32 = np.maximum(of32, 0)
            # 16-bit weight quantisation (reported): Frobenius-relative vs the unrounded fp32 weights
            assert elementwise_errors(fout, of32)[2] <= 1e-3, o
            worst = (max(worst[0], mx), max(worst[1], mean))
            checked += 1
        elif o.kind == N.ADD:
            xb, fb = net.read(o.b)
            ref = fin + fb
            np.testing.assert_array_equal(fout, f16(np.maximum(ref, 0) if o.relu else ref))
        else:
            xb, fb = net.read(o.b)
            np.testing.assert_array_equal(fout, np.concatenate([fin, fb], 1))
    return net, checked, worst


@pytest.mark.parametrize("dataflow", [sc.DATAFLOW_GMAS, sc.DATAFLOW_FUSED])
def test_minkunet42_small_scan(ctx, dataflow):
    coords, feats = D.kitti_scan(3, n_azimuth=400)
    g = N.minkunet42()
    w = N.init_weights(g, 7)
    net, checked, worst = teacher_forced(ctx, g, w, coords, feats, dataflow)
    assert checked == 49
    st = net.stats()
    # 5 submanifold (ts 1..16) + 4 down + 4 transposed + 4 1x1 identity maps (ts 2..16 ... ts 1)
    assert st["convs"] == 49 and st["maps_built"] <= 18
    assert all(s["dataflow"] == dataflow for s in net.conv_stats())
    print(f"MinkUNet42 teacher-forced (dataflow={dataflow}): per-layer worst {worst}")


def test_minkunet42_end_to_end(ctx):
    """Default network (AUTO dataflow per conv, residual ADDs folded into conv epilogues) and
    the unfolded GMaS-only network against the fp32 oracle graph."""
    coords, feats = D.kitti_scan(3, n_azimuth=400)
    g = N.minkunet42()
    w = N.init_weights(g, 7)
    q, ref = oracle_graph(g, w, coords, feats)
    outs = {}
    for name, cfg in [("default", sc.exec_cfg(dataflow=sc.DATAFLOW_AUTO)),
                      ("fused", sc.exec_cfg(dataflow=sc.DATAFLOW_FUSED)),
                      ("gmas-unfolded", sc.exec_cfg(dataflow=sc.DATAFLOW_GMAS, fuse_residual=0))]:
        net = N.Network(ctx, g, w, cfg)
        net.forward(coords, feats)
        xo, fo = net.read(g.output)
        np.testing.assert_array_equal(xo, q)
        mx, mean, fro = elementwise_errors(fo, ref)
        st = net.conv_stats()
        print(f"MinkUNet42 end-to-end ({name}): |P|={len(coords)} max_rel={mx:.2e} mean_rel={mean:.2e} "
              f"fro={fro:.2e} fused={sum(s['dataflow'] for s in st)}/{len(st)} folded={sum(s['residual'] for s in st)}")
        # 16-bit activations and weights through 49 layers: end to end gated on the Frobenius-relative
        # error (the per-layer §8(c) check above is the parity gate)
        assert fro <= 2e-2, (name, mx, mean, fro)
        outs[name] = fo
        if name != "gmas-unfolded":
            assert sum(s["residual"] for s in st) == 16  # every residual ADD folded
            with pytest.raises(sc.LogicError):
                net.read(g.ops[-2].out)  # the folded conv's own output is never materialised
    # folding the ADD changes only where one rounding happens
    assert elementwise_errors(outs["fused"], outs["gmas-unfolded"])[2] <= 2e-2


def test_minkunet42_bf16_end_to_end(ctx):
    """bf16 activations and weights (compute_dtype=BF16) through the whole network: fused
    dataflow, folded residuals, derived K=2 maps; output coordinates exact, features against the
    fp32 oracle graph (bf16 keeps 8 mantissa bits: the Frobenius bound is 8x the f16 one)."""
    coords, feats = D.kitti_scan(3, n_azimuth=400)
    g = N.minkunet42()
    w = N.init_weights(g, 7)
    q, ref = oracle_graph(g, w, coords, feats)
    net = N.Network(ctx, g, w, sc.exec_cfg(dataflow=sc.DATAFLOW_FUSED, compute_dtype=sc.BF16))
    net.forward(coords, feats)
    xo, fo = net.read(g.output)
    np.testing.assert_array_equal(xo, q)
    mx, mean, fro = elementwise_errors(fo, ref)
    print(f"MinkUNet42 bf16 end-to-end: max_rel={mx:.2e} mean_rel={mean:.2e} fro={fro:.2e}")
    assert fro <= 1.6e-1, (mx, mean, fro)
    assert sum(s["dataflow"] for s in net.conv_stats()) == 49


@pytest.mark.parametrize("dataflow", [sc.DATAFLOW_GMAS, sc.DATAFLOW_FUSED])
def test_sparse_resnet21d_small_room(ctx, dataflow):
    coords, feats = D.s3dis_room(2, n_points=60000, resolution=0.05)
    g = N.sparse_resnet21d()
    w = N.init_weights(g, 3)
    net, checked, _ = teacher_forced(ctx, g, w, coords, feats, dataflow)
    assert checked == 21


@pytest.mark.parametrize("dataflow", [sc.DATAFLOW_GMAS, sc.DATAFLOW_FUSED])
def test_unet_pair_object(ctx, dataflow):
    coords, feats = D.shapenet_object(5, n_points=40000)
    g = N.unet_pair()
    w = N.init_weights(g, 5)
    net, checked, _ = teacher_forced(ctx, g, w, coords, feats, dataflow)
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


def test_batched_clouds_match_individual(ctx):
    """Batch-in-coordinates (datasets.batch_clouds): one forward over 3 shifted objects gives each
    object's output rows exactly as its own forward does (no cross-object neighbours)."""
    objs = [D.shapenet_object(20 + b, n_points=15000) for b in range(3)]
    g = N.unet_pair()
    w = N.init_weights(g, 5)
    coords, feats, ranges = D.batch_clouds(objs)
    net = N.Network(ctx, g, w)
    net.forward(coords, feats, True)
    _, fb = net.read(g.output)
    for (c, f), (a, b) in zip(objs, ranges):
        order = np.lexsort((c[:, 2], c[:, 1], c[:, 0]))
        one = N.Network(ctx, g, w)
        one.forward(c[order], f[order], True)
        _, fo = one.read(g.output)
        np.testing.assert_allclose(fb[a:b], fo, rtol=0, atol=1e-6 * max(np.abs(fo).max(), 1e-30))



def test_read_async_pipelined(ctx):
    """sconv_net_read_async + sconv_net_prefetch_inputs: back-to-back forwards on different scans,
    each one's inputs staged while the previous forward runs and its result read back while the
    next runs (two staging slots each, reused), equal the synchronous results bit for bit; a
    non-matching prefetch is ignored; a bad tensor id fails loudly."""
    import torch
    g = N.minkunet42()
    w = N.init_weights(g, 1)
    net = N.Network(ctx, g, w)
    scans = [D.kitti_scan(s, n_azimuth=200) for s in (4, 5, 6)]
    want = []
    for c, f in scans:
        net.forward(c, f)
        want.append(net.read(g.output)[1])
    pinned = [(torch.from_numpy(c).pin_memory().numpy(), torch.from_numpy(f).pin_memory().numpy()) for c, f in scans]
    order = [0, 1, 2, 0, 2, 1]
    got = []
    for r, i in enumerate(order):
        net.forward(*pinned[i])
        if r + 1 < len(order):  # next request's inputs staged beside this forward
            net.prefetch(*pinned[order[r + 1]])
        n, ch, _ = net.info(g.output)
        buf = torch.empty((n, ch), dtype=torch.float32, pin_memory=True).numpy()
        net.read_async(g.output, buf)
        got.append(buf)
    net.wait_reads()
    for i, b in zip(order, got):
        np.testing.assert_array_equal(want[i], b)
    # a prefetch that the next forward does not match is ignored (that forward stages its own)
    net.prefetch(*pinned[0])
    net.forward(*pinned[1])
    np.testing.assert_array_equal(want[1], net.read(g.output)[1])
    net.forward(*pinned[0])
    np.testing.assert_array_equal(want[0], net.read(g.output)[1])
    with pytest.raises(sc.InvalidArgument):
        net.read_async(10 ** 6, got[0])
