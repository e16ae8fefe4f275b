"""autotune_network (Alg. 2) and the tile-size acceptance criterion #6
 on the GPU path.

* autotune_network over 3 sample clouds: every conv's pick is a supported divisor of its channel
  count and attains the minimum of the summed medians, smallest tile on ties;
  tuning never changes results (bit-identical to tile 1); an empty sample is an
  argument error.
* #6: on a synthetic layer per (channels in {16, 64, 128}) x (points in {1e4, 1e5}) the measured
  gather-latency-vs-tile curve is non-constant, the tuner's pick re-measures within 5% of the
  exhaustive minimum (plus 1 us of timer slack: single-digit-us kernels), and the GPU's IMT-lookup
  counter equals (C_in / T) x |M| exactly for every candidate T. Tiles are the supported divisors
  (T <= 64: one thread keeps its T channels in registers), so C = 128 tunes over 1..64.
"""
import numpy as np
import pytest
import torch

import paper_2401_06145_b200 as sc
from paper_2401_06145_b200 import datasets as D
from paper_2401_06145_b200 import network as N

pytestmark = pytest.mark.gpu

SUPPORTED = (1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64)


def candidates(c):
    return [t for t in SUPPORTED if c % t == 0]


def argmin_smallest(ms):
    return min(ms, key=lambda t: (ms[t], t))


def test_autotune_network(ctx):
    g = N.minkunet42()
    w = N.init_weights(g, 1)
    samples = [(c, f, True) for c, f in (D.kitti_scan(s, n_azimuth=300) for s in (11, 12, 13))]
    net = N.Network(ctx, g, w, sc.exec_cfg(dataflow=sc.DATAFLOW_GMAS))
    res = net.autotune(samples, rounds=3)
    convs = [i for i, o in enumerate(g.ops) if o.kind == N.CONV]
    assert sorted(res) == convs
    for i in convs:
        o, r = g.ops[i], res[i]
        gm, sm = r["gather_ms"], r["scatter_ms"]
        assert list(gm) == candidates(o.c_in) and list(sm) == candidates(o.c_out)
        assert all(v > 0 for v in gm.values()) and all(v > 0 for v in sm.values())
        assert r["gather_tile"] == argmin_smallest(gm), (i, gm, r["gather_tile"])
        assert r["scatter_tile"] == argmin_smallest(sm), (i, sm, r["scatter_tile"])
    # tuned tiles never change the numbers: bit-identical to tile 1 on a fourth cloud
    coords, feats = D.kitti_scan(14, n_azimuth=300)
    net.forward(coords, feats, True)
    _, out_t = net.read(g.output)
    ref = N.Network(ctx, g, w, sc.exec_cfg(dataflow=sc.DATAFLOW_GMAS, gather_tile=1, scatter_tile=1))
    ref.forward(coords, feats, True)
    _, out_1 = ref.read(g.output)
    np.testing.assert_array_equal(out_t, out_1)
    with pytest.raises(sc.InvalidArgument, match="sample must be nonempty"):
        net.autotune([], rounds=3)


@pytest.mark.parametrize("points,extent", [(10_000, 40), (100_000, 90)])
@pytest.mark.parametrize("channels", [16, 64, 128])
def test_tile_curve_acceptance6(ctx, channels, points, extent):
    xyz, F = sc.generate_synthetic(points, extent, channels, 5)
    m = sc.KernelMap.build(ctx, xyz, False, 3, 1, 1)
    matches = int(m.info().total_matches)
    w = sc.Weights(ctx, sc.generate_weights(5, 1, 27, channels, channels))
    f_dev = torch.from_numpy(F).cuda()
    torch.cuda.synchronize()
    cand = candidates(channels)
    tg, _, lat = sc.tune_layer(ctx, m, w, f_dev.data_ptr(), sc.F32, rounds=5)
    g_lat = dict(zip(cand, lat[:len(cand)]))
    assert tg == argmin_smallest(g_lat)
    assert max(g_lat.values()) > 1.05 * min(g_lat.values()), g_lat  # non-constant curve
    # re-measurement: the pick against the exhaustive minimum
    _, _, lat2 = sc.tune_layer(ctx, m, w, f_dev.data_ptr(), sc.F32, rounds=9)
    g2 = dict(zip(cand, lat2[:len(cand)]))
    assert g2[tg] <= 1.05 * min(g2.values()) + 1e-3, (tg, g2)
    # IMT lookups = (C_in / T) * |M| for every candidate tile (exact device counter)
    ctx.count_lookups(True)
    try:
        ctx.lookup_count()
        for t in cand:
            sc.layer_forward(ctx, m, w, F, sc.exec_cfg(gather_tile=t))
            assert ctx.lookup_count() == (channels // t) * matches, t
    finally:
        ctx.count_lookups(False)
