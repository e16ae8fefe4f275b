#!/usr/bin/env python3
"""Per-conv breakdown of a network forward with the per-conv roofline.

For every conv: shape, |M|, the AUTO tuner's GMaS and fused times (CUDA events, warm L2, min
of 2 after a warm-up) and the attainable time of the conv at roofline,

    t* = max(bytes / HBM peak, useful flops / tensor peak)
    bytes = 2*C_in*N + 4*|M| + 2*C_out*|Q| (x2 with a folded residual) + 2*K3*C_in*C_out
    flops = 2*C_in*C_out*|M|

(peaks from MEASURED_PEAKS.json: hbm_gbs, bf16_tflops), so frac = t* / t_fused per conv and
sum(t*) / sum(t) for the whole network.

  python profiles/net_layers.py --workload c2_minkunet42_kitti [--json out.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402,F401

import paper_2401_06145_b200 as sc  # noqa: E402
from paper_2401_06145_b200 import network as N  # noqa: E402
from paper_2401_06145_b200 import workloads as WL  # noqa: E402


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"])
    except Exception:
        return 6515.1, 1640.8


def conv_roofline(s, hbm_gbs, tc_tflops):
    n, q, M, ci, co, K3, res = s["n_in"], s["n_out"], s["M"], s["c_in"], s["c_out"], s["K3"], s["residual"]
    byts = 2 * ci * n + 4 * M + 2 * co * q * (2 if res else 1) + 2 * K3 * ci * co
    flops = 2 * ci * co * M
    t_hbm = byts / (hbm_gbs * 1e9)
    t_tc = flops / (tc_tflops * 1e12)
    return byts, flops, max(t_hbm, t_tc), "tensor" if t_tc > t_hbm else "hbm"


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--workload", default="c2_minkunet42_kitti")
    p.add_argument("--json", default=None)
    a = p.parse_args()
    hbm, tc = peaks()
    ctx = sc.Context(0)
    g = WL.graph(a.workload)
    w = N.init_weights(g, WL.WEIGHT_SEED)
    coords, feats = WL.scenes(a.workload)[0]
    net = N.Network(ctx, g, w, sc.exec_cfg(dataflow=sc.DATAFLOW_AUTO))
    net.forward(coords, feats, True)
    st = net.conv_stats()
    tm = net.auto_timings()
    conv_ops = [i for i, o in enumerate(g.ops) if o.kind == N.CONV]
    rows = []
    tot = dict(gmas=0.0, fused=0.0, best=0.0, tstar=0.0, flops=0.0, bytes=0.0)
    print(f"{'op':>3} {'K3':>3} {'n_in':>7} {'n_out':>7} {'|M|':>8} {'cin':>4} {'cout':>4} {'gmas_us':>8} "
          f"{'fused_us':>8} {'t*_us':>7} {'bound':>6} {'frac':>5} {'TF/s':>6} {'res':>3}")
    for s, i in zip(st, conv_ops):
        gm, fu = tm[i]
        byts, flops, tstar, bound = conv_roofline(s, hbm, tc)
        best = min(x for x in (gm, fu) if x > 0) * 1e-3
        tot["gmas"] += gm
        tot["fused"] += fu
        tot["best"] += best * 1e3
        tot["tstar"] += tstar * 1e3
        tot["flops"] += flops
        tot["bytes"] += byts
        rows.append(dict(op=i, **s, gmas_ms=gm, fused_ms=fu, bytes=byts, flops=flops, tstar_ms=tstar * 1e3,
                         bound=bound, frac=tstar / best))
        print(f"{i:>3} {s['K3']:>3} {s['n_in']:>7} {s['n_out']:>7} {s['M']:>8} {s['c_in']:>4} {s['c_out']:>4} "
              f"{1e3 * gm:>8.1f} {1e3 * fu:>8.1f} {1e6 * tstar:>7.1f} {bound:>6} {tstar / best:>5.2f} "
              f"{flops / best / 1e12:>6.0f} {s['residual']:>3}")
    print(f"total: gmas {tot['gmas']:.3f} ms, fused {tot['fused']:.3f} ms, best-of {tot['best']:.3f} ms, "
          f"roofline {tot['tstar']:.3f} ms -> frac {tot['tstar'] / tot['best']:.3f}; "
          f"{tot['flops'] / 1e9:.1f} GFLOP, {tot['bytes'] / 1e6:.1f} MB")
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"workload": a.workload, "peaks": {"hbm_gbs": hbm, "bf16_tflops": tc}, "convs": rows,
                       "totals": tot}, f, indent=1)


if __name__ == "__main__":
    main()
