"""Parity of the BENCHED networks at the bench's own sizes (north_star "on all
five configs").

Each config runs exactly as bench.py runs it — same scenes (paper_2401_06145_b200/workloads.py),
same weights, default network config (AUTO dataflow per conv, residual ADDs folded into conv
epilogues, f16 activations, B=256, C=512), second forward (after the AUTO choice) — and is
checked layer by layer with teacher forcing: every conv's GPU input tensor (16-bit, read back
exactly) goes through the CPU oracle's sc_layer_forward (fp64 accumulation)
with the same 16-bit weight values the GPU multiplies, and

  * output coordinates must be bit-exact (canonical sorted order);
  * features must meet §8(c)'s per-element metric rel_e = |g-r| / max(|r|, 1e-3 ||r||_inf):
    max <= 1e-2 and mean <= 1e-3 (tests/parity.py).

A folded conv (its ADD fused into the epilogue) is checked through the ADD's output:
relu(oracle conv + the GPU's residual operand). The quantisation effect of 16-bit weights is
reported separately against the unrounded fp32 weights (Frobenius-relative), and so is the
end-to-end error of the whole graph against the fp32 oracle graph.
"""
import json
import os

import numpy as np
import pytest

import paper_2401_06145_b200 as sc
from paper_2401_06145_b200 import network as N
from paper_2401_06145_b200 import workloads as WL
from oracle_lib import load_oracle
from oracle_net import oracle_graph
from parity import MAX_TOL, MEAN_TOL, elementwise_errors

pytestmark = pytest.mark.gpu

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


def f16(a):
    return a.astype(np.float16).astype(np.float32)


def teacher_forced_bench(ctx, g, w, coords, feats):
    """Teacher-forced check of the bench's own network; returns per-conv error records."""
    ora = load_oracle()
    net = N.Network(ctx, g, w, sc.exec_cfg(compute_dtype=sc.F16), 256, 512)
    net.forward(coords, feats, True)  # AUTO dataflow choice happens here (bench warm-up)
    net.forward(coords, feats, True)  # the steady-state forward the bench times
    cache = {}

    def read(t):
        if t not in cache:
            cache[t] = net.read(t)
        return cache[t]

    consumers = {}
    for j, o in enumerate(g.ops):
        if o.kind == N.ADD:
            consumers.setdefault(o.a, []).append((j, o.b))
            consumers.setdefault(o.b, []).append((j, o.a))
    dflows = [s["dataflow"] for s in net.conv_stats()]
    recs, conv_i = [], 0
    for o in g.ops:
        if o.kind != N.CONV:
            continue
        xin, fin = read(o.a)
        assert np.array_equal(fin, f16(fin)), "activations must be 16-bit values"
        tgt = read(o.b)[0] if o.transposed else None
        W16 = f16(w[o.weight])
        oq, of, _ = ora.layer_forward(xin, True, fin, W16, o.K, o.offset_scale, o.out_stride, bool(o.transposed),
                                      tgt, workers=os.cpu_count())
        _, of32, _ = ora.layer_forward(xin, True, fin, w[o.weight], o.K, o.offset_scale, o.out_stride,
                                       bool(o.transposed), tgt, workers=os.cpu_count())
        if o.relu:
            of, of32 = np.maximum(of, 0), np.maximum(of32, 0)
        try:
            xout, fout = read(o.out)
            folded = False
        except sc.LogicError:  # residual ADD folded into this conv's epilogue
            (j, other), = consumers[o.out]
            add = g.ops[j]
            xout, fout = read(add.out)
            res = read(other)[1]
            of, of32 = of + res, of32 + res
            if add.relu:
                of, of32 = np.maximum(of, 0), np.maximum(of32, 0)
            folded = True
        np.testing.assert_array_equal(xout, oq)
        mx, mean, fro = elementwise_errors(fout, of)
        q = elementwise_errors(fout, of32)[2]
        recs.append({"conv": conv_i, "K": o.K, "c_in": o.c_in, "c_out": o.c_out, "n_out": int(len(oq)),
                     "dataflow": "fused" if dflows[conv_i] == 1 else "gmas", "folded": folded,
                     "max_rel_e": mx, "mean_rel_e": mean, "fro": fro, "fro_vs_fp32_weights": q})
        assert mx <= MAX_TOL and mean <= MEAN_TOL, recs[-1]
        conv_i += 1
    out = net.read(g.output)
    net.free()
    return recs, out


def run_config(ctx, name, clouds, end_to_end=True):
    g = WL.graph(name)
    w = N.init_weights(g, WL.WEIGHT_SEED)
    summary = {"config": name, "scenes": []}
    for coords, feats in clouds:
        recs, (xo, fo) = teacher_forced_bench(ctx, g, w, coords, feats)
        assert len(recs) == len(g.convs())
        scene = {"voxels": int(len(coords)), "convs": len(recs),
                 "worst_max_rel_e": max(r["max_rel_e"] for r in recs),
                 "worst_mean_rel_e": max(r["mean_rel_e"] for r in recs),
                 "worst_fro_vs_fp32_weights": max(r["fro_vs_fp32_weights"] for r in recs),
                 "fused_convs": sum(r["dataflow"] == "fused" for r in recs),
                 "folded_convs": sum(r["folded"] for r in recs), "layers": recs}
        if end_to_end:
            q, ref = oracle_graph(g, w, coords, feats)
            np.testing.assert_array_equal(xo, q)
            mx, mean, fro = elementwise_errors(fo, ref)
            scene["end_to_end"] = {"max_rel_e": mx, "mean_rel_e": mean, "fro": fro}
            assert fro <= 2e-2, scene["end_to_end"]  # 49 layers of 16-bit activations: reported, loosely gated
        summary["scenes"].append(scene)
        print(json.dumps({k: v for k, v in scene.items() if k != "layers"}))
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"parity_fullsize_{name}.json"), "w") as f:
        json.dump(summary, f, indent=1)
    return summary


def test_c2_full_scan(ctx):
    s = run_config(ctx, "c2_minkunet42_kitti", WL.scenes("c2_minkunet42_kitti"))
    assert s["scenes"][0]["voxels"] == 118964


def test_c3_full_room(ctx):
    s = run_config(ctx, "c3_resnet21d_s3dis", WL.scenes("c3_resnet21d_s3dis"))
    assert s["scenes"][0]["voxels"] == 336813


def test_c4_object_batch(ctx):
    clouds = WL.scenes("c4_unet_pair_shapenet")
    s = run_config(ctx, "c4_unet_pair_shapenet", clouds)
    assert s["scenes"][0]["voxels"] == sum(len(WL.D.shapenet_object(i)[0]) for i in range(WL.C4_OBJECTS))


def test_c5_two_scenes(ctx):
    """Two scenes of the 64-scan batch (the first and the last of the 8-GPU shards' extremes)."""
    run_config(ctx, "c5_minkunet42_batch64", [WL.kitti_scene(1), WL.kitti_scene(63)], end_to_end=False)
