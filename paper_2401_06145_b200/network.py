"""Network graphs for BASELINE configs 2-5 and the ctypes wrapper of the network driver.

The reference gives only the SC layer and a sequential netdef; the
backbones it cites (MinkUNet42, SparseResNet21D) are not specified there,
so the topologies below are this builder's definitions, with BN folded away
(inference) and ReLU fused into the conv epilogues:

  MinkUNet42      stem 2 x conv3 | 4 x [down K=2 s=2, 2 residual blocks] | 4 x [transposed
                  K=2 s=2, concat skip, 2 residual blocks]  -> 42 SC convs + 7 1x1 shortcuts
  SparseResNet21D stem conv3 | stage1 2 residual blocks | 4 x [conv3 s=2, 2 residual blocks]
                  with the last stage a single strided conv  -> 21 SC convs (x2 width "wide")
  UNetPair        K=2 s=2 down 32->64, transposed K=2 s=2 64->32 onto the input coordinates

Weights: U[-a, a] from Rng(stream_seed(seed, weight_id + 1)) (SPEC.md:528 draws U[-0.1, 0.1];
here a = sqrt(3 / (nbr * c_in)) with nbr the expected neighbours per voxel, so activations
neither explode nor vanish through 42 layers with random weights — the SPEC scale is the
special case nbr * c_in = 300).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import sconv as S

CONV, ADD, CONCAT = 1, 2, 3


@dataclass
class Op:
    kind: int
    out: int
    a: int
    b: int = -1  # second operand (ADD/CONCAT) or target tensor (transposed CONV)
    K: int = 3
    offset_scale: int = 1
    out_stride: int = 1
    transposed: int = 0
    c_in: int = 0
    c_out: int = 0
    weight: int = -1
    relu: int = 0

    def row(self):
        return [self.kind, self.out, self.a, self.b, self.K, self.offset_scale, self.out_stride, self.transposed,
                self.c_in, self.c_out, self.weight, self.relu]


@dataclass
class Graph:
    ops: List[Op] = field(default_factory=list)
    n_tensors: int = 0
    input: int = 0
    output: int = 0
    in_channels: int = 0
    channels: dict = field(default_factory=dict)
    stride: dict = field(default_factory=dict)  # tensor stride per tensor (for docs / checks)
    nbr: dict = field(default_factory=dict)     # expected neighbours used for the weight scale

    def tensor(self, c, ts):
        t = self.n_tensors
        self.n_tensors += 1
        self.channels[t], self.stride[t] = c, ts
        return t

    def conv(self, x, c_out, K=3, out_stride=None, relu=True, nbr=9.0):
        """out_stride = the output TENSOR stride; the op's Eq. 1 stride is 1 when it equals the
        input's (submanifold: Q = P) and the new tensor stride otherwise (floor to it)."""
        ts = self.stride[x]
        out_ts = ts if out_stride is None else out_stride
        y = self.tensor(c_out, out_ts)
        w = len([o for o in self.ops if o.kind == CONV])
        eq1 = 1 if out_ts == ts else out_ts
        self.ops.append(Op(CONV, y, x, -1, K, ts, eq1, 0, self.channels[x], c_out, w, int(relu)))
        self.nbr[w] = nbr
        return y

    def down(self, x, c_out, relu=True):  # K=2 s=2 (offsets {0, ts}^3, Q = floor(P / 2ts) * 2ts)
        return self.conv(x, c_out, K=2, out_stride=2 * self.stride[x], relu=relu, nbr=4.0)

    def up(self, x, target, c_out, relu=True):  # transposed K=2 s=2 onto `target`'s coordinates
        ts = self.stride[target]
        y = self.tensor(c_out, ts)
        w = len([o for o in self.ops if o.kind == CONV])
        self.ops.append(Op(CONV, y, x, target, 2, ts, ts, 1, self.channels[x], c_out, w, int(relu)))
        self.nbr[w] = 1.0
        return y

    def add(self, a, b, relu=True):
        y = self.tensor(self.channels[a], self.stride[a])
        self.ops.append(Op(ADD, y, a, b, relu=int(relu)))
        return y

    def concat(self, a, b):
        y = self.tensor(self.channels[a] + self.channels[b], self.stride[a])
        self.ops.append(Op(CONCAT, y, a, b))
        return y

    def residual(self, x, c_out):
        h = self.conv(x, c_out)
        h = self.conv(h, c_out, relu=False)
        sc = x if self.channels[x] == c_out else self.conv(x, c_out, K=1, relu=False, nbr=1.0)
        return self.add(h, sc)

    def convs(self):
        return [o for o in self.ops if o.kind == CONV]


def minkunet42(in_ch=4, cs=(32, 32, 64, 128, 256, 256, 128, 96, 96)) -> Graph:
    g = Graph(in_channels=in_ch)
    x = g.tensor(in_ch, 1)
    g.input = x
    x = g.conv(x, cs[0])
    x0 = g.conv(x, cs[0])
    enc, h = [x0], x0
    for i in range(4):
        h = g.down(h, cs[i])
        h = g.residual(h, cs[i + 1])
        h = g.residual(h, cs[i + 1])
        enc.append(h)
    for i in range(4):
        skip = enc[3 - i]
        h = g.up(h, skip, cs[5 + i])
        h = g.concat(h, skip)
        h = g.residual(h, cs[5 + i])
        h = g.residual(h, cs[5 + i])
    g.output = h
    return g


def sparse_resnet21d(in_ch=6, width=2) -> Graph:
    c = [16 * width, 32 * width, 64 * width, 128 * width]
    g = Graph(in_channels=in_ch)
    x = g.tensor(in_ch, 1)
    g.input = x
    h = g.conv(x, c[0])
    h = g.residual(h, c[0])
    h = g.residual(h, c[0])
    for i in range(1, 4):
        h = g.conv(h, c[i], K=3, out_stride=2 * g.stride[h], nbr=3.0)  # conv3 stride 2
        h = g.residual(h, c[i])
        h = g.residual(h, c[i])
    h = g.conv(h, c[3], K=3, out_stride=2 * g.stride[h], nbr=3.0)  # last stage: one strided conv
    g.output = h
    return g


def unet_pair(c_in=32, c_mid=64) -> Graph:
    g = Graph(in_channels=c_in)
    x = g.tensor(c_in, 1)
    g.input = x
    d = g.down(x, c_mid, relu=False)
    g.output = g.up(d, x, c_in, relu=False)
    return g


def init_weights(g: Graph, seed: int):
    """Per conv weight id: U[-a, a] with a = sqrt(3 / (nbr * c_in)) (see module docstring)."""
    out = {}
    for o in g.convs():
        K3 = o.K ** 3
        w = S.generate_weights(seed, o.weight + 1, K3, o.c_in, o.c_out)  # U[-0.1, 0.1]
        a = np.sqrt(3.0 / (g.nbr[o.weight] * o.c_in))
        out[o.weight] = (w * np.float32(a / 0.1)).astype(np.float32)
    return out


class Network:
    """Device-resident network (sconv_net): weights uploaded once, forward = graph run."""

    def __init__(self, ctx: S.Context, g: Graph, weights: dict, cfg: Optional[S.ExecCfg] = None, B=256, Cq=512):
        self.ctx, self.g = ctx, g
        rows = np.array([o.row() for o in g.ops], np.int32).reshape(-1, 12)
        h = C.c_void_p()
        cfg = cfg or S.exec_cfg()
        ctx.check(ctx.lib.sconv_net_create(ctx.h, S._ptr(rows), len(g.ops), g.n_tensors, g.input, g.output,
                                           C.byref(cfg), B, Cq, C.byref(h)))
        self.h = h
        ctx.adopt(self)
        for wid, w in weights.items():
            w = np.ascontiguousarray(w, np.float32)
            ctx.check(ctx.lib.sconv_net_set_weights(ctx.h, h, wid, S._ptr(w), S.MEM_HOST, *w.shape))

    def forward(self, coords=None, feats=None, sorted_=True, device_xyz=None, device_feats=None, n=None):
        if device_xyz is not None:
            self.ctx.check(self.ctx.lib.sconv_net_forward(self.ctx.h, self.h, device_xyz, n, S.MEM_DEVICE,
                                                          int(sorted_), device_feats, S.MEM_DEVICE,
                                                          self.g.in_channels))
        else:
            c = np.ascontiguousarray(coords, np.int32)
            f = np.ascontiguousarray(feats, np.float32)
            self.ctx.check(self.ctx.lib.sconv_net_forward(self.ctx.h, self.h, S._ptr(c), len(c), S.MEM_HOST,
                                                          int(sorted_), S._ptr(f), S.MEM_HOST, f.shape[1]))

    def info(self, t):
        n, ch, cs = C.c_int64(), C.c_int(), C.c_int()
        self.ctx.check(self.ctx.lib.sconv_net_tensor_info(self.ctx.h, self.h, t, C.byref(n), C.byref(ch),
                                                          C.byref(cs)))
        return n.value, ch.value, cs.value

    def read(self, t, feats_out: Optional[np.ndarray] = None, coords: bool = True):
        """Host copy of tensor t: (coords or None, fp32 features). feats_out (e.g. a pinned
        array) receives the features in place when given."""
        n, ch, _ = self.info(t)
        xyz = np.empty((n, 3), np.int32) if coords else None
        if feats_out is not None:
            if feats_out.shape != (n, ch) or feats_out.dtype != np.float32 or not feats_out.flags.c_contiguous:
                raise ValueError("feats_out must be a contiguous float32 array of shape (n, channels)")
            f = feats_out
        else:
            f = np.empty((n, ch), np.float32)
        self.ctx.check(self.ctx.lib.sconv_net_read_tensor(self.ctx.h, self.h, t, S._ptr(xyz) if coords else None,
                                                          S._ptr(f)))
        return xyz, f

    def device_output(self):
        """(pointer, dtype, row stride) of the output tensor on device."""
        p, dt, ld = C.c_void_p(), C.c_int(), C.c_int64()
        self.ctx.check(self.ctx.lib.sconv_net_tensor_device(self.h, self.g.output, C.byref(p), C.byref(dt),
                                                            C.byref(ld)))
        return p.value, dt.value, ld.value

    def stats(self):
        mb, nc = C.c_int(), C.c_int()
        self.ctx.check(self.ctx.lib.sconv_net_stats(self.h, C.byref(mb), C.byref(nc)))
        return dict(maps_built=mb.value, convs=nc.value)

    STAT_KEYS = ["n_in", "n_out", "M", "R", "c_in", "c_out", "k_pad", "K3", "dataflow", "residual"]

    def conv_stats(self):
        """Per conv (execution order): n_in, n_out, M, R_pad (0 when fused), c_in, c_out, k_pad, K3,
        dataflow (0 GMaS / 1 fused), residual (ADD folded into the epilogue)."""
        out = []
        for i in range(len(self.g.convs())):
            v = np.zeros(10, np.int64)
            if self.ctx.lib.sconv_net_conv_stats(self.h, i, S._ptr(v)) != S.OK:
                break
            out.append(dict(zip(self.STAT_KEYS, v.tolist())))
        return out

    def auto_timings(self):
        """Per op index: (GMaS ms, fused ms) measured by the AUTO tuning forward (-1: not tuned)."""
        out = {}
        for i, o in enumerate(self.g.ops):
            if o.kind != CONV:
                continue
            a, b = C.c_double(), C.c_double()
            self.ctx.check(self.ctx.lib.sconv_net_conv_timings(self.h, i, C.byref(a), C.byref(b)))
            out[i] = (a.value, b.value)
        return out

    def algo_bytes(self, part_bytes=2):
        """Algorithmic bytes per kernel type summed over the convs (SURVEY §8d with this path's dtypes:
        16-bit activations, 16-bit gather buffer, `part_bytes` GEMM partials, 16-bit outputs).
        Fused convs: input rows read once (2*ci*n), the nbr table (4*K3*q), output (+residual) once."""
        g = e = s = f = 0
        maps = {}  # distinct searched maps (identity 1x1 maps need no search): SURVEY §8d Map bytes
        for st in self.conv_stats():
            n, q, M, R, ci, co, kp, K3, df, res = (st[k] for k in self.STAT_KEYS)
            if K3 > 1:
                maps[(n, q, M, K3)] = 8 * n + 8 * q + 8 * M + 4 * K3
            if df == 1:
                f += 2 * ci * n + 4 * K3 * q + 2 * co * q * (2 if res else 1)
                continue
            g += 2 * ci * n + 2 * kp * R + 4 * M
            e += 2 * kp * R + part_bytes * co * R + 2 * K3 * ci * co
            s += part_bytes * co * M + 4 * K3 * q + 2 * co * q * (2 if res else 1)
        return {"k_gather": g, "k_gemm_grouped": e, "k_scatter": s, "k_conv_fused": f,
                "k_search": sum(maps.values()), "_k_search_launches": len(maps)}

    def free(self):
        if self.h:
            self.ctx.lib.sconv_net_free(self.ctx.h, self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
