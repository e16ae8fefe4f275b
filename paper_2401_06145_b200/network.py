"""ctypes wrapper of the network driver (sconv_net_*, include/sconv_b200.h); the graphs
themselves live in graphs.py (pure Python)."""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import sconv as S
from .graphs import (ADD, CONCAT, CONV, PRESETS, Graph, Op, minkunet42, sparse_resnet21d, spec_chain,  # noqa: F401
                     unet_pair, weight_scale)
from . import graphs as _graphs


def init_weights(g: Graph, seed: int):
    """graphs.init_weights with the engine's SPEC PRNG (sconv_generate_weights)."""
    return _graphs.init_weights(g, seed, S.generate_weights)


def forward_network(ctx: S.Context, layers, cloud: S.PointCloud, seed: int, cfg: Optional[S.ExecCfg] = None,
                    B: int = 256, Cq: int = 512):
    """SPEC forward_network(spec, cloud, config, seed): the sequential chain
    `layers` [(K, s, c_in, c_out), ...] with SPEC weights (stream l+1, U[-0.1, 0.1]) on the GPU.
    Returns (output PointCloud (sorted), coordinate sorts performed)."""
    g = spec_chain(layers)
    net = Network(ctx, g, _graphs.spec_weights(g, seed, S.generate_weights), cfg, B, Cq)
    net.forward(cloud.coords, cloud.features, cloud.sorted)
    xyz, f = net.read(g.output)
    sorts = net.sort_count()
    net.free()
    return S.PointCloud(xyz, f, True), sorts


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

    def read_async(self, t, feats_out: np.ndarray):
        """Queues the fp32 features of tensor t into feats_out (pinned for an asynchronous copy)
        without waiting: the device->host copy runs on the net's copy stream beside the next
        forward (sconv_net_read_async). feats_out is valid after wait_reads()."""
        n, ch, _ = self.info(t)
        if feats_out.shape != (n, ch) or feats_out.dtype != np.float32 or not feats_out.flags.c_contiguous:
            raise ValueError("feats_out must be a contiguous float32 array of shape (n, channels)")
        self.ctx.check(self.ctx.lib.sconv_net_read_async(self.ctx.h, self.h, t, S._ptr(feats_out)))

    def prefetch(self, coords, feats):
        """Queues the host->device copy of the NEXT forward's host inputs now (it overlaps the
        current forward); forward() with the same arrays then uses the staged copy
        (sconv_net_prefetch_inputs). The arrays must stay unchanged until that forward."""
        if coords.dtype != np.int32 or feats.dtype != np.float32 or not coords.flags.c_contiguous \
                or not feats.flags.c_contiguous:
            raise ValueError("prefetch needs contiguous int32 coordinates and float32 features")
        self.ctx.check(self.ctx.lib.sconv_net_prefetch_inputs(self.ctx.h, self.h, S._ptr(coords), len(coords),
                                                              S._ptr(feats), S.MEM_HOST, feats.shape[1]))

    def wait_reads(self):
        """Blocks until every read_async of this network has landed (sconv_net_read_wait)."""
        self.ctx.check(self.ctx.lib.sconv_net_read_wait(self.ctx.h, self.h))

    def device_output(self):
        """(pointer, dtype, row stride) of the output tensor on device."""
        p, dt, ld = C.c_void_p(), C.c_int(), C.c_int64()
        self.ctx.check(self.ctx.lib.sconv_net_tensor_device(self.h, self.g.output, C.byref(p), C.byref(dt),
                                                            C.byref(ld)))
        return p.value, dt.value, ld.value

    def copy_tensor(self, t, dst_ptr: int, dtype=S.F16, mem=S.MEM_DEVICE):
        """Features of tensor t into a caller buffer (n x channels, dense): asynchronous on the
        context stream for a device destination (sconv_net_copy_tensor)."""
        self.ctx.check(self.ctx.lib.sconv_net_copy_tensor(self.ctx.h, self.h, t, dst_ptr, dtype, mem))

    def sort_count(self):
        """Coordinate sorts of the last forward (acceptance #7 accounting)."""
        v = C.c_int64()
        self.ctx.check(self.ctx.lib.sconv_net_sort_count(self.h, C.byref(v)))
        return v.value

    def stats(self):
        mb, nc = C.c_int(), C.c_int()
        self.ctx.check(self.ctx.lib.sconv_net_stats(self.h, C.byref(mb), C.byref(nc)))
        return dict(maps_built=mb.value, convs=nc.value)

    STAT_KEYS = ["n_in", "n_out", "M", "R", "c_in", "c_out", "k_pad", "K3", "dataflow", "residual"]

    def conv_stats(self):
        """Per conv (execution order): n_in, n_out, M, R_pad (0 when fused), c_in, c_out, k_pad, K3,
        dataflow (0 GMaS / 1 fused), residual (ADD folded into the epilogue)."""
        self.ctx.check(self.ctx.lib.sconv_net_resolve_stats(self.ctx.h, self.h))  # |M| of lazily built maps
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

    def autotune(self, samples, rounds: int = 5):
        """SPEC autotune_network(layers, sample, R) (Alg. 2): `samples` is a list
        of (coords int32 [n,3], feats f32 [n,c_in], sorted) clouds. Every CONV op's GMaS gather /
        scatter tiles are profiled on each sample (1 warm-up + R rounds, median), medians summed
        over the samples, argmin kept (smallest tile on ties) and used by later GMaS forwards.
        Returns {op index: TunedLayerConfig dict(gather_tile, scatter_tile, gather_ms{T: ms},
        scatter_ms{T: ms})}."""
        keep = []
        xyz_p, n_v, srt, f_p = [], [], [], []
        for c, f, srt_i in samples:
            c = np.ascontiguousarray(c, np.int32)
            f = np.ascontiguousarray(f, np.float32)
            keep += [c, f]
            xyz_p.append(c.ctypes.data)
            f_p.append(f.ctypes.data)
            n_v.append(len(c))
            srt.append(int(srt_i))
        k = len(samples)
        arr_p = (C.c_void_p * max(1, k))(*xyz_p)
        arr_f = (C.c_void_p * max(1, k))(*f_p)
        arr_n = (C.c_int64 * max(1, k))(*n_v)
        arr_s = (C.c_int * max(1, k))(*srt)
        tiles = np.zeros(2 * len(self.g.ops), np.int32)
        self.ctx.check(self.ctx.lib.sconv_net_autotune(self.ctx.h, self.h, k, C.cast(arr_p, C.c_void_p),
                                                       C.cast(arr_n, C.c_void_p), C.cast(arr_s, C.c_void_p),
                                                       C.cast(arr_f, C.c_void_p), self.g.in_channels, rounds,
                                                       S._ptr(tiles)))
        out = {}
        for i, o in enumerate(self.g.ops):
            if o.kind != CONV:
                continue
            cap = 64
            t = np.zeros(cap, np.int32)
            ms = np.zeros(cap, np.float64)
            ng, ns = C.c_int(), C.c_int()
            self.ctx.check(self.ctx.lib.sconv_net_tune_latencies(self.h, i, S._ptr(t), S._ptr(ms), cap, C.byref(ng),
                                                                 C.byref(ns)))
            g, s_ = ng.value, ns.value
            out[i] = dict(gather_tile=int(tiles[2 * i]), scatter_tile=int(tiles[2 * i + 1]),
                          gather_ms={int(a): float(b) for a, b in zip(t[:g], ms[:g])},
                          scatter_ms={int(a): float(b) for a, b in zip(t[g:g + s_], ms[g:g + s_])})
        return out

    def algo_bytes(self, part_bytes=2):
        """Algorithmic bytes per kernel type summed over the convs (SURVEY §8d with this path's dtypes:
        16-bit activations, 16-bit gather buffer, `part_bytes` GEMM partials, 16-bit outputs).
        Fused convs: input rows read once (2*ci*n), the nbr table (4*K3*q), output (+residual) once,
        the weights once (2*K3*ci*co)."""
        g = e = s = f = 0
        maps = {}  # distinct searched maps (identity 1x1 maps need no search): SURVEY §8d Map bytes
        eq1 = {}  # distinct Eq. 1 output sets (strided convs / downsamples): floor + sort + unique
        for st in self.conv_stats():
            n, q, M, R, ci, co, kp, K3, df, res = (st[k] for k in self.STAT_KEYS)
            if K3 > 1:
                # (+ 12|P| + 8|Q| for an Eq. 1 downsample, which creates the smaller output set)
                maps[(n, q, M, K3)] = 8 * n + 8 * q + 8 * M + 4 * K3 + ((12 * n + 8 * q) if q < n else 0)
            if q < n:
                eq1[(n, q)] = 12 * n + 8 * q  # read |P| keys + indices, write |Q| keys
            if df == 1:
                f += 2 * ci * n + 4 * K3 * q + 2 * co * q * (2 if res else 1) + 2 * K3 * ci * co
                continue
            g += 2 * ci * n + 2 * kp * R + 4 * M
            e += 2 * kp * R + part_bytes * co * R + 2 * K3 * ci * co
            s += part_bytes * co * M + 4 * K3 * q + 2 * co * q * (2 if res else 1)
        return {"k_gather": g, "k_gemm_grouped": e, "k_scatter": s, "k_conv_fused": f,
                "k_search": sum(maps.values()), "_k_search_launches": len(maps),
                "k_floor_unique": sum(eq1.values()), "_k_floor_unique_launches": len(eq1)}

    def free(self):
        if self.h:
            self.ctx.lib.sconv_net_free(self.ctx.h, self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
