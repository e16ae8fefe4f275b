"""ctypes binding of libsconv_b200 (include/sconv_b200.h).

Mirrors the reference SC-layer API (namespace ``sconv`` in
proj/include/sconv/geometry.hpp plus the SPEC.md operation signatures) for Python
callers: ``PointCloud``, ``weight_offsets``, ``build_kernel_map_sorted``,
``sc_layer_forward``, ``generate_synthetic``. Reference exceptions map to
``InvalidArgument`` (std::invalid_argument), ``OutOfRange`` (std::out_of_range) and
``LogicError`` (std::logic_error) with identical message text.

There is no CPU fallback: if the CUDA library is missing this module raises on import
of the library (``load()``), and every compute call goes through the sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
import weakref
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsconv_b200.so")
# SCONV_LIB overrides the library path (A/B measurements of two builds on the same box)
LIB_PATH = os.environ.get("SCONV_LIB", LIB_PATH)

OK, ERR_ARG, ERR_RANGE, ERR_CUDA, ERR_OOM, ERR_STATE = range(6)
MEM_HOST, MEM_DEVICE = 0, 1
F32, F16, BF16 = 0, 1, 2
GROUP_MAP_ORDER, GROUP_SORTED = 0, 1
DATAFLOW_GMAS, DATAFLOW_FUSED, DATAFLOW_AUTO = 0, 1, 2
MAP_SORTED, MAP_HASH, MAP_SORTED_SPEC = 0, 1, 2


class SconvError(RuntimeError):
    pass


class InvalidArgument(SconvError, ValueError):
    pass


class OutOfRange(SconvError, IndexError):
    pass


class CudaError(SconvError):
    pass


class LogicError(SconvError):
    pass


class MapCfg(C.Structure):
    _fields_ = [("kernel_size", C.c_int), ("offset_scale", C.c_int), ("out_stride", C.c_int),
                ("transposed", C.c_int), ("block_B", C.c_int), ("block_C", C.c_int), ("backend", C.c_int)]


class ExecCfg(C.Structure):
    _fields_ = [("policy", C.c_int), ("epsilon", C.c_double), ("max_batch", C.c_int),
                ("gather_tile", C.c_int), ("scatter_tile", C.c_int), ("compute_dtype", C.c_int),
                ("partial_f16", C.c_int), ("dataflow", C.c_int), ("fuse_residual", C.c_int)]


class MapInfo(C.Structure):
    _fields_ = [("num_inputs", C.c_int64), ("num_outputs", C.c_int64), ("num_offsets", C.c_int32),
                ("total_matches", C.c_int64), ("buffer_length", C.c_int64), ("groups", C.c_int32),
                ("padding_overhead", C.c_double), ("gather_tile", C.c_int32), ("scatter_tile", C.c_int32)]


_lib = None

# (name, restype, argtypes) for every entry point declared in include/sconv_b200.h
_P, _I, _I64, _U64, _D, _S = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double, C.c_size_t
SIGNATURES = [
    ("sconv_ctx_create", _I, [_I, C.POINTER(_P)]),
    ("sconv_ctx_destroy", None, [_P]),
    ("sconv_last_error", C.c_char_p, [_P]),
    ("sconv_ctx_set_stream", _I, [_P, _P]),
    ("sconv_ctx_stream", _P, [_P]),
    ("sconv_ctx_synchronize", _I, [_P]),
    ("sconv_ctx_launch_count", _I64, [_P]),
    ("sconv_ctx_set_lookup_counting", _I, [_P, _I]),
    ("sconv_ctx_lookup_count", _I, [_P, C.POINTER(_U64)]),
    ("sconv_ctx_set_profiling", _I, [_P, _I]),
    ("sconv_ctx_set_profile_filter", _I, [_P, C.c_char_p]),
    ("sconv_ctx_profile_count", _I, [_P]),
    ("sconv_ctx_profile_entry", _I, [_P, _I, C.POINTER(C.c_char_p), C.POINTER(_I64), C.POINTER(_D)]),
    ("sconv_ctx_profile_reset", _I, [_P]),
    ("sconv_ctx_flush_l2", _I, [_P, _S]),
    ("sconv_device_alloc", _I, [_P, _S, C.POINTER(_P)]),
    ("sconv_device_free", _I, [_P, _P]),
    ("sconv_memcpy", _I, [_P, _P, _P, _S, _I]),
    ("sconv_map_build", _I, [_P, _P, _I64, _I, _I, C.POINTER(MapCfg), _P, _I64, _I, C.POINTER(_P)]),
    ("sconv_map_build_explicit", _I, [_P, _P, _I64, _I, _I, _P, _I64, _I, _P, _I, _I, _I, _I, C.POINTER(_P)]),
    ("sconv_map_search_counters", _I, [_P, _P, C.c_void_p]),
    ("sconv_theoretical_hyperparams", _I, [_I64, _I64, C.POINTER(_I), C.POINTER(_I)]),
    ("sconv_map_build_chained", _I, [_P, _P, C.POINTER(MapCfg), _P, C.POINTER(_P)]),
    ("sconv_map_get_info", _I, [_P, _P, C.POINTER(MapInfo)]),
    ("sconv_map_read", _I, [_P, _P, _P, _P, _P, _P]),
    ("sconv_map_device_views", _I, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]),
    ("sconv_map_free", None, [_P, _P]),
    ("sconv_weights_create", _I, [_P, _P, _I, _I, _I, _I, _I, C.POINTER(_P)]),
    ("sconv_weights_free", None, [_P, _P]),
    ("sconv_layer_forward", _I, [_P, _P, _P, _P, _I, _I, C.POINTER(ExecCfg), _P, _I, _I]),
    ("sconv_tune_layer", _I, [_P, _P, _P, _P, _I, _I, C.POINTER(_I), C.POINTER(_I), _P, C.POINTER(_I)]),
    ("sconv_sc_layer_forward", _I, [_P, _P, _I64, _I, _P, _I, _P, _I, _I, _I, C.POINTER(ExecCfg), _P,
                                    C.POINTER(_I64), _P]),
    ("sconv_plan_groups", _I, [_P, _I, _I, _D, _I, _P, C.POINTER(_I), _P, _P, _P, C.POINTER(_I), _P,
                               C.POINTER(_I64), C.POINTER(_D)]),
    ("sconv_net_create", _I, [_P, _P, _I, _I, _I, _I, C.POINTER(ExecCfg), _I, _I, C.POINTER(_P)]),
    ("sconv_net_set_weights", _I, [_P, _P, _I, _P, _I, _I, _I, _I]),
    ("sconv_net_forward", _I, [_P, _P, _P, _I64, _I, _I, _P, _I, _I]),
    ("sconv_net_tensor_info", _I, [_P, _P, _I, C.POINTER(_I64), C.POINTER(_I), C.POINTER(_I)]),
    ("sconv_net_read_tensor", _I, [_P, _P, _I, _P, _P]),
    ("sconv_net_tensor_device", _I, [_P, _I, C.POINTER(_P), C.POINTER(_I), C.POINTER(_I64)]),
    ("sconv_net_copy_tensor", _I, [_P, _P, _I, _P, _I, _I]),
    ("sconv_net_read_async", _I, [_P, _P, _I, _P]),
    ("sconv_net_prefetch_inputs", _I, [_P, _P, _P, _I64, _P, _I, _I]),
    ("sconv_net_read_wait", _I, [_P, _P]),
    ("sconv_net_sort_count", _I, [_P, C.POINTER(_I64)]),
    ("sconv_net_conv_timings", _I, [_P, _I, C.POINTER(_D), C.POINTER(_D)]),
    ("sconv_voxelize", _I, [_P, _P, _I64, _I, _P, _I64, _I, _D, _P, _P, _I, C.POINTER(_I64)]),
    ("sconv_net_stats", _I, [_P, C.POINTER(_I), C.POINTER(_I)]),
    ("sconv_net_conv_stats", _I, [_P, _I, _P]),
    ("sconv_net_resolve_stats", _I, [_P, _P]),
    ("sconv_net_autotune", _I, [_P, _P, _I, _P, _P, _P, _P, _I, _I, _P]),
    ("sconv_net_tune_latencies", _I, [_P, _I, _P, _P, _I, C.POINTER(_I), C.POINTER(_I)]),
    ("sconv_net_free", None, [_P, _P]),
    ("sconv_cloud_file_info", _I, [C.c_char_p, C.POINTER(_I), C.POINTER(_I64), C.POINTER(_I64)]),
    ("sconv_mpc_read", _I, [C.c_char_p, _P, _P, _I64, _I64]),
    ("sconv_mpc_write", _I, [C.c_char_p, _P, _P, _I64, _I64]),
    ("sconv_xyz_read", _I, [C.c_char_p, _P, _P, _I64, _I64]),
    ("sconv_xyz_write", _I, [C.c_char_p, _P, _P, _I64, _I64]),
    ("sconv_generate_synthetic", _I, [_I64, _I64, _I64, _U64, _P, _P]),
    ("sconv_generate_weights", _I, [_U64, _U64, _I, _I, _I, _P]),
    ("sconv_global_last_error", C.c_char_p, []),
    ("sconv_version", C.c_char_p, []),
]


def load(path: str = LIB_PATH):
    """Load the CUDA library (raises if it was not built: there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libsconv_b200.so not built at {path}; run `make` (or __graft_entry__.build())")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _raise(status: int, msg: str):
    cls = {ERR_ARG: InvalidArgument, ERR_RANGE: OutOfRange, ERR_CUDA: CudaError, ERR_OOM: CudaError,
           ERR_STATE: LogicError}.get(status, SconvError)
    raise cls(msg)


class Context:
    """One context per (host thread, device); calls are serialised on its stream."""

    def __init__(self, device: int = 0):
        self.lib = load()
        h = C.c_void_p()
        st = self.lib.sconv_ctx_create(device, C.byref(h))
        if st != OK:
            _raise(st, self.lib.sconv_global_last_error().decode())
        self.h = h
        self._children = weakref.WeakSet()  # maps / weights / networks: freed before the context

    def adopt(self, obj):
        self._children.add(obj)
        return obj

    def check(self, st: int):
        if st != OK:
            _raise(st, self.lib.sconv_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            for c in list(getattr(self, "_children", ())):  # device objects die before their context
                try:
                    c.free()
                except Exception:
                    pass
            self.lib.sconv_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: Optional[int]):
        self.check(self.lib.sconv_ctx_set_stream(self.h, stream_handle))

    def synchronize(self):
        self.check(self.lib.sconv_ctx_synchronize(self.h))

    def count_lookups(self, enabled: bool = True):
        """Gather IMT-lookup counting on / off (SPEC.md:340 counter)."""
        self.check(self.lib.sconv_ctx_set_lookup_counting(self.h, int(enabled)))

    def lookup_count(self) -> int:
        """IMT lookups since the last call (resets; synchronises)."""
        v = C.c_uint64()
        self.check(self.lib.sconv_ctx_lookup_count(self.h, C.byref(v)))
        return int(v.value)

    @property
    def launch_count(self) -> int:
        return int(self.lib.sconv_ctx_launch_count(self.h))

    def set_profiling(self, on: bool):
        self.check(self.lib.sconv_ctx_set_profiling(self.h, 1 if on else 0))

    def set_profile_filter(self, label: Optional[str]):
        self.check(self.lib.sconv_ctx_set_profile_filter(self.h, label.encode() if label else None))

    def profile(self) -> dict:
        self.synchronize()  # resolves pending per-launch events
        out = {}
        for i in range(self.lib.sconv_ctx_profile_count(self.h)):
            name, n, ms = C.c_char_p(), C.c_int64(), C.c_double()
            self.check(self.lib.sconv_ctx_profile_entry(self.h, i, C.byref(name), C.byref(n), C.byref(ms)))
            out[name.value.decode()] = (int(n.value), float(ms.value))
        return out

    def profile_reset(self):
        self.check(self.lib.sconv_ctx_profile_reset(self.h))

    def flush_l2(self, nbytes: int = 256 << 20):
        self.check(self.lib.sconv_ctx_flush_l2(self.h, nbytes))


def map_cfg(K=3, offset_scale=1, out_stride=1, transposed=False, B=256, Cq=512, backend=0) -> MapCfg:
    """backend: MAP_SORTED (Minuet double-traversed search) or MAP_HASH (SPEC hash baseline)."""
    return MapCfg(K, offset_scale, out_stride, 1 if transposed else 0, B, Cq, backend)


def exec_cfg(policy=GROUP_SORTED, epsilon=0.25, max_batch=16, gather_tile=0, scatter_tile=0,
             compute_dtype=F16, partial_f16=0, dataflow=None, fuse_residual=1) -> ExecCfg:
    """dataflow: GMAS (Minuet gather/GEMM/scatter), FUSED (one output-stationary kernel) or
    AUTO (networks: per-conv choice by timing); None = GMAS for layers, AUTO for networks."""
    return ExecCfg(policy, epsilon, max_batch, gather_tile, scatter_tile, compute_dtype, partial_f16,
                   -1 if dataflow is None else dataflow, fuse_residual)


class SearchCountersC(C.Structure):
    _fields_ = [("backward_comparisons", C.c_uint64), ("forward_comparisons", C.c_uint64),
                ("source_elements_loaded", C.c_uint64), ("queries_executed", C.c_uint64), ("sorts", C.c_uint64),
                ("counted", C.c_int32)]


class KernelMap:
    """Device-resident kernel map + sorted output coordinates."""

    def __init__(self, ctx: Context, handle):
        self.ctx, self.h = ctx, handle
        ctx.adopt(self)

    @classmethod
    def build(cls, ctx: Context, coords, sorted_: bool = False, K=3, offset_scale=1, out_stride=1,
              transposed=False, target=None, B=256, Cq=512, device_ptr: Optional[int] = None, backend=0,
              n: Optional[int] = None) -> "KernelMap":
        cfg = map_cfg(K, offset_scale, out_stride, transposed, B, Cq, backend)
        h = C.c_void_p()
        tgt = None
        if target is not None:
            tgt = np.ascontiguousarray(target, dtype=np.int32).reshape(-1, 3)
        if device_ptr is not None:
            ctx.check(ctx.lib.sconv_map_build(ctx.h, device_ptr, n, MEM_DEVICE, int(sorted_), C.byref(cfg),
                                              _ptr(tgt), 0 if tgt is None else len(tgt), MEM_HOST, C.byref(h)))
        else:
            c = np.ascontiguousarray(coords, dtype=np.int32).reshape(-1, 3)
            ctx.check(ctx.lib.sconv_map_build(ctx.h, _ptr(c), len(c), MEM_HOST, int(sorted_), C.byref(cfg),
                                              _ptr(tgt), 0 if tgt is None else len(tgt), MEM_HOST, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def chained(cls, ctx: Context, prev: "KernelMap", K=3, offset_scale=1, out_stride=1, transposed=False,
                target_of: Optional["KernelMap"] = None, B=256, Cq=512) -> "KernelMap":
        cfg = map_cfg(K, offset_scale, out_stride, transposed, B, Cq)
        h = C.c_void_p()
        ctx.check(ctx.lib.sconv_map_build_chained(ctx.h, prev.h, C.byref(cfg),
                                                  None if target_of is None else target_of.h, C.byref(h)))
        return cls(ctx, h)

    def info(self) -> MapInfo:
        i = MapInfo()
        self.ctx.check(self.ctx.lib.sconv_map_get_info(self.ctx.h, self.h, C.byref(i)))
        return i

    @classmethod
    def build_explicit(cls, ctx: Context, P, P_sorted: bool, Q, offsets, B=256, Cq=512,
                       backend=0) -> "KernelMap":
        """SPEC build_kernel_map_sorted(P, Q, offsets, B, C): arbitrary sorted
        unique queries Q and an arbitrary offset list (host arrays)."""
        P = np.ascontiguousarray(P, np.int32).reshape(-1, 3)
        Q = np.ascontiguousarray(Q, np.int32).reshape(-1, 3)
        offs = np.ascontiguousarray(offsets, np.int32).reshape(-1, 3)
        h = C.c_void_p()
        ctx.check(ctx.lib.sconv_map_build_explicit(ctx.h, _ptr(P), len(P), MEM_HOST, int(P_sorted), _ptr(Q), len(Q),
                                                   MEM_HOST, _ptr(offs), len(offs), B, Cq, backend, C.byref(h)))
        return cls(ctx, h)

    def search_counters(self) -> dict:
        """SearchCounters: comparison tallies when built with MAP_SORTED_SPEC,
        plus the coordinate sorts the build performed."""
        c = SearchCountersC()
        self.ctx.check(self.ctx.lib.sconv_map_search_counters(self.ctx.h, self.h, C.byref(c)))
        return {f: getattr(c, f) for f, _ in SearchCountersC._fields_}

    def read(self):
        """(output coords [n_out,3], sizes [K3], in_idx [|M|], out_idx [|M|]) in canonical order."""
        inf = self.info()
        q = np.empty((inf.num_outputs, 3), np.int32)
        sizes = np.empty(inf.num_offsets, np.int64)
        j = np.empty(inf.total_matches, np.int32)
        i = np.empty(inf.total_matches, np.int32)
        self.ctx.check(self.ctx.lib.sconv_map_read(self.ctx.h, self.h, _ptr(q), _ptr(sizes), _ptr(j), _ptr(i)))
        return q, sizes, j, i

    def free(self):
        if self.h:
            self.ctx.lib.sconv_map_free(self.ctx.h, self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Weights:
    def __init__(self, ctx: Context, w: np.ndarray, dtype=F16):
        w = np.ascontiguousarray(w, dtype=np.float32)
        assert w.ndim == 3, "weights are [num_offsets, c_in, c_out]"
        self.ctx, self.shape, self.dtype = ctx, w.shape, dtype
        h = C.c_void_p()
        ctx.check(ctx.lib.sconv_weights_create(ctx.h, _ptr(w), MEM_HOST, w.shape[0], w.shape[1], w.shape[2],
                                               dtype, C.byref(h)))
        self.h = h
        ctx.adopt(self)

    def free(self):
        if self.h:
            self.ctx.lib.sconv_weights_free(self.ctx.h, self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def voxelize(ctx: Context, points: np.ndarray, features: Optional[np.ndarray], resolution: float) -> "PointCloud":
    """GPU voxelize (reference geometry.hpp:180-255): points [n, 3] float64, features [n, C] float32
    or None -> PointCloud of sorted voxel coordinates and mean-merged features (sorted=True)."""
    pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    n = len(pts)
    f = None if features is None else np.ascontiguousarray(features, np.float32).reshape(n, -1)
    ch = 0 if f is None else f.shape[1]
    oxyz = np.empty((max(n, 1), 3), np.int32)
    of = np.empty((max(n, 1), max(ch, 1)), np.float32)
    nv = C.c_int64()
    ctx.check(ctx.lib.sconv_voxelize(ctx.h, _ptr(pts), n, MEM_HOST, _ptr(f) if f is not None else None, ch, MEM_HOST,
                                     float(resolution), _ptr(oxyz), _ptr(of), MEM_HOST, C.byref(nv)))
    k = nv.value
    feats_out = of[:k, :ch].copy() if ch else np.zeros((k, 0), np.float32)
    return PointCloud(oxyz[:k].copy(), feats_out, True)


def layer_forward(ctx: Context, kmap: KernelMap, w: Weights, features: np.ndarray, cfg: Optional[ExecCfg] = None,
                  out_dtype=F32) -> np.ndarray:
    """GMaS on host arrays: features [n_in, c_in] fp32 (P order) -> [n_out, c_out] (Q order)."""
    f = np.ascontiguousarray(features, dtype=np.float32)
    inf = kmap.info()
    out = np.empty((inf.num_outputs, w.shape[2]), np.float32 if out_dtype == F32 else np.uint16)
    cfg = cfg or exec_cfg(compute_dtype=w.dtype)
    ctx.check(ctx.lib.sconv_layer_forward(ctx.h, kmap.h, w.h, _ptr(f), F32, MEM_HOST, C.byref(cfg), _ptr(out),
                                          out_dtype, MEM_HOST))
    return out


def layer_forward_device(ctx: Context, kmap: KernelMap, w: Weights, f_in_ptr: int, f_in_dtype: int,
                         f_out_ptr: int, f_out_dtype: int, cfg: Optional[ExecCfg] = None):
    cfg = cfg or exec_cfg(compute_dtype=w.dtype)
    ctx.check(ctx.lib.sconv_layer_forward(ctx.h, kmap.h, w.h, f_in_ptr, f_in_dtype, MEM_DEVICE, C.byref(cfg),
                                          f_out_ptr, f_out_dtype, MEM_DEVICE))


def tune_layer(ctx: Context, kmap: KernelMap, w: Weights, f_in_ptr: int, f_in_dtype=F32, rounds=5):
    tg, ts, n = C.c_int(), C.c_int(), C.c_int(64)
    lat = np.zeros(64, np.float64)
    ctx.check(ctx.lib.sconv_tune_layer(ctx.h, kmap.h, w.h, f_in_ptr, f_in_dtype, rounds, C.byref(tg), C.byref(ts),
                                       _ptr(lat), C.byref(n)))
    return tg.value, ts.value, lat[: n.value].copy()


# ---------------------------------------------------------------- reference-shaped API
@dataclass
class PointCloud:
    """Reference PointCloud (geometry.hpp:114-121): coords [N,3] int32, features [N,C] fp32."""
    coords: np.ndarray
    features: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.float32))
    sorted: bool = False

    def size(self) -> int:
        return len(self.coords)

    def channels(self) -> int:
        return self.features.shape[1] if self.features.ndim == 2 else 0


def weight_offsets(K: int, s: int) -> np.ndarray:
    """Reference weight_offsets (geometry.hpp:133-148): odd K only, lexicographic."""
    if K < 1 or K % 2 == 0:
        raise InvalidArgument("kernel size must be a positive odd integer")
    if s < 1:
        raise InvalidArgument("stride must be positive")
    h = K // 2
    t = np.arange(-h, h + 1, dtype=np.int32) * s
    return np.stack(np.meshgrid(t, t, t, indexing="ij"), -1).reshape(-1, 3)


def build_kernel_map_sorted(ctx: Context, P: PointCloud, K: int, s: int, B: int = 256, Cq: int = 512):
    """SPEC build_kernel_map_sorted for a SPEC-literal layer (Q = Eq. 1 coords of P with stride s).

    Returns (Q coords, list of K^3 arrays of (j, i) pairs sorted by i)."""
    m = KernelMap.build(ctx, P.coords, P.sorted, K, s, s, B=B, Cq=Cq)
    q, sizes, j, i = m.read()
    lists, pos = [], 0
    for n in sizes:
        lists.append(np.stack([j[pos:pos + n], i[pos:pos + n]], 1))
        pos += n
    m.free()
    return q, lists


def build_kernel_map_sorted_explicit(ctx: Context, P: "PointCloud", Q, offsets, B: int = 256, Cq: int = 512,
                                     backend: int = MAP_SORTED_SPEC):
    """SPEC build_kernel_map_sorted(P, Q, offsets, B, C) -> (KernelMap, SearchCounters): list of
    per-offset (j, i) arrays sorted by i, and the counters dict."""
    m = KernelMap.build_explicit(ctx, P.coords, P.sorted, Q, offsets, B, Cq, backend)
    _, sizes, j, i = m.read()
    lists, pos = [], 0
    for n in sizes:
        lists.append(np.stack([j[pos:pos + n], i[pos:pos + n]], 1))
        pos += n
    cnt = m.search_counters()
    m.free()
    return lists, cnt


def theoretical_hyperparams(num_inputs: int, num_outputs: int):
    """SPEC theoretical_hyperparams(|P|, |Q|) -> (B, C); advisory."""
    b, c = C.c_int(), C.c_int()
    lib = load()
    st = lib.sconv_theoretical_hyperparams(int(num_inputs), int(num_outputs), C.byref(b), C.byref(c))
    if st != OK:
        _raise(st, lib.sconv_global_last_error().decode())
    return b.value, c.value


def sc_layer_forward(ctx: Context, cloud: PointCloud, W: np.ndarray, K: int, s: int,
                     cfg: Optional[ExecCfg] = None, out_coords: Optional[np.ndarray] = None,
                     out_features: Optional[np.ndarray] = None) -> PointCloud:
    """SPEC sc_layer_forward through the one-shot C entry point.
    out_coords [n, 3] int32 / out_features [n, c_out] float32: optional caller buffers (e.g.
    pinned host memory, so the device->host copies are DMA at full link speed)."""
    xyz = np.ascontiguousarray(cloud.coords, dtype=np.int32).reshape(-1, 3)
    f = np.ascontiguousarray(cloud.features, dtype=np.float32)
    W = np.ascontiguousarray(W, dtype=np.float32)
    c_in, c_out = W.shape[1], W.shape[2]
    out_xyz = np.empty_like(xyz) if out_coords is None else out_coords
    out_f = np.empty((len(xyz), c_out), np.float32) if out_features is None else out_features
    if out_xyz.shape != xyz.shape or out_xyz.dtype != np.int32 or not out_xyz.flags.c_contiguous:
        raise InvalidArgument("out_coords must be a contiguous int32 [n, 3] array")
    if out_f.shape != (len(xyz), c_out) or out_f.dtype != np.float32 or not out_f.flags.c_contiguous:
        raise InvalidArgument("out_features must be a contiguous float32 [n, c_out] array")
    n_out = C.c_int64()
    cfg = cfg or exec_cfg()
    ctx.check(ctx.lib.sconv_sc_layer_forward(ctx.h, _ptr(xyz), len(xyz), int(cloud.sorted), _ptr(f), c_in, _ptr(W),
                                             c_out, K, s, C.byref(cfg), _ptr(out_xyz), C.byref(n_out), _ptr(out_f)))
    n = n_out.value
    if out_coords is not None or out_features is not None:
        return PointCloud(out_xyz[:n], out_f[:n], True)  # views of the caller's buffers
    return PointCloud(out_xyz[:n].copy(), out_f[:n].copy(), True)


def plan_groups(sizes, policy=GROUP_SORTED, epsilon=0.25, max_batch=16) -> dict:
    """SPEC group_gemms + padding_overhead through the library's planner."""
    lib = load()
    s = np.ascontiguousarray(sizes, np.int64)
    n = len(s)
    order, gb, ge = np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n, np.int32)
    heights, boff = np.empty(n, np.int64), np.empty(n, np.int64)
    no, ng, blen, ovh = C.c_int(), C.c_int(), C.c_int64(), C.c_double()
    st = lib.sconv_plan_groups(_ptr(s), n, policy, epsilon, max_batch, _ptr(order), C.byref(no), _ptr(gb), _ptr(ge),
                               _ptr(heights), C.byref(ng), _ptr(boff), C.byref(blen), C.byref(ovh))
    if st != OK:
        _raise(st, lib.sconv_global_last_error().decode())
    return dict(order=order[: no.value], groups=list(zip(gb[: ng.value], ge[: ng.value], heights[: ng.value])),
                buffer_offsets=boff, buffer_length=blen.value, overhead=ovh.value)


FILE_MPC, FILE_XYZ = 0, 1


def _gcheck(lib, st):
    if st != OK:
        _raise(st, lib.sconv_global_last_error().decode())


def cloud_file_info(path: str):
    """(format, N, C) of a point-cloud file: FILE_MPC (voxel coordinates) or FILE_XYZ (float points)."""
    lib = load()
    fmt, n, c = C.c_int(), C.c_int64(), C.c_int64()
    _gcheck(lib, lib.sconv_cloud_file_info(os.fsencode(path), C.byref(fmt), C.byref(n), C.byref(c)))
    return fmt.value, n.value, c.value


def read_cloud(path: str):
    """Read a SPEC.md:585 file. '.mpc' -> PointCloud (int32 voxel coordinates, sorted=False);
    '.xyz' -> (points [N,3] float64, features [N,C] float32), the input of ``voxelize``."""
    lib = load()
    fmt, n, c = cloud_file_info(path)
    f = np.empty((n, c), np.float32)
    if fmt == FILE_MPC:
        xyz = np.empty((n, 3), np.int32)
        _gcheck(lib, lib.sconv_mpc_read(os.fsencode(path), _ptr(xyz), _ptr(f), n, c))
        return PointCloud(xyz, f, False)
    pts = np.empty((n, 3), np.float64)
    _gcheck(lib, lib.sconv_xyz_read(os.fsencode(path), _ptr(pts), _ptr(f), n, c))
    return pts, f


def write_mpc(path: str, coords: np.ndarray, features: Optional[np.ndarray] = None):
    lib = load()
    xyz = np.ascontiguousarray(coords, np.int32).reshape(-1, 3)
    f = np.zeros((len(xyz), 0), np.float32) if features is None else np.ascontiguousarray(features, np.float32)
    _gcheck(lib, lib.sconv_mpc_write(os.fsencode(path), _ptr(xyz), _ptr(f), len(xyz), f.shape[1] if f.ndim == 2 else 0))


def write_xyz(path: str, points: np.ndarray, features: Optional[np.ndarray] = None):
    lib = load()
    pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    f = np.zeros((len(pts), 0), np.float32) if features is None else np.ascontiguousarray(features, np.float32)
    _gcheck(lib, lib.sconv_xyz_write(os.fsencode(path), _ptr(pts), _ptr(f), len(pts), f.shape[1] if f.ndim == 2 else 0))


def load_cloud(ctx: "Context", path: str, resolution: Optional[float] = None) -> "PointCloud":
    """File -> PointCloud ready for the layer/network API: an '.mpc' file is returned as stored;
    an '.xyz' file is voxelized on the GPU at ``resolution`` (required for '.xyz')."""
    fmt, _, _ = cloud_file_info(path)
    if fmt == FILE_MPC:
        return read_cloud(path)
    if resolution is None:
        raise InvalidArgument("resolution is required to voxelize an .xyz file")
    pts, f = read_cloud(path)
    return voxelize(ctx, pts, f if f.shape[1] else None, resolution)


def generate_synthetic(N: int, E: int, Cch: int, seed: int):
    lib = load()
    xyz = np.empty((N, 3), np.int32)
    f = np.empty((N, Cch), np.float32)
    st = lib.sconv_generate_synthetic(N, E, Cch, seed, _ptr(xyz), _ptr(f))
    if st != OK:
        _raise(st, lib.sconv_global_last_error().decode())
    return xyz, f


def generate_weights(seed: int, stream: int, K3: int, c_in: int, c_out: int) -> np.ndarray:
    lib = load()
    w = np.empty((K3, c_in, c_out), np.float32)
    st = lib.sconv_generate_weights(seed, stream, K3, c_in, c_out, _ptr(w))
    if st != OK:
        _raise(st, lib.sconv_global_last_error().decode())
    return w
