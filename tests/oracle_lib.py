"""ctypes access to the CPU oracle (oracle/liboracle.so) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import this.
"""
import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE = os.path.join(ROOT, "oracle", "liboracle.so")
ORACLE_REF = os.path.join(ROOT, "oracle", "_ref", "liboracle_ref.so")

_P, _I, _I64, _U64, _D = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double
_SIGS = {
    "so_last_error": (C.c_char_p, []),
    "so_pack_keys": (_I, [_P, _I64, _P]),
    "so_unpack_keys": (_I, [_P, _I64, _P]),
    "so_saturating_pack": (_I, [_P, _I64, _P]),
    "so_weight_offsets": (_I, [_I, _I, _I, _P, C.POINTER(_I64)]),
    "so_generate_output_coords": (_I, [_P, _I64, _I, _I, _P, C.POINTER(_I64), C.POINTER(_I), C.POINTER(_I)]),
    "so_voxelize": (_I, [_P, _I64, _P, _I64, _D, _P, _P, C.POINTER(_I64)]),
    "so_stream_seed": (_U64, [_U64, _U64]),
    "so_rng_draw": (_I, [_U64, _I64, _I, _U64, _P]),
    "so_generate_synthetic": (_I, [_I64, _I64, _I64, _U64, _P, _P]),
    "so_generate_weights": (_I, [_U64, _U64, _I, _I, _I, _P]),
    "so_map_build": (_I, [_P, _I64, _I, _P, _I64, _P, _I, _I, _I, _I, _I, C.POINTER(_P), _P]),
    "so_layer_map": (_I, [_P, _I64, _I, _I, _I, _I, _I, _P, _I64, _I, _I, _I, _I, C.POINTER(_P), _P]),
    "so_map_nq": (_I64, [_P]),
    "so_map_nk": (_I, [_P]),
    "so_map_total": (_I64, [_P]),
    "so_map_q": (_I, [_P, _P]),
    "so_map_read": (_I, [_P, _P, _P, _P]),
    "so_map_free": (None, [_P]),
    "so_group_gemms": (_I, [_P, _I, _I, _D, _I, _P, C.POINTER(_I), _P, _P, _P, C.POINTER(_I), _P, C.POINTER(_I64),
                            C.POINTER(_D)]),
    "so_layer_forward": (_I, [_P, _I64, _I, _P, _I, _P, _I, _I, _I, _I, _I, _P, _I64, _I, _I, _D, _I, _I, _I, _I, _I,
                              _I, _P, _P, C.POINTER(_I64), _P]),
    "so_dense_conv": (_I, [_P, _I64, _I, _P, _I, _P, _I, _I, _I, _I, _I, _P, _I64, _P, C.POINTER(_I64)]),
    "so_forward_network": (_I, [_P, _I, _P, _I64, _I, _P, _U64, _I, _I, _P, _P, C.POINTER(_I64), C.POINTER(_U64)]),
    "so_candidate_tiles": (_I, [_I, _P, C.POINTER(_I)]),
    "so_theoretical_hyperparams": (_I, [_I64, _I64, C.POINTER(_I), C.POINTER(_I)]),
}


class OracleError(Exception):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Oracle:
    def __init__(self, path=ORACLE):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(self.lib, name)
            fn.restype, fn.argtypes = res, args

    def _chk(self, st):
        if st != 0:
            raise OracleError(st, self.lib.so_last_error().decode())

    # ---- geometry
    def pack_keys(self, xyz):
        xyz = np.ascontiguousarray(xyz, np.int32).reshape(-1, 3)
        out = np.empty(len(xyz), np.uint64)
        self._chk(self.lib.so_pack_keys(_p(xyz), len(xyz), _p(out)))
        return out

    def unpack_keys(self, keys):
        keys = np.ascontiguousarray(keys, np.uint64)
        out = np.empty((len(keys), 3), np.int32)
        self._chk(self.lib.so_unpack_keys(_p(keys), len(keys), _p(out)))
        return out

    def saturating_pack(self, xyz):
        xyz = np.ascontiguousarray(xyz, np.int64).reshape(-1, 3)
        out = np.empty(len(xyz), np.uint64)
        self._chk(self.lib.so_saturating_pack(_p(xyz), len(xyz), _p(out)))
        return out

    def weight_offsets(self, K, s, ext=False):
        n = C.c_int64()
        self._chk(self.lib.so_weight_offsets(K, s, int(ext), None, C.byref(n)))
        out = np.empty((n.value, 3), np.int32)
        self._chk(self.lib.so_weight_offsets(K, s, int(ext), _p(out), C.byref(n)))
        return out

    def generate_output_coords(self, xyz, sorted_, s):
        xyz = np.ascontiguousarray(xyz, np.int32).reshape(-1, 3)
        out = np.empty_like(xyz)
        n, srt, al = C.c_int64(), C.c_int(), C.c_int()
        self._chk(self.lib.so_generate_output_coords(_p(xyz), len(xyz), int(sorted_), s, _p(out), C.byref(n),
                                                     C.byref(srt), C.byref(al)))
        return out[: n.value], bool(srt.value), bool(al.value)

    def voxelize(self, pts, feats, res):
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        feats = np.ascontiguousarray(feats, np.float32).reshape(len(pts), -1)
        Cc = feats.shape[1]
        oxyz = np.empty((len(pts), 3), np.int32)
        of = np.empty((len(pts), Cc), np.float32)
        n = C.c_int64()
        self._chk(self.lib.so_voxelize(_p(pts), len(pts), _p(feats), Cc, res, _p(oxyz), _p(of), C.byref(n)))
        return oxyz[: n.value], of[: n.value]

    def rng(self, seed, n, kind=0, bound=0):
        out = np.empty(n, np.float64 if kind == 1 else np.uint64)
        self._chk(self.lib.so_rng_draw(seed, n, kind, bound, _p(out)))
        return out

    def stream_seed(self, seed, idx):
        return int(self.lib.so_stream_seed(seed, idx))

    def generate_synthetic(self, N, E, Cch, seed):
        xyz = np.empty((N, 3), np.int32)
        f = np.empty((N, Cch), np.float32)
        self._chk(self.lib.so_generate_synthetic(N, E, Cch, seed, _p(xyz), _p(f)))
        return xyz, f

    def generate_weights(self, seed, stream, K3, cin, cout):
        w = np.empty((K3, cin, cout), np.float32)
        self._chk(self.lib.so_generate_weights(seed, stream, K3, cin, cout, _p(w)))
        return w

    # ---- maps
    def _read_map(self, h, counters):
        nq = self.lib.so_map_nq(h)
        nk = self.lib.so_map_nk(h)
        tot = self.lib.so_map_total(h)
        q = np.empty((nq, 3), np.int32)
        sizes = np.empty(nk, np.int64)
        j = np.empty(tot, np.int32)
        i = np.empty(tot, np.int32)
        self._chk(self.lib.so_map_q(h, _p(q)))
        self._chk(self.lib.so_map_read(h, _p(sizes), _p(j), _p(i)))
        self.lib.so_map_free(h)
        return q, sizes, j, i, counters

    def layer_map(self, xyz, sorted_, K=3, offset_scale=1, out_stride=1, transposed=False, target=None,
                  backend=0, B=256, Cq=512, workers=1):
        xyz = np.ascontiguousarray(xyz, np.int32).reshape(-1, 3)
        tgt = None if target is None else np.ascontiguousarray(target, np.int32).reshape(-1, 3)
        h = C.c_void_p()
        counters = np.zeros(5, np.uint64)
        self._chk(self.lib.so_layer_map(_p(xyz), len(xyz), int(sorted_), K, offset_scale, out_stride, int(transposed),
                                        _p(tgt), 0 if tgt is None else len(tgt), backend, B, Cq, workers, C.byref(h),
                                        _p(counters)))
        return self._read_map(h, counters)

    def map_build(self, P, P_sorted, Q, offsets, backend=0, B=256, Cq=512, workers=1):
        """build_kernel_map_sorted(P, Q, offsets, B, C) over explicit queries and offsets; backend
        0 sorted (counters), 1 hash, 2 brute force. Returns (Q, sizes, j, i, counters[5])."""
        P = np.ascontiguousarray(P, np.int32).reshape(-1, 3)
        Q = np.ascontiguousarray(Q, np.int32).reshape(-1, 3)
        offs = np.ascontiguousarray(offsets, np.int32).reshape(-1, 3)
        h = C.c_void_p()
        counters = np.zeros(5, np.uint64)
        self._chk(self.lib.so_map_build(_p(P), len(P), int(P_sorted), _p(Q), len(Q), _p(offs), len(offs), backend, B,
                                        Cq, workers, C.byref(h), _p(counters)))
        return self._read_map(h, counters)

    def forward_network(self, layers, xyz, sorted_, feats, seed, workers=1):
        """SPEC forward_network over a sequential NetworkSpec (K, s, c_in, c_out) per layer ->
        (coords, feats, sorts)."""
        L = np.ascontiguousarray(layers, np.int32).reshape(-1, 4)
        xyz = np.ascontiguousarray(xyz, np.int32).reshape(-1, 3)
        feats = np.ascontiguousarray(feats, np.float32)
        oxyz = np.empty((max(len(xyz), 1), 3), np.int32)
        of = np.empty((max(len(xyz), 1), int(L[-1, 3])), np.float32)
        n, sorts = C.c_int64(), C.c_uint64()
        self._chk(self.lib.so_forward_network(_p(L), len(L), _p(xyz), len(xyz), int(sorted_), _p(feats), seed, 0,
                                              workers, _p(oxyz), _p(of), C.byref(n), C.byref(sorts)))
        return oxyz[: n.value], of[: n.value], sorts.value

    def theoretical_hyperparams(self, P, Q):
        b, c = C.c_int(), C.c_int()
        self._chk(self.lib.so_theoretical_hyperparams(P, Q, C.byref(b), C.byref(c)))
        return b.value, c.value

    def group_gemms(self, sizes, policy=1, eps=0.25, max_batch=16):
        sizes = np.ascontiguousarray(sizes, np.int64)
        n = len(sizes)
        order = np.empty(n, np.int32)
        gb, ge = np.empty(n, np.int32), np.empty(n, np.int32)
        hts = np.empty(n, np.int64)
        boff = np.empty(n, np.int64)
        no, ng, blen, ovh = C.c_int(), C.c_int(), C.c_int64(), C.c_double()
        self._chk(self.lib.so_group_gemms(_p(sizes), n, policy, eps, max_batch, _p(order), C.byref(no), _p(gb), _p(ge),
                                          _p(hts), C.byref(ng), _p(boff), C.byref(blen), C.byref(ovh)))
        return dict(order=order[: no.value], groups=list(zip(gb[: ng.value], ge[: ng.value], hts[: ng.value])),
                    buffer_offsets=boff, buffer_length=blen.value, overhead=ovh.value)

    def layer_forward(self, xyz, sorted_, feats, W, K=3, offset_scale=1, out_stride=1, transposed=False, target=None,
                      backend=0, policy=1, eps=0.25, max_batch=16, Tg=0, Ts=0, B=256, Cq=512, workers=1):
        xyz = np.ascontiguousarray(xyz, np.int32).reshape(-1, 3)
        feats = np.ascontiguousarray(feats, np.float32)
        W = np.ascontiguousarray(W, np.float32)
        tgt = None if target is None else np.ascontiguousarray(target, np.int32).reshape(-1, 3)
        cap = len(xyz) if tgt is None else len(tgt)
        oxyz = np.empty((max(cap, 1), 3), np.int32)
        of = np.empty((max(cap, 1), W.shape[2]), np.float32)
        n = C.c_int64()
        stats = np.zeros(10, np.float64)
        self._chk(self.lib.so_layer_forward(_p(xyz), len(xyz), int(sorted_), _p(feats), W.shape[1], _p(W), W.shape[2],
                                            K, offset_scale, out_stride, int(transposed), _p(tgt),
                                            0 if tgt is None else len(tgt), backend, policy, eps, max_batch, Tg, Ts, B,
                                            Cq, workers, _p(oxyz), _p(of), C.byref(n), _p(stats)))
        keys = ["matches", "buffer_length", "groups", "padding_overhead", "imt_lookups", "sorts", "ms_map",
                "ms_gather", "ms_gemm", "ms_scatter"]
        return oxyz[: n.value], of[: n.value], dict(zip(keys, stats.tolist()))

    def dense_conv(self, xyz, sorted_, feats, W, K=3, offset_scale=1, out_stride=1, transposed=False, target=None):
        xyz = np.ascontiguousarray(xyz, np.int32).reshape(-1, 3)
        feats = np.ascontiguousarray(feats, np.float32)
        W = np.ascontiguousarray(W, np.float32)
        tgt = None if target is None else np.ascontiguousarray(target, np.int32).reshape(-1, 3)
        cap = len(xyz) if tgt is None else len(tgt)
        of = np.empty((max(cap, 1), W.shape[2]), np.float32)
        n = C.c_int64()
        self._chk(self.lib.so_dense_conv(_p(xyz), len(xyz), int(sorted_), _p(feats), W.shape[1], _p(W), W.shape[2], K,
                                         offset_scale, out_stride, int(transposed), _p(tgt),
                                         0 if tgt is None else len(tgt), _p(of), C.byref(n)))
        return of[: n.value]


def load_oracle():
    return Oracle(ORACLE)


def load_ref_oracle():
    return Oracle(ORACLE_REF) if os.path.exists(ORACLE_REF) else None
