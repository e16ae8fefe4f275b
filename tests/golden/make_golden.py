#!/usr/bin/env python3
"""Generate tests/golden/*.json from the REFERENCE build of the oracle
(oracle/_ref/liboracle_ref.so: the oracle compiled against /root/reference's own
proj/include/sconv/geometry.hpp + prng.hpp). Run here (needs /root/reference):

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures are committed; tests compare the self-contained restatement
(oracle/liboracle.so) and the product library against them on machines without the
reference (the GPU box).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import OracleError, load_ref_oracle  # noqa: E402


def main():
    ref = load_ref_oracle()
    if ref is None:
        raise SystemExit("oracle/_ref/liboracle_ref.so missing: run `make -C oracle ref` where /root/reference exists")
    rng = np.random.default_rng(20240111)
    M = 2 ** 20 - 1
    coords = [[0, 0, 0], [0, 0, 1], [0, 1, 0], [0, 0, M], [-5, 3, M], [M, M, M], [-M, -M, -M], [1, -1, 7]]
    coords += rng.integers(-M, M + 1, size=(40, 3)).tolist()
    keys = ref.pack_keys(np.array(coords, np.int32))
    out = {"source": "oracle/_ref/liboracle_ref.so (reference geometry.hpp/prng.hpp)"}
    out["pack_key"] = {"coords": coords, "keys": [str(int(k)) for k in keys]}
    errs = []
    for c in ([M + 1, 0, 0], [0, -M - 1, 0], [0, 0, 2 ** 21], [M + 1, M + 1, 0]):
        try:
            ref.pack_keys(np.array([c], np.int32))
            errs.append({"coord": c, "error": None})
        except OracleError as e:
            errs.append({"coord": c, "status": e.status, "error": str(e)})
    out["pack_key_errors"] = errs
    wo = []
    for K, s in [(1, 1), (1, 7), (3, 1), (3, 2), (5, 2), (5, 1), (7, 3)]:
        wo.append({"K": K, "s": s, "offsets": ref.weight_offsets(K, s).tolist()})
    for K, s in [(2, 1), (0, 1), (3, 0)]:
        try:
            ref.weight_offsets(K, s)
        except OracleError as e:
            wo.append({"K": K, "s": s, "status": e.status, "error": str(e)})
    out["weight_offsets"] = wo
    goc = []
    clouds = [[[3, 5, 7]], [[0, 0, 0], [1, 1, 1]], [[-1, -3, 2], [-2, -4, 3], [5, 5, 5]]]
    clouds.append(rng.integers(-20, 20, size=(60, 3)).tolist())
    for cl in clouds:
        for s in (1, 2, 3):
            q, srt, al = ref.generate_output_coords(np.array(cl, np.int32), False, s)
            goc.append({"coords": cl, "s": s, "out": q.tolist(), "sorted": srt, "aliased": al})
    out["generate_output_coords"] = goc
    vox = []
    cases = [([[0.4, 0.4, 0.4], [0.6, 0.6, 0.6]], None, 0.5), ([[0.1, 0, 0], [0.2, 0, 0]], [[2.0], [4.0]], 1.0)]
    pts = (rng.random((50, 3)) * 4 - 2).round(3)
    feats = rng.random((50, 2)).round(3)
    cases.append((pts.tolist(), feats.tolist(), 0.5))
    for p, f, r in cases:
        fa = np.zeros((len(p), 0), np.float32) if f is None else np.array(f, np.float32)
        xyz, of = ref.voxelize(np.array(p), fa, r)
        vox.append({"points": p, "features": f, "resolution": r, "coords": xyz.tolist(),
                    "out_features": of.astype(float).tolist()})
    out["voxelize"] = vox
    out["rng"] = {
        "stream_seed": [[s, i, str(ref.stream_seed(s, i))] for s, i in [(1, 0), (1, 1), (42, 7), (2 ** 63, 3)]],
        "next": {str(seed): [str(int(v)) for v in ref.rng(seed, 8, 0)] for seed in (0, 1, 12345)},
        "next_unit": {str(seed): [float(v) for v in ref.rng(seed, 8, 1)] for seed in (0, 1)},
        "next_below": {f"{seed}:{b}": [str(int(v)) for v in ref.rng(seed, 8, 2, b)] for seed, b in
                       [(1, 400), (7, 3), (9, 2 ** 40 + 1)]},
    }
    # a tiny kernel map pinned by brute force on the reference build
    two = np.array([[0, 0, 0], [0, 0, 1]], np.int32)
    q, sizes, j, i, _ = ref.layer_map(two, True, 3, 1, 1, backend=2)
    out["kernel_map_two_points"] = {"coords": two.tolist(), "sizes": sizes.tolist(), "in": j.tolist(),
                                    "out": i.tolist()}
    with open(os.path.join(HERE, "geometry_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", os.path.join(HERE, "geometry_golden.json"))


if __name__ == "__main__":
    main()
