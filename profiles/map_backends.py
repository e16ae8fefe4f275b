#!/usr/bin/env python3
"""Minuet's Shortcoming #1 on B200 (the Fig. 2 / Fig. 12b analogue): the
sorted double-traversed search vs the SPEC's hash-table baseline, both on the GPU, building the
same canonical kernel map. Reports the search-stage kernel time per backend (CUDA events per
launch, median of 5) and checks the maps are identical. L2 hit rates come from ncu:
  ncu --metrics lts__t_sector_hit_rate.pct,gpu__time_duration.sum -k regex:"k_search|k_hash" \\
      python profiles/map_backends.py --ncu
"""
import argparse, os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2401_06145_b200 as sc
from paper_2401_06145_b200 import datasets as D

ap = argparse.ArgumentParser()
ap.add_argument("--ncu", action="store_true", help="one build per backend and cloud (for ncu)")
a = ap.parse_args()
ctx = sc.Context(0)
rng = np.random.default_rng(0)
clouds = {"kitti_120k_sorted (C2 L0)": (D.kitti_scan(0)[0], True),
          "s3dis_room_sorted (C3 L0)": (D.s3dis_room(0)[0], True)}
g = np.random.default_rng(1)
for n, e in ((100_000, 400), (1_000_000, 150), (10_000_000, 300)):
    flat = rng.choice(e ** 3, size=n, replace=False)
    clouds[f"uniform_{n:.0e}_in_{e}^3"] = (np.stack(np.unravel_index(flat, (e,) * 3), 1).astype(np.int32), False)
stages = {sc.MAP_SORTED: ("k_search",), sc.MAP_HASH: ("k_hash_insert", "k_hash_query")}
HBM = 6552.3  # MEASURED_PEAKS.json hbm_gbs


def algo_bytes(n_p, n_q, M, K3, strided=False):
    """SURVEY 8(d) Map algorithmic bytes: 8|P| + 8|Q| + 8|M| + 4 K^3 (+ 12|P| + 8|Q| for Eq. 1)."""
    return 8 * n_p + 8 * n_q + 8 * M + 4 * K3 + ((12 * n_p + 8 * n_q) if strided else 0)
for name, (xyz, srt) in clouds.items():
    res, maps, whole = {}, {}, {}
    for be in (sc.MAP_SORTED, sc.MAP_HASH):
        reps = 1 if a.ncu else 6
        ts, tw = [], []
        for r in range(reps):
            ctx.set_profiling(True)
            ctx.profile_reset()
            m = sc.KernelMap.build(ctx, xyz, srt, 3, 1, 1, backend=be)
            prof = ctx.profile()
            ctx.set_profiling(False)
            ts.append(sum(prof[k][1] for k in stages[be] if k in prof))
            tw.append(sum(v[1] for v in prof.values()))
            if r == reps - 1:
                maps[be] = m.read()
            m.free()
        res[be] = statistics.median(ts[1:] if len(ts) > 1 else ts)
        whole[be] = statistics.median(tw[1:] if len(tw) > 1 else tw)
    same = all(np.array_equal(x, y) for x, y in zip(maps[sc.MAP_SORTED], maps[sc.MAP_HASH]))
    M = int(maps[sc.MAP_SORTED][1].sum())
    ab = algo_bytes(len(xyz), len(maps[sc.MAP_SORTED][0]), M, 27)
    gbs = lambda ms: ab / (ms * 1e-3) / 1e9  # noqa: E731
    print(f"{name:28s} |P|={len(xyz):>9,} |M|={M:>10,} search: sorted {1e3 * res[sc.MAP_SORTED]:8.1f} us"
          f"  hash {1e3 * res[sc.MAP_HASH]:8.1f} us  ratio {res[sc.MAP_HASH] / res[sc.MAP_SORTED]:.2f}x  identical={same}"
          f" | whole build (sort + search + canonical lists): sorted {1e3 * whole[sc.MAP_SORTED]:8.1f} us"
          f" hash {1e3 * whole[sc.MAP_HASH]:8.1f} us | algorithmic {ab / 1e6:.1f} MB -> sorted build"
          f" {gbs(whole[sc.MAP_SORTED]):.0f} GB/s ({100 * gbs(whole[sc.MAP_SORTED]) / HBM:.1f} % of HBM),"
          f" search stage {gbs(res[sc.MAP_SORTED]):.0f} GB/s ({100 * gbs(res[sc.MAP_SORTED]) / HBM:.1f} %)",
          flush=True)
