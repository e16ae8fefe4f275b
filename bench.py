#!/usr/bin/env python3
"""Benchmark driver (contract: one JSON line on rank 0).

metric (BASELINE.json): "SC layer latency (Map + GMaS, ms) and end-to-end network points/sec".
value = input voxels processed per second by the whole job (higher is better);
ms_per_step = latency of one step. Workloads (BASELINE.json configs):

  c2_minkunet42_kitti  (default, configs[1]) MinkUNet42 forward on a synthetic KITTI-shaped
                       scan (~120k voxels at 5 cm, 4 channels); step = Map for every distinct
                       geometry + GMaS for all 49 convs (42 SC + 7 1x1) + residual/concat ops
  c1_layer_100k        (configs[0]) one submanifold 3^3 layer, 32->32, 100k voxels in 400^3
  c3_resnet21d_s3dis   (configs[2]) SparseResNet21D (width x2) on an S3DIS-shaped room
  c4_unet_pair_shapenet (configs[3]) K=2 s=2 down + transposed pair on 8 ShapeNet-shaped
                       objects batched in the coordinates
  c5_minkunet42_batch64 (configs[4]) MinkUNet42 on 64 KITTI-shaped scans; a step runs this
                       rank's contiguous share (64/N scans) and gathers every result to rank 0

Inputs, graphs and weights come from paper_2401_06145_b200/workloads.py (shared with the
CPU reference arm and the full-size parity tests). Multi-GPU: one process per GPU; scenes
are independent units (no data-path collective; weak scaling). NCCL carries the one-time
weight broadcast from rank 0 (shard.broadcast_weights), the c5 result gather
(shard.SceneResultGather: per-scene isend/irecv overlapped with the next scene), the barrier
and the max-over-ranks timing. At N > 1 the c2 workload runs scan r of the batch on rank r.

Inputs are device resident before the timed region; L2 (126 MB) is flushed by a 256 MB
memset between timed steps, outside the events. Timing: CUDA events per step on the
launching stream, summed, max over ranks.

--impl reference: the CPU oracle (oracle/liboracle.so — the restatement of the reference
SPEC's Map/GMaS on its geometry) on all host threads, on the GPU arm's own step input (c5:
one whole scan per step); it imports nothing from the engine package.
"""
import argparse
import gc
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SC layer latency (Map + GMaS, ms) and end-to-end network points/sec"
DEFAULT_WORKLOAD = "c2_minkunet42_kitti"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default=DEFAULT_WORKLOAD,
                   choices=["c2_minkunet42_kitti", "c1_layer_100k", "c3_resnet21d_s3dis", "c4_unet_pair_shapenet",
                            "c5_minkunet42_batch64"])
    p.add_argument("--dtype", default="f16", choices=["f16", "bf16"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--B", type=int, default=256, help="source block size (SPEC default 256)")
    p.add_argument("--C", type=int, default=512, help="query block cap (SPEC default 512)")
    return p.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def load_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    def __init__(self, index):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.ok = False
        # NVML calls take driver locks and the GIL: polled too often they stall the forward's
        # host syncs (measured: sporadic 5-8 ms steps at a 5 ms interval)
        self.interval = float(os.environ.get("BENCH_CLOCK_INTERVAL", "0.05"))
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self.stop_ev.is_set():
            self._sample_once()
            self.stop_ev.wait(self.interval)

    def _sample_once(self):
        nv = self.nv
        names = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for k, bit in names.items():
                if r & bit:
                    self.reasons.add(k)
        except Exception:
            pass

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def sample_now(self):
        """One extra sample at a known point of the timed region (the steps are short: a 50 ms
        interval alone may land only once inside it)."""
        if self.ok:
            self._sample_once()

    def __exit__(self, *a):
        if self.ok:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- workloads
def oracle_crop(c, f, n):
    """The n voxels closest to the scene's median point (profiling tools only)."""
    ctr = np.median(c, axis=0)
    idx = np.sort(np.argsort(np.linalg.norm((c - ctr).astype(np.float64), axis=1), kind="stable")[:n])
    return c[idx], f[idx]


class NetWorkload:
    """A whole network forward per scene; a step runs every scene of this rank's share.

    c2/c3: one scene per step on every rank (weak scaling: rank r runs scene r of the KITTI
    batch for c2, the same room for c3); c4: the 8-object batch as one sparse tensor;
    c5: this rank's contiguous share of the 64 scans, each result copied into a device slot
    and gathered to rank 0 (NCCL isend/irecv overlapped with the next scene)."""

    def __init__(self, name, ctx, torch, dtype, B, C, world, rank, dist=None):
        import paper_2401_06145_b200 as sc
        from paper_2401_06145_b200 import network as N
        from paper_2401_06145_b200 import workloads as WL
        self.name, self.sc, self.torch = name, sc, torch
        self.g = WL.graph(name)
        if dist is not None:  # scene sharding: weights made on rank 0, one NCCL broadcast
            from paper_2401_06145_b200.shard import broadcast_weights
            shapes = {o.weight: (o.K ** 3, o.c_in, o.c_out) for o in self.g.convs()}
            w0 = N.init_weights(self.g, WL.WEIGHT_SEED) if dist.get_rank() == 0 else None
            self.w = broadcast_weights(w0, shapes, src=0, device=torch.device("cuda", torch.cuda.current_device()))
        else:
            self.w = N.init_weights(self.g, WL.WEIGHT_SEED)
        self.net = N.Network(ctx, self.g, self.w, sc.exec_cfg(compute_dtype=dtype), B, C)
        if name == "c2_minkunet42_kitti" and world > 1:
            self.scenes = [WL.kitti_scene(rank)]  # each rank its own scan (rank 0: the C2 scan)
        else:
            self.scenes = WL.scenes(name, world, rank)
        self.scene_ids = list(range(*WL.shard_range(WL.C5_SCENES, rank, world))) if name == "c5_minkunet42_batch64" \
            else list(range(len(self.scenes)))
        self.dev = [(torch.from_numpy(c).cuda(), torch.from_numpy(f).cuda()) for c, f in self.scenes]
        # e2e leg: inputs and the result live in pinned host memory (page-locked numpy views)
        pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
        self.pinned = [(pin(c), pin(f)) for c, f in self.scenes]
        self.out_pinned = {}
        self.points = WL.total_points(self.scenes)
        self.gather = None
        if name == "c5_minkunet42_batch64":
            from paper_2401_06145_b200.shard import SceneResultGather
            if dist is None:
                import types
                dist = types.SimpleNamespace(get_rank=lambda: 0, get_world_size=lambda: 1,
                                             all_gather_object=lambda out, obj: out.__setitem__(0, obj))
                import paper_2401_06145_b200.shard as SH
                SH._dist = lambda: dist  # noqa: E731  (single process: local slots only)
            self.gather = SceneResultGather([len(c) for c, _ in self.scenes], WL.C5_SCENES,
                                            self.g.channels[self.g.output], dtype=torch.float16,
                                            device=torch.device("cuda", torch.cuda.current_device()))
        model = WL.NETWORKS[name][0]
        self.config = {"model": model, "scenes_per_step": len(self.scenes), "voxels_per_step": self.points,
                       "batching": "batch-in-coordinates (x shifted by 256 per object)" if name.startswith("c4")
                       else ("scene-sharded: scenes %d..%d of 64 on this rank, results gathered to rank 0"
                             % (self.scene_ids[0], self.scene_ids[-1]) if self.gather else "none"),
                       "convs": len(self.g.convs()), "in_channels": self.g.in_channels}

    def step(self):
        if self.gather:
            self.gather.begin_step()
        for sid, (xyz, f) in zip(self.scene_ids, self.dev):
            self.net.forward(device_xyz=xyz.data_ptr(), device_feats=f.data_ptr(), n=xyz.shape[0], sorted_=True)
            if self.gather:
                self.net.copy_tensor(self.g.output, self.gather.slot(sid).data_ptr(), self.sc.F16)
                self.gather.produced(sid)
        if self.gather:
            self.gather.end_step()

    def e2e_step(self):
        torch = self.torch
        h2d = d2h = 0
        for i, (c, f) in enumerate(self.pinned):
            self.net.forward(c, f, True)
            n, ch, _ = self.net.info(self.g.output)
            if self.out_pinned.get(i) is None or self.out_pinned[i].shape != (n, ch):
                self.out_pinned[i] = torch.empty((n, ch), dtype=torch.float32, pin_memory=True).numpy()
            self.net.read(self.g.output, feats_out=self.out_pinned[i], coords=False)  # output coords = input coords
            h2d += c.nbytes + f.nbytes
            d2h += self.out_pinned[i].nbytes
        return h2d, d2h

    def e2e_run(self, k, fwd_ms=None):
        """k steps back to back through the public API as a serving loop runs them: every scene's
        inputs from pinned host memory (H2D inside sconv_net_forward, on the net's input stream), every scene's fp32 result
        read back with sconv_net_read_async -- its D2H copy runs on the net's copy stream beside
        the next scene's forward; result j is waited for (landed in host memory) once scene j+1
        is queued, before result j+1 is queued. Two pinned result buffers per scene alternate."""
        torch = self.torch
        h2d = d2h = 0
        first = True
        # prefetch the next request's inputs when their H2D (~50 GB/s pinned) is >= 5 % of a
        # forward (r02cq same box: C3 12 MB inputs 1.307 -> 1.290 ms, C4 27 MB 0.822 -> 0.799;
        # r02cj: C2 3.3 MB 2.24 -> 2.54, so not there); BENCH_E2E_PREFETCH=0/1 forces it
        env = os.environ.get("BENCH_E2E_PREFETCH")
        in_bytes = max(c.nbytes + f.nbytes for c, f in self.pinned)
        self.prefetch = env == "1" if env in ("0", "1") else \
            (fwd_ms is not None and in_bytes / 5e7 >= 0.05 * fwd_ms)
        reqs = [(s, i) for s in range(k) for i in range(len(self.pinned))]
        for r, (s, i) in enumerate(reqs):
            c, f = self.pinned[i]
            self.net.forward(c, f, True)
            # sconv_net_prefetch_inputs of the next request (BENCH_E2E_PREFETCH=1; r02cj same box:
            # C2 2.24 -> 2.54 ms, C4 0.83 -> 0.80: the next request's map builds then start at once
            # and slow this forward's convs)
            if self.prefetch and r + 1 < len(reqs):
                self.net.prefetch(*self.pinned[reqs[r + 1][1]])
            n, ch, _ = self.net.info(self.g.output)
            key = (i, s & 1)
            if self.out_pinned.get(key) is None or self.out_pinned[key].shape != (n, ch):
                self.out_pinned[key] = torch.empty((n, ch), dtype=torch.float32, pin_memory=True).numpy()
            if not first:
                self.net.wait_reads()
            first = False
            self.net.read_async(self.g.output, self.out_pinned[key])
            if s == 0:
                h2d += c.nbytes + f.nbytes
                d2h += self.out_pinned[key].nbytes
        self.net.wait_reads()
        return h2d, d2h

    def extra(self):
        return {"maps_built_per_scene": self.net.stats()["maps_built"]}

    def algo_bytes(self):
        """Per launch, averaged over the network's convs (the roofline divides by the average
        launch duration of the dominant kernel type)."""
        tot = self.net.algo_bytes()
        nconv = len(self.g.convs())
        per = {k: v / nconv for k, v in tot.items() if not k.startswith("_") and k not in ("k_search", "k_floor_unique")}
        per["k_search"] = tot["k_search"] / max(1, tot["_k_search_launches"])  # one launch per map
        # one cooperative launch per distinct Eq. 1 output set
        per["k_floor_unique"] = tot["k_floor_unique"] / max(1, tot["_k_floor_unique_launches"])
        return per

    def map_algo_bytes(self):
        """SURVEY §8d Map bytes of one step: the distinct maps of every scene of the step."""
        return self.net.algo_bytes()["k_search"] * len(self.scenes)

    def algo_flops(self):
        """Useful flops per launch of the conv kernels (2 C_in C_out |M|)."""
        st = self.net.conv_stats()
        tot = sum(2 * s["c_in"] * s["c_out"] * s["M"] for s in st)
        return tot / max(1, len(st))

    def cpu_sample(self, workers, budget_s=20.0):
        """The CPU oracle on this workload's first scene, whole (same input as the GPU step)."""
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle_net import oracle_graph, oracle_weights  # the checker / CPU baseline (test infrastructure)
        c, f = self.scenes[0]
        w = oracle_weights(self.g, 1)
        times = []
        while not times or (sum(times) < budget_s / 2 and len(times) < 3):
            t0 = time.perf_counter()
            oracle_graph(self.g, w, c, f, workers=workers)
            times.append(time.perf_counter() - t0)
        return len(c) / statistics.median(times), (
            f"oracle {self.config['model']} forward on the whole first scene of the step ({len(c)} voxels, "
            f"{len(times)} runs, median {statistics.median(times):.1f} s)")


class LayerWorkload:
    def __init__(self, name, ctx, torch, seed, dtype, B, C):
        import paper_2401_06145_b200 as sc
        self.name, self.sc, self.ctx, self.dtype, self.B, self.C = name, sc, ctx, dtype, B, C
        self.N, self.E, self.c = 100000, 400, 32
        self.xyz, self.F = sc.generate_synthetic(self.N, self.E, self.c, seed)
        self.W = sc.generate_weights(1, 1, 27, self.c, self.c)
        self.w = sc.Weights(ctx, self.W, dtype)
        self.xyz_d, self.F_d = torch.from_numpy(self.xyz).cuda(), torch.from_numpy(self.F).cuda()
        # e2e host buffers in pinned memory (inputs and results), as for the network workloads
        pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
        self.xyz_h, self.F_h = pin(self.xyz), pin(self.F)
        self.oxyz_h = torch.empty((self.N, 3), dtype=torch.int32).pin_memory().numpy()
        self.of_h = torch.empty((self.N, self.c), dtype=torch.float32).pin_memory().numpy()
        self.out_d = torch.empty((self.N, self.c), dtype=torch.float32, device="cuda")
        self.points = self.N
        m = self._map()
        self.tg, self.ts, _ = sc.tune_layer(ctx, m, self.w, self.F_d.data_ptr(), sc.F32, rounds=5)
        sc.layer_forward_device(ctx, m, self.w, self.F_d.data_ptr(), sc.F32, self.out_d.data_ptr(), sc.F32,
                                sc.exec_cfg(compute_dtype=dtype, gather_tile=self.tg, scatter_tile=self.ts))
        self.info = m.info()
        m.free()
        # dataflow choice (Alg. 2 style, setup only): time whole steps (Map + layer) with each
        # and keep the faster -- Minuet's GMaS with tuned tiles, or the fused kernel
        best = None
        for df in (sc.DATAFLOW_GMAS, sc.DATAFLOW_FUSED):
            self.cfg = sc.exec_cfg(compute_dtype=dtype, gather_tile=self.tg, scatter_tile=self.ts, dataflow=df)
            for _ in range(3):
                self.step()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
            for a, e in ev:
                a.record()
                self.step()
                e.record()
            torch.cuda.synchronize()
            ms = statistics.median(a.elapsed_time(e) for a, e in ev)
            if best is None or ms < best[0]:
                best = (ms, df)
        self.dataflow = best[1]
        self.cfg = sc.exec_cfg(compute_dtype=dtype, gather_tile=self.tg, scatter_tile=self.ts, dataflow=self.dataflow)
        self.config = {"model": "single SC layer K=3 s=1", "N": self.N, "E": self.E, "C_in": self.c,
                       "C_out": self.c, "gather_tile": self.tg, "scatter_tile": self.ts,
                       "matches": self.info.total_matches, "buffer_length": self.info.buffer_length,
                       "groups": self.info.groups, "padding_overhead": self.info.padding_overhead,
                       "dataflow": "fused" if self.dataflow == sc.DATAFLOW_FUSED else "gmas"}

    def _map(self):
        return self.sc.KernelMap.build(self.ctx, None, False, 3, 1, 1, device_ptr=self.xyz_d.data_ptr(), n=self.N,
                                       B=self.B, Cq=self.C)

    def step(self):
        m = self._map()
        self.sc.layer_forward_device(self.ctx, m, self.w, self.F_d.data_ptr(), self.sc.F32, self.out_d.data_ptr(),
                                     self.sc.F32, self.cfg)
        m.free()

    def e2e_step(self):
        out = self.sc.sc_layer_forward(self.ctx, self.sc.PointCloud(self.xyz_h, self.F_h, False), self.W, 3, 1,
                                       self.cfg, out_coords=self.oxyz_h, out_features=self.of_h)
        return self.xyz_h.nbytes + self.F_h.nbytes + self.W.nbytes, out.coords.nbytes + out.features.nbytes

    def extra(self):
        return {}

    def map_algo_bytes(self):  # 8|P| + 8|Q| + 8|M| + 4 K^3 (stride 1: Q = P)
        i = self.info
        return 8 * self.N + 8 * i.num_outputs + 8 * i.total_matches + 4 * 27

    def algo_bytes(self):  # per launch (SURVEY §8d with this path's dtypes)
        i, N, c, K3 = self.info, self.N, self.c, 27
        M, R, nq = i.total_matches, i.buffer_length, i.num_outputs
        return {"k_search": 8 * N + 8 * nq + 12 * K3, "k_emit": 8 * M + 4 * K3 * nq,
                "k_gather": 4 * c * N + 2 * c * R + 4 * M, "k_gemm_grouped": 2 * c * R + 4 * c * R + 2 * K3 * c * c,
                "k_scatter": 4 * c * M + 4 * K3 * nq + 4 * c * nq, "k_bucket_rank": 8 * N + 12 * N,
                "k_conv_fused": 2 * c * N + 4 * K3 * nq + 4 * c * nq,
                "k_bucket_scatter": 16 * N, "k_pack_compact": 20 * N, "k_bbox": 12 * N}

    def cpu_sample(self, workers, budget_s=20.0):
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle_lib import load_oracle  # CPU baseline only (test infrastructure)
        o = load_oracle()
        times = []
        while sum(times) < budget_s / 2 and len(times) < 5:
            t0 = time.perf_counter()
            o.layer_forward(self.xyz, False, self.F, self.W, 3, 1, 1, workers=workers)
            times.append(time.perf_counter() - t0)
        return self.N / statistics.median(times), f"{len(times)} full C1 layers on the oracle, median"


def make_workload(args, ctx, torch, world, rank, dist=None):
    dtype = 1 if args.dtype == "f16" else 2
    if args.workload == "c1_layer_100k":
        return LayerWorkload(args.workload, ctx, torch, 1 + rank, dtype, args.B, args.C)
    return NetWorkload(args.workload, ctx, torch, dtype, args.B, args.C, world, rank, dist)


# ---------------------------------------------------------------- reference arm (CPU oracle)
def reference_arm(args):
    """The reference's CPU path (the oracle restatement of SPEC Map + GMaS on the reference's
    geometry; the reference ships no runnable Map/GMaS code) on the SAME inputs as the GPU arm,
    all host threads. Imports nothing from the engine package: scenes, graphs and weights come
    from the pure-Python workload modules (loaded by path) and the oracle's own PRNG."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    workers = os.cpu_count() or 1
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import load_oracle
    from oracle_net import load_pure, oracle_graph, oracle_weights
    o = load_oracle()
    WL = load_pure("workloads")
    if args.workload == "c1_layer_100k":
        xyz, F = o.generate_synthetic(100000, 400, 32, 1)
        W = o.generate_weights(1, 1, 27, 32, 32)
        units = [lambda: o.layer_forward(xyz, False, F, W, 3, 1, 1, B=args.B, Cq=args.C, workers=workers)]
        pts = [100000]
        sample = "the full C1 layer (100k voxels, K=3, 32->32) per step"
    else:
        g = WL.graph(args.workload)
        w = oracle_weights(g, WL.WEIGHT_SEED)
        if args.workload == "c5_minkunet42_batch64":
            # 64 scans x ~6 s on the CPU do not fit a bench run: step i runs scan i of the batch
            # (whole, same input as the GPU arm's scene i)
            scenes = [WL.kitti_scene(i) for i in range(min(args.steps, WL.C5_SCENES))]
            sample = "one whole scan of the 64-scan batch per step (scan i at step i)"
        else:
            scenes = WL.scenes(args.workload)
            sample = "the whole workload per step (the GPU arm's step input)"
        units = [(lambda c=c, f=f: oracle_graph(g, w, c, f, workers=workers)) for c, f in scenes]
        pts = [len(c) for c, _ in scenes]
    per_step = len(units) == 1 or args.workload != "c5_minkunet42_batch64"

    def step(i):
        if per_step:
            for u in units:
                u()
            return sum(pts)
        units[i % len(units)]()
        return pts[i % len(units)]

    for i in range(args.warmup):
        step(i)
    times, done = [], 0
    for i in range(args.steps):
        t0 = time.perf_counter()
        done += step(i)
        times.append(time.perf_counter() - t0)
    pps = done / sum(times)
    print(json.dumps({
        "metric": METRIC, "value": pps, "unit": "points/s", "n_gpus": args.gpus, "steps": len(times),
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (fp64 accumulate)", "data": "synthetic",
        "config": {"workload": args.workload, "voxels_per_step": done // max(1, len(times)), "B": args.B,
                   "C": args.C, "same_input_as_gpu_arm": True}, "impl": "reference",
        "cpu_baseline": {"value": pps, "unit": "points/s", "cores": workers, "kind": "port", "sample": sample},
        "e2e": {"value": pps, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    import torch
    import paper_2401_06145_b200 as sc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")  # gloo: exercise N>1 on one GPU (tests)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    ctx = sc.Context(local)
    # One real (non-default) stream shared by torch and the library: events, the L2 flush and
    # every kernel are ordered on it (the legacy default stream, handle 0, is not ordered with
    # the context's own non-blocking stream).
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    wl = make_workload(args, ctx, torch, world, rank, dist)
    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()

    # per-kernel breakdown (untimed pass; every launch bracketed by events)
    ctx.set_profiling(True)
    ctx.profile_reset()
    n_bd = 3
    for _ in range(n_bd):
        ctx.flush_l2(256 << 20)
        wl.step()
    breakdown = ctx.profile()
    dominant = max(breakdown.items(), key=lambda kv: kv[1][1])[0] if breakdown else None
    ctx.profile_reset()
    ctx.set_profiling(False)  # timed region: no per-kernel events (an event between two convs
    # would serialise their programmatic dependent launch); the roofline pass below times them

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = ctx.launch_count
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    # a generational GC pass (~30 ms with torch loaded) inside a step stalls the host syncs of
    # the forward and shows up as one slow step: collect now, none inside the timed loops
    gc.collect()
    gc.disable()
    with ClockSampler(local) as clk:
        for a, b in ev:
            ctx.flush_l2(256 << 20)
            a.record(stream)
            wl.step()
            b.record(stream)
        clk.sample_now()  # the last steps are still queued / running on the GPU
        torch.cuda.synchronize()
    launches = ctx.launch_count - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    # roofline pass: the same K steps again with CUDA events around the dominant kernel only
    # (on the library's stream), giving its average launch duration
    ctx.set_profiling(True)
    ctx.set_profile_filter(dominant)
    ctx.profile_reset()
    for _ in range(args.steps):
        ctx.flush_l2(256 << 20)
        wl.step()
    torch.cuda.synchronize()
    prof = ctx.profile()
    ctx.set_profiling(False)
    ctx.set_profile_filter(None)
    total_ms = sum(step_ms)
    print("step ms: " + " ".join(f"{t:.3f}" for t in step_ms), file=sys.stderr)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_total_ms = float(t.item())
    pts = torch.tensor([float(wl.points)], dtype=torch.float64, device="cuda")  # ranks' scenes may differ in size
    if dist:
        dist.all_reduce(pts, op=dist.ReduceOp.SUM)
    job_points = float(pts.item())
    pps = job_points * args.steps / (max_total_ms / 1e3)

    # end-to-end through the public API with host buffers (H2D + D2H inside the timing)
    e2e_times, h2d, d2h = [], 0, 0
    for i in range(2 + min(args.steps, 10)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h2d, d2h = wl.e2e_step()
        torch.cuda.synchronize()
        if i >= 2:
            e2e_times.append(time.perf_counter() - t0)
    lat_t = torch.tensor([statistics.median(e2e_times)], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(lat_t, op=dist.ReduceOp.MAX)
    # serving throughput: K steps back to back, each step's result read back asynchronously so
    # that its D2H copy overlaps the next step's forward (network workloads; sconv_net_read_async)
    e2e_mode = "per-step latency (sequential: H2D, forward, D2H, sync)"
    e2e_t = lat_t
    if hasattr(wl, "e2e_run"):
        k_e2e = max(5, min(args.steps, 20))
        fwd_ms = max_total_ms / args.steps / max(1, len(getattr(wl, "pinned", [None])))  # per request
        wl.e2e_run(2, fwd_ms)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h2d, d2h = wl.e2e_run(k_e2e, fwd_ms)
        torch.cuda.synchronize()
        e2e_t = torch.tensor([(time.perf_counter() - t0) / k_e2e], dtype=torch.float64, device="cuda")
        if dist:
            dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        e2e_mode = ("pipelined: %d steps back to back, each step's inputs H2D from pinned memory%s and its fp32 "
                    "result D2H (sconv_net_read_async, overlapping the next step's forward), host clock around all"
                    % (k_e2e, " (prefetched beside the previous forward)" if getattr(wl, "prefetch", False) else ""))
    e2e_pps = job_points / float(e2e_t.item())
    gc.enable()

    # roofline of the dominant kernel: algorithmic bytes / measured duration
    hbm, tc, peak_kind = load_peaks()
    roofline = None
    if dominant and dominant in prof:
        n_launch, tot = prof[dominant]
        avg_ms = tot / n_launch
        algo = wl.algo_bytes().get(dominant)
        flops = wl.algo_flops() if dominant == "k_conv_fused" and hasattr(wl, "algo_flops") else 0.0
        ach = algo / (avg_ms / 1e3) / 1e9 if algo else None
        hbm_b = {"achieved": ach, "peak": hbm, "unit": "GB/s", "frac": (ach / hbm) if ach else None,
                 "t_min_ms": algo / hbm / 1e6 if algo else None}
        tfs = flops / (avg_ms / 1e3) / 1e12 if flops else None
        tc_b = {"achieved": tfs, "peak": tc, "unit": "TFLOP/s", "frac": tfs / tc if tfs else None,
                "t_min_ms": flops / tc / 1e9 if flops else None}
        # the binding bound: the one whose attainable time (algorithmic bytes / HBM peak vs useful
        # flops / tensor peak) is longer
        bind = "tensor" if flops and tc_b["t_min_ms"] > (hbm_b["t_min_ms"] or 0) else "hbm"
        b = tc_b if bind == "tensor" else hbm_b
        roofline = {"kernel": dominant, "bound": bind, "achieved": b["achieved"], "peak": b["peak"],
                    "unit": b["unit"], "frac": b["frac"], "traffic": load_traffic().get(dominant),
                    "peak_source": f"MEASURED_PEAKS.json {'bf16_tflops' if bind == 'tensor' else 'hbm_gbs'} "
                                   f"({peak_kind})",
                    "avg_launch_ms": avg_ms, "launches_per_step": n_launch / args.steps,
                    "algorithmic_bytes_per_launch": algo, "useful_flops_per_launch": flops or None,
                    "bounds": {"hbm": hbm_b, "tensor": tc_b if flops else None},
                    "timing": "CUDA events around each launch on the library stream, a second pass over "
                              "the K timed steps", "share_of_step": tot / total_ms}
    phases = {k: {"launches_per_step": n / n_bd, "us_per_step": 1e3 * ms / n_bd}
              for k, (n, ms) in sorted(breakdown.items(), key=lambda kv: -kv[1][1])}
    # the Map step: every kernel that builds the kernel maps of a step (key packing /
    # sorting, Eq. 1 output coordinates, search, canonical lists), event-timed in the breakdown
    # pass, against the algorithmic bytes of the step's distinct maps
    map_kernels = ("k_search", "k_floor", "k_pack", "k_init_flags", "k_bbox", "k_hist_scan", "k_bucket_scatter",
                   "k_bucket_rank", "k_scan_counts", "k_emit", "k_identity_map", "k_hash", "cub_")
    map_us = sum(v["us_per_step"] for k, v in phases.items() if k.startswith(map_kernels))
    map_b = wl.map_algo_bytes() if hasattr(wl, "map_algo_bytes") else None
    map_roof = None
    if map_us > 0 and map_b:
        gbs = map_b / (map_us * 1e-6) / 1e9
        map_roof = {"algorithmic_bytes_per_step": map_b, "kernel_us_per_step": map_us, "achieved": gbs,
                    "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                    "kernels": "event-timed sum of the map-building kernels (breakdown pass), serialised"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        workers = os.cpu_count() or 1
        v, sample = wl.cpu_sample(workers)
        cpu = {"value": v, "unit": "points/s", "cores": workers, "kind": "port", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": pps, "unit": "points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": args.workload, **wl.config, "B": args.B, "C": args.C,
                       "parallelism": f"scene-sharded x{world}", "l2": "flushed (256 MB memset) between timed steps",
                       **wl.extra()},
            "e2e": {"value": e2e_pps, "unit": "points/s", "ms": 1e3 * float(e2e_t.item()), "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "mode": e2e_mode,
                    "latency_ms": 1e3 * float(lat_t.item()),
                    "api": "host buffers through the C ABI (sconv_net_forward + sconv_net_read_async / "
                           "sconv_sc_layer_forward + readback)"},
            "gpu_launches": launches,
            "roofline": roofline,
            "phases": phases,
            "map_roofline": map_roof,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
