"""Scene sharding across GPUs (BASELINE config 5: a batch of KITTI-shaped scans
scene-sharded over 1/2/4/8 B200s).

Scenes are independent units: each rank runs whole scenes (Map + GMaS for every layer) on its
own GPU with the weights replicated, so the data path has no collective. torch.distributed
(NCCL on GPUs, gloo on CPU) is used only for

  * the one-time weight broadcast from rank 0 (``broadcast_weights``), and
  * the result gather to rank 0 (``gather_results``), scene order preserved,

plus the barrier / max-over-ranks timing in bench.py. Host logic only: the compute stays in
the CUDA library (Network / layer calls made by ``run_shard``'s callback).
"""
from __future__ import annotations

from typing import Callable, Dict, List, Optional, Sequence, Tuple  # noqa: F401

import numpy as np

from .workloads import shard_range  # noqa: F401  (one definition for bench, tests and this module)


def _dist():
    import torch.distributed as dist
    return dist


def broadcast_weights(weights: Optional[Dict[int, np.ndarray]], shapes: Dict[int, Tuple[int, ...]], src: int = 0,
                      device=None) -> Dict[int, np.ndarray]:
    """Rank ``src`` sends every weight tensor (fp32 [K3][C_in][C_out]) to all ranks, ids in
    ascending order (one broadcast per tensor; NCCL over NVLink when ``device`` is a GPU).
    ``shapes`` (known to every rank from the graph) sizes the receive buffers."""
    import torch
    dist = _dist()
    rank = dist.get_rank()
    out = {}
    for wid in sorted(shapes):
        if rank == src:
            t = torch.from_numpy(np.ascontiguousarray(weights[wid], np.float32))
        else:
            t = torch.empty(shapes[wid], dtype=torch.float32)
        if device is not None:
            t = t.to(device)
        dist.broadcast(t, src)
        out[wid] = t.cpu().numpy()
    return out


def gather_results(local: Sequence, n_units: int, dst: int = 0, device=None) -> Optional[List]:
    """Gather every rank's per-scene outputs (ragged row counts allowed) to ``dst`` in global
    scene order; other ranks get None. Sizes travel first, then one flat buffer per rank.

    ``local``: numpy arrays or torch tensors (any float dtype, 2-D). ``device``: where the
    communication buffers live — a CUDA device for NCCL (which rejects host tensors), None for
    host tensors (gloo). Results on ``dst`` are numpy arrays when the inputs were numpy, torch
    tensors on ``device`` otherwise."""
    import torch
    dist = _dist()
    rank, world = dist.get_rank(), dist.get_world_size()
    start, end = shard_range(n_units, rank, world)
    if len(local) != end - start:
        raise ValueError("local result count does not match this rank's shard")
    as_numpy = all(isinstance(a, np.ndarray) for a in local)
    tens = [torch.from_numpy(np.ascontiguousarray(a, np.float32)) if isinstance(a, np.ndarray) else a for a in local]
    dev = torch.device("cpu") if device is None else torch.device(device)
    cols = {int(t.shape[1]) for t in tens if t.dim() == 2} or {0}
    if len(cols) > 1:
        raise ValueError("all results of a rank need the same channel count")
    dtype = tens[0].dtype if tens else torch.float32
    meta = torch.tensor([int(t.shape[0]) for t in tens] + [max(cols)], dtype=torch.int64, device=dev)
    if rank == dst:
        metas = []
        for r in range(world):
            a, b = shard_range(n_units, r, world)
            m = meta if r == dst else torch.zeros(b - a + 1, dtype=torch.int64, device=dev)
            if r != dst:
                dist.recv(m, src=r)
            metas.append(m)
    else:
        dist.send(meta, dst=dst)
    flat = (torch.cat([t.to(dev).reshape(-1) for t in tens]) if tens else torch.zeros(0, dtype=dtype, device=dev))
    if rank != dst:
        dist.send(flat.contiguous(), dst=dst)
        return None
    results: List = []
    for r in range(world):
        rows, c = metas[r][:-1].tolist(), int(metas[r][-1])
        if r == dst:
            buf = flat
        else:
            buf = torch.empty(sum(rows) * c, dtype=dtype, device=dev)
            dist.recv(buf, src=r)
        off = 0
        for n in rows:
            piece = buf[off:off + n * c].reshape(n, c)
            results.append(piece.cpu().numpy() if as_numpy else piece)
            off += n * c
    return results


class SceneResultGather:
    """Result gather of a scene-sharded step, overlapped with compute.

    Every rank writes scene s's result into ``slot(s)`` (preallocated, [rows_s, channels]);
    a rank other than ``dst`` sends it with ``dist.isend`` right after the producing work is
    enqueued (``produced(s)``) — on NCCL the send's stream waits for the producing stream at
    that point and runs beside the next scene's compute — while ``dst`` pre-posts one
    ``irecv`` per remote scene into its own slots at ``begin_step()``. ``end_step()`` waits
    for the step's transfers. Row counts of every scene are exchanged once at construction
    (``rows_local``: this rank's scenes), so no size message precedes the data."""

    def __init__(self, rows_local: Sequence[int], n_units: int, channels: int, dtype=None, device=None, dst: int = 0):
        import torch
        dist = _dist()
        self.dist, self.dst = dist, dst
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.lo, self.hi = shard_range(n_units, self.rank, self.world)
        if len(rows_local) != self.hi - self.lo:
            raise ValueError("row counts do not match this rank's shard")
        dev = torch.device("cpu") if device is None else torch.device(device)
        allr = [None] * self.world
        dist.all_gather_object(allr, [int(r) for r in rows_local])
        self.rows = [r for part in allr for r in part]
        self.owner = [r for r in range(self.world) for _ in allr[r]]
        dtype = dtype or torch.float16
        keep = range(n_units) if self.rank == dst else range(self.lo, self.hi)
        self.slots = {s: torch.zeros((self.rows[s], channels), dtype=dtype, device=dev) for s in keep}
        self.works = []

    def slot(self, s: int):
        return self.slots[s]

    def begin_step(self):
        if self.rank == self.dst:
            self.works = [self.dist.irecv(self.slots[s], src=self.owner[s]) for s in sorted(self.slots)
                          if self.owner[s] != self.dst]
        else:
            self.works = []

    def produced(self, s: int):
        if self.rank != self.dst:
            self.works.append(self.dist.isend(self.slots[s], dst=self.dst))

    def end_step(self):
        for w in self.works:
            w.wait()
        self.works = []

    def results(self):
        """On dst: every scene's result slot in global order (None elsewhere)."""
        return [self.slots[s] for s in range(len(self.rows))] if self.rank == self.dst else None


def run_shard(n_units: int, run_one: Callable[[int], np.ndarray], rank: int, world: int) -> List[np.ndarray]:
    """Runs this rank's contiguous scene range through ``run_one(scene_index)``."""
    start, end = shard_range(n_units, rank, world)
    return [run_one(s) for s in range(start, end)]
