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

from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np


def shard_range(n_units: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [start, end) of ``n_units`` for ``rank``; the first n_units % world ranks
    take one extra unit (64 scenes over 8 GPUs -> 8 each)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    if n_units < 0:
        raise ValueError("unit count must be nonnegative")
    base, extra = divmod(n_units, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


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


def gather_results(local: Sequence[np.ndarray], n_units: int, dst: int = 0) -> Optional[List[np.ndarray]]:
    """Gather every rank's per-scene outputs (ragged row counts allowed) to ``dst`` in global
    scene order; other ranks get None. Sizes travel first, then one flat buffer per rank."""
    import torch
    dist = _dist()
    rank, world = dist.get_rank(), dist.get_world_size()
    start, end = shard_range(n_units, rank, world)
    if len(local) != end - start:
        raise ValueError("local result count does not match this rank's shard")
    cols = {a.shape[1] for a in local if a.ndim == 2} or {0}
    meta = torch.tensor([a.shape[0] for a in local] + [max(cols)], dtype=torch.int64)
    metas = [torch.zeros(shard_range(n_units, r, world)[1] - shard_range(n_units, r, world)[0] + 1, dtype=torch.int64)
             for r in range(world)] if rank == dst else None
    if rank == dst:
        for r in range(world):
            if r == dst:
                metas[r].copy_(meta)
            else:
                dist.recv(metas[r], src=r)
    else:
        dist.send(meta, dst=dst)
    flat = torch.from_numpy(np.concatenate([np.ascontiguousarray(a, np.float32).reshape(-1) for a in local])
                            if local else np.zeros(0, np.float32))
    if rank != dst:
        dist.send(flat, dst=dst)
        return None
    results: List[np.ndarray] = []
    for r in range(world):
        rows, c = metas[r][:-1].tolist(), int(metas[r][-1])
        if r == dst:
            buf = flat
        else:
            buf = torch.empty(sum(rows) * c, dtype=torch.float32)
            dist.recv(buf, src=r)
        off = 0
        for n in rows:
            results.append(buf[off:off + n * c].numpy().reshape(n, c))
            off += n * c
    return results


def run_shard(n_units: int, run_one: Callable[[int], np.ndarray], rank: int, world: int) -> List[np.ndarray]:
    """Runs this rank's contiguous scene range through ``run_one(scene_index)``."""
    start, end = shard_range(n_units, rank, world)
    return [run_one(s) for s in range(start, end)]
