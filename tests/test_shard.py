"""Scene sharding host logic on CPU: shard ranges, and a world_size-2 gloo run
of the weight broadcast + per-rank scene runs + ordered result gather (the N > 1 path of
bench.py / BASELINE config 5 without the GPU compute)."""
import os
import socket

import numpy as np
import pytest

from paper_2401_06145_b200 import network as N
from paper_2401_06145_b200.shard import SceneResultGather, broadcast_weights, gather_results, run_shard, shard_range


@pytest.mark.parametrize("n,world", [(64, 1), (64, 2), (64, 8), (7, 3), (3, 8), (0, 2)])
def test_shard_range_partitions(n, world):
    seen = []
    for r in range(world):
        a, b = shard_range(n, r, world)
        assert 0 <= a <= b <= n
        seen.extend(range(a, b))
    assert seen == list(range(n))  # contiguous, disjoint, ordered, complete
    sizes = [shard_range(n, r, world)[1] - shard_range(n, r, world)[0] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def test_shard_range_errors():
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)
    with pytest.raises(ValueError):
        shard_range(-1, 0, 1)


def fake_scene(s):
    """Stand-in for one scene's network output: ragged rows, deterministic per scene."""
    rng = np.random.default_rng(1000 + s)
    return rng.random((5 + 3 * s, 6), dtype=np.float32)


def _worker(rank, world, port, n_scenes, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = N.minkunet42()
        shapes = {o.weight: (o.K ** 3, o.c_in, o.c_out) for o in g.convs()}
        w = N.init_weights(g, 3) if rank == 0 else None
        got = broadcast_weights(w, shapes, src=0)
        ref = N.init_weights(g, 3)
        ok_w = all(np.array_equal(got[k], ref[k]) for k in ref)
        local = run_shard(n_scenes, fake_scene, rank, world)
        res = gather_results(local, n_scenes, dst=0)
        if rank == 0:
            ok_g = len(res) == n_scenes and all(np.array_equal(res[s], fake_scene(s)) for s in range(n_scenes))
        else:
            ok_g = res is None
        # the overlapped per-scene gather of bench.py's C5 step (same code path, host tensors on gloo)
        import torch
        lo, hi = shard_range(n_scenes, rank, world)
        rg = SceneResultGather([5 + 3 * s for s in range(lo, hi)], n_scenes, 6, dtype=torch.float32)
        ok_s = True
        for step in range(2):
            rg.begin_step()
            for s in range(lo, hi):
                rg.slot(s).copy_(torch.from_numpy(fake_scene(s)) + step)
                rg.produced(s)
            rg.end_step()
            if rank == 0:
                got = rg.results()
                ok_s &= len(got) == n_scenes and all(np.array_equal(got[s].numpy(), fake_scene(s) + step)
                                                     for s in range(n_scenes))
            else:
                ok_s &= rg.results() is None
        with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as f:
            f.write(f"{int(ok_w)} {int(ok_g and ok_s)}")
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n_scenes", [5, 2])
def test_gloo_world2_broadcast_shard_gather(tmp_path, n_scenes):
    import torch.multiprocessing as mp
    mp.start_processes(_worker, args=(2, free_port(), n_scenes, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    for r in range(2):
        assert (tmp_path / f"rank{r}.txt").read_text() == "1 1", r
