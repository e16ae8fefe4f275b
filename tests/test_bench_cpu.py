"""bench.py's CPU legs and multi-process plumbing, on CPU.

* The reference arm (`--impl reference`) runs the oracle on the GPU arm's own inputs and never
  loads the engine library (its process maps only oracle/ code).
* Under a 2-process launch (torchrun environment) only rank 0 of the reference arm runs and
  prints; the other rank exits 0 without output.
* workloads.py feeds the GPU arm, the reference arm and the parity tests the same scenes.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import json, os, sys
sys.argv = ["bench.py", "--impl", "reference", "--workload", "c4_unet_pair_shapenet", "--steps", "1", "--warmup", "0"]
sys.path.insert(0, os.getcwd())
import bench
bench.main()
maps = open("/proc/self/maps").read()
print(json.dumps({"engine_loaded": "libsconv_b200" in maps, "oracle_loaded": "liboracle" in maps,
                  "engine_modules": sorted(m for m in sys.modules if m.startswith("paper_2401_06145_b200"))}))
"""


def test_reference_arm_is_oracle_only():
    r = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    line, probe = lines[0], lines[1]
    assert line["impl"] == "reference" and line["config"]["workload"] == "c4_unet_pair_shapenet"
    assert line["config"]["voxels_per_step"] > 150_000  # the whole 8-object batch, not a crop
    assert line["value"] > 0 and line["cpu_baseline"]["cores"] >= 1
    assert probe == {"engine_loaded": False, "oracle_loaded": True, "engine_modules": []}


def test_reference_arm_rank1_exits_silently():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c4_unet_pair_shapenet",
                        "--steps", "1", "--warmup", "0", "--gpus", "2"], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "", (r.stdout, r.stderr)


def test_workloads_same_inputs_by_path_and_package():
    """The by-path copy (reference arm) and the package module (GPU arm) make identical inputs."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_net import load_pure
    from paper_2401_06145_b200 import workloads as WL
    P = load_pure("workloads")
    for name in ["c4_unet_pair_shapenet"]:
        a, b = WL.scenes(name)[0], P.scenes(name)[0]
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])
    assert [o.row() for o in WL.graph("c2_minkunet42_kitti").ops] == [o.row() for o in P.graph("c2_minkunet42_kitti").ops]
    assert WL.shard_range(64, 3, 8) == (24, 32)


@pytest.mark.parametrize("world", [1, 2, 8])
def test_c5_shards_cover_the_batch(world):
    from paper_2401_06145_b200 import workloads as WL
    ids = [i for r in range(world) for i in range(*WL.shard_range(WL.C5_SCENES, r, world))]
    assert ids == list(range(64))
