"""CPU oracle: SPEC acceptance criteria (selftest binary), pinning of the restatement
against the reference's own headers (golden fixtures + oracle/_ref build), Python-level
SPEC examples. No GPU needed."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle_lib import ROOT, OracleError, load_oracle, load_ref_oracle

GOLDEN = os.path.join(ROOT, "tests", "golden", "geometry_golden.json")


@pytest.fixture(scope="module")
def oracle():
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "all"], check=True)
    return load_oracle()


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def test_selftest_acceptance_criteria():
    """SPEC.md:598-607 criteria 1, 2, 3, 5, 7, 8 + every known-answer example (C++)."""
    exe = os.path.join(ROOT, "oracle", "selftest")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "all"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAILED" not in r.stdout


def test_golden_pack_unpack(oracle, golden):
    g = golden["pack_key"]
    keys = oracle.pack_keys(np.array(g["coords"], np.int32))
    assert [str(int(k)) for k in keys] == g["keys"]
    np.testing.assert_array_equal(oracle.unpack_keys(keys), np.array(g["coords"]))
    assert int(keys[0]) == 0x4000020000100000
    for e in golden["pack_key_errors"]:
        with pytest.raises(OracleError) as ex:
            oracle.pack_keys(np.array([e["coord"]], np.int32))
        assert ex.value.status == e["status"] and str(ex.value) == e["error"]


def test_golden_weight_offsets(oracle, golden):
    for e in golden["weight_offsets"]:
        if "offsets" in e:
            np.testing.assert_array_equal(oracle.weight_offsets(e["K"], e["s"]), np.array(e["offsets"]))
        else:
            with pytest.raises(OracleError) as ex:
                oracle.weight_offsets(e["K"], e["s"])
            assert str(ex.value) == e["error"] and ex.value.status == e["status"]


def test_golden_output_coords(oracle, golden):
    for e in golden["generate_output_coords"]:
        q, srt, al = oracle.generate_output_coords(np.array(e["coords"], np.int32), False, e["s"])
        np.testing.assert_array_equal(q.reshape(-1, 3), np.array(e["out"]).reshape(-1, 3))
        assert srt == e["sorted"] and al == e["aliased"]


def test_golden_voxelize(oracle, golden):
    for e in golden["voxelize"]:
        f = np.zeros((len(e["points"]), 0), np.float32) if e["features"] is None else np.array(e["features"], np.float32)
        xyz, of = oracle.voxelize(np.array(e["points"]), f, e["resolution"])
        np.testing.assert_array_equal(xyz, np.array(e["coords"]).reshape(-1, 3))
        np.testing.assert_array_equal(of.astype(float), np.array(e["out_features"]).reshape(of.shape))


def test_golden_rng(oracle, golden):
    g = golden["rng"]
    for s, i, v in g["stream_seed"]:
        assert str(oracle.stream_seed(s, i)) == v
    for seed, vals in g["next"].items():
        assert [str(int(v)) for v in oracle.rng(int(seed), 8, 0)] == vals
    for seed, vals in g["next_unit"].items():
        assert oracle.rng(int(seed), 8, 1).tolist() == vals
    for key, vals in g["next_below"].items():
        seed, b = map(int, key.split(":"))
        assert [str(int(v)) for v in oracle.rng(seed, 8, 2, b)] == vals


def test_golden_kernel_map(oracle, golden):
    g = golden["kernel_map_two_points"]
    for backend in (0, 1, 2):
        q, sizes, j, i, _ = oracle.layer_map(np.array(g["coords"], np.int32), True, 3, 1, 1, backend=backend)
        assert sizes.tolist() == g["sizes"] and j.tolist() == g["in"] and i.tolist() == g["out"]
        assert sizes.sum() == 4


@pytest.mark.skipif(load_ref_oracle() is None, reason="reference headers not built here (oracle/_ref)")
def test_restatement_matches_reference_build():
    """Restated geometry/prng/oracle == the same oracle compiled on the reference headers."""
    ora, ref = load_oracle(), load_ref_oracle()
    rng = np.random.default_rng(1)
    M = 2 ** 20 - 1
    c = rng.integers(-M, M + 1, size=(5000, 3)).astype(np.int32)
    np.testing.assert_array_equal(ora.pack_keys(c), ref.pack_keys(c))
    for K in (1, 3, 5, 7):
        for s in (1, 2, 5):
            np.testing.assert_array_equal(ora.weight_offsets(K, s), ref.weight_offsets(K, s))
    for s in (1, 2, 3, 4):
        small = rng.integers(-300, 300, size=(2000, 3)).astype(np.int32)
        a, b = ora.generate_output_coords(small, False, s), ref.generate_output_coords(small, False, s)
        np.testing.assert_array_equal(a[0], b[0])
    pts = rng.random((3000, 3)) * 10 - 5
    f = rng.random((3000, 3)).astype(np.float32)
    for res in (0.05, 0.5, 1.7):
        a, b = ora.voxelize(pts, f, res), ref.voxelize(pts, f, res)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])
    for seed in (0, 3, 2 ** 40):
        np.testing.assert_array_equal(ora.rng(seed, 100, 0), ref.rng(seed, 100, 0))
        np.testing.assert_array_equal(ora.rng(seed, 100, 2, 12345), ref.rng(seed, 100, 2, 12345))
    xyz, F = ora.generate_synthetic(3000, 30, 4, 9)
    rx, rF = ref.generate_synthetic(3000, 30, 4, 9)
    np.testing.assert_array_equal(xyz, rx)
    np.testing.assert_array_equal(F, rF)
    W = ora.generate_weights(9, 1, 27, 4, 8)
    oq, of, _ = ora.layer_forward(xyz, False, F, W, 3, 1, 1)
    rq, rf, _ = ref.layer_forward(xyz, False, F, W, 3, 1, 1)
    np.testing.assert_array_equal(oq, rq)
    np.testing.assert_array_equal(of, rf)


def test_three_way_map_equivalence(oracle):
    """SPEC.md:255 at the ctypes level: sorted == hash == brute on random layers."""
    rng = np.random.default_rng(7)
    for trial in range(12):
        K = [1, 3, 5][trial % 3]
        s = 1 + trial % 2
        n = int(rng.integers(50, 600))
        xyz = rng.integers(0, 12, size=(n, 3)).astype(np.int32)
        xyz = np.unique(xyz, axis=0)[rng.permutation(len(np.unique(xyz, axis=0)))]
        outs = [oracle.layer_map(xyz, False, K, s, s, backend=b, B=int(rng.integers(4, 64)),
                                 Cq=int(rng.integers(4, 100))) for b in (0, 1, 2)]
        for o in outs[1:]:
            for a, b in zip(outs[0][:4], o[:4]):
                np.testing.assert_array_equal(a, b)


def test_layer_vs_dense_oracle(oracle):
    rng = np.random.default_rng(11)
    for K, s in [(3, 1), (3, 2), (5, 1), (2, 2)]:
        xyz = np.unique(rng.integers(-8, 8, size=(400, 3)).astype(np.int32), axis=0)
        F = rng.random((len(xyz), 8)).astype(np.float32)
        W = oracle.generate_weights(3, 1, K ** 3, 8, 16)
        _, out, st = oracle.layer_forward(xyz, True, F, W, K, s, s)
        ref = oracle.dense_conv(xyz, True, F, W, K, s, s)
        scale = np.abs(ref).max()
        assert np.abs(out - ref).max() <= 1e-5 * scale
        assert st["padding_overhead"] <= 0.25 + 1e-12


def test_grouping_examples(oracle):
    g = oracle.group_gemms([3, 3, 2], policy=0)
    assert len(g["groups"]) == 1 and g["buffer_length"] == 9 and abs(g["overhead"] - 0.125) < 1e-12
    assert len(oracle.group_gemms([1, 100], policy=1)["groups"]) == 2
    g = oracle.group_gemms([2, 3], policy=0)
    assert g["buffer_length"] == 6 and g["buffer_offsets"].tolist() == [0, 3]


def test_candidate_tiles_and_hyperparams(oracle):
    import ctypes as C
    out, n = (C.c_int * 64)(), C.c_int()
    assert oracle.lib.so_candidate_tiles(96, out, C.byref(n)) == 0
    assert list(out)[: n.value] == [1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 96]
    B, Cq = C.c_int(), C.c_int()
    assert oracle.lib.so_theoretical_hyperparams(2 ** 16, 2 ** 16, C.byref(B), C.byref(Cq)) == 0
    assert B.value == 16


@pytest.mark.parametrize("sorted_,s,expect", [(False, 1, 1), (True, 1, 0), (False, 2, 2), (True, 2, 1)])
def test_layer_map_sort_accounting(oracle, sorted_, s, expect):
    """a stride-1 layer sorts its one coordinate array once (none when flagged
    sorted); Eq. 1 adds one sort."""
    xyz, _ = oracle.generate_synthetic(3000, 30, 0, 4)
    if sorted_:
        xyz = xyz[np.lexsort((xyz[:, 2], xyz[:, 1], xyz[:, 0]))]
    assert int(oracle.layer_map(xyz, sorted_, 3, s, s)[4][4]) == expect
