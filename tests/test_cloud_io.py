"""Point-cloud files (SURVEY §8f rank 3 "ingestion") through the C ABI. These
entry points are host-only, so they run on CPU: ".mpc" binary round trips, ".xyz" text round
trips (exact for double points and float features), and the parse errors the SPEC's cli
names ("malformed files -> parse error with line/offset")."""
import struct

import numpy as np
import pytest

import paper_2401_06145_b200 as sc


@pytest.mark.parametrize("n,c", [(0, 0), (1, 0), (5, 3), (1000, 4)])
def test_mpc_round_trip(tmp_path, n, c):
    rng = np.random.default_rng(n + c)
    xyz = rng.integers(-2 ** 20 + 1, 2 ** 20, size=(n, 3)).astype(np.int32)
    f = rng.standard_normal((n, c)).astype(np.float32)
    p = str(tmp_path / "a.mpc")
    sc.write_mpc(p, xyz, f)
    raw = open(p, "rb").read()
    assert raw[:4] == b"MPC1" and struct.unpack("<II", raw[4:12]) == (n, c)
    assert len(raw) == 12 + 12 * n + 4 * n * c
    assert sc.cloud_file_info(p) == (sc.FILE_MPC, n, c)
    cloud = sc.read_cloud(p)
    np.testing.assert_array_equal(cloud.coords, xyz)
    np.testing.assert_array_equal(cloud.features, f)
    assert cloud.sorted is False


def test_mpc_layout_is_little_endian_rows(tmp_path):
    p = tmp_path / "b.mpc"
    p.write_bytes(b"MPC1" + struct.pack("<II", 2, 1) + struct.pack("<6i", 1, -2, 3, 4, 5, -6) +
                  struct.pack("<2f", 0.5, -1.25))
    cloud = sc.read_cloud(str(p))
    np.testing.assert_array_equal(cloud.coords, [[1, -2, 3], [4, 5, -6]])
    np.testing.assert_array_equal(cloud.features, [[0.5], [-1.25]])


@pytest.mark.parametrize("payload,msg", [
    (b"MPC2" + bytes(8), "mpc parse error at offset 0: bad magic"),
    (b"MPC1" + struct.pack("<I", 3), "mpc parse error at offset 8: truncated header"),
    (b"MPC1" + struct.pack("<II", 2, 1) + bytes(20), "mpc parse error at offset 32: expected 44 bytes, file has 32"),
    (b"MPC1" + struct.pack("<II", 1, 0) + bytes(16), "mpc parse error at offset 24: expected 24 bytes, file has 28"),
])
def test_mpc_errors(tmp_path, payload, msg):
    p = tmp_path / "bad.mpc"
    p.write_bytes(payload)
    with pytest.raises(sc.InvalidArgument, match=msg):
        sc.read_cloud(str(p))


def test_xyz_round_trip_exact(tmp_path):
    rng = np.random.default_rng(3)
    pts = rng.uniform(-80, 80, size=(500, 3))
    f = rng.random((500, 4)).astype(np.float32)
    p = str(tmp_path / "a.xyz")
    sc.write_xyz(p, pts, f)
    assert sc.cloud_file_info(p) == (sc.FILE_XYZ, 500, 4)
    got_p, got_f = sc.read_cloud(p)
    np.testing.assert_array_equal(got_p, pts)
    np.testing.assert_array_equal(got_f, f)


def test_xyz_text_forms(tmp_path):
    p = tmp_path / "b.xyz"
    p.write_text("# header comment\n\n1 2 3 0.5\n  -1.5\t2e3   3 7  # trailing comment\r\n4 5 6 1")
    pts, f = sc.read_cloud(str(p))
    np.testing.assert_array_equal(pts, [[1, 2, 3], [-1.5, 2000, 3], [4, 5, 6]])
    np.testing.assert_array_equal(f, np.array([[0.5], [7], [1]], np.float32))
    q = tmp_path / "c.xyz"
    q.write_text("1 2 3\n4 5 6\n")
    pts, f = sc.read_cloud(str(q))
    assert pts.shape == (2, 3) and f.shape == (2, 0)
    e = tmp_path / "empty.xyz"
    e.write_text("\n# nothing\n")
    assert sc.cloud_file_info(str(e)) == (sc.FILE_XYZ, 0, 0)


@pytest.mark.parametrize("text,msg", [
    ("1 2 3 4\n1 2 3\n", "xyz parse error at line 2: expected 4 columns, got 3"),
    ("1 2\n", "xyz parse error at line 1: expected at least 3 columns, got 2"),
    ("\n1 2 3\n1 2 x3\n", "xyz parse error at line 3: invalid number 'x3'"),
    ("1 2 3,5\n", "xyz parse error at line 1: invalid number '3,5'"),
])
def test_xyz_errors(tmp_path, text, msg):
    p = tmp_path / "bad.xyz"
    p.write_text(text)
    with pytest.raises(sc.InvalidArgument, match=msg):
        sc.read_cloud(str(p))


def test_missing_file(tmp_path):
    with pytest.raises(sc.InvalidArgument, match="cannot open file"):
        sc.read_cloud(str(tmp_path / "nope.mpc"))
