"""C ABI boundary checks that need no GPU: the library loads, exports every entry point
declared in include/sconv_b200.h, and its host-side logic (synthetic inputs, weights,
GEMM grouping, reference-shaped Python mirror) matches the oracle exactly."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2401_06145_b200 as sc
from oracle_lib import ROOT, load_oracle

HEADER = os.path.join(ROOT, "include", "sconv_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sconv_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["sconv_ctx_create", "sconv_map_build", "sconv_map_read", "sconv_layer_forward",
                 "sconv_sc_layer_forward", "sconv_tune_layer", "sconv_weights_create", "sconv_plan_groups"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(sc.sconv.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers all of them
    bound = {name for name, _, _ in sc.sconv.SIGNATURES}
    assert set(declared_functions()) <= bound, set(declared_functions()) - bound


def test_version():
    assert b"sm_100a" in sc.load().sconv_version()


def test_synthetic_and_weights_match_oracle():
    ora = load_oracle()
    for N, E, Cc, seed in [(0, 5, 3, 1), (1000, 20, 4, 3), (5000, 400, 32, 1)]:
        a = sc.generate_synthetic(N, E, Cc, seed)
        b = ora.generate_synthetic(N, E, Cc, seed)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])
    np.testing.assert_array_equal(sc.generate_weights(1, 1, 27, 32, 32), ora.generate_weights(1, 1, 27, 32, 32))
    with pytest.raises(sc.InvalidArgument):
        sc.generate_synthetic(1001, 10, 1, 1)


def test_plan_groups_matches_oracle():
    ora = load_oracle()
    rng = np.random.default_rng(4)
    for trial in range(300):
        n = int(rng.integers(1, 30))
        sizes = rng.integers(0, 200, size=n)
        if trial % 5 == 0:
            sizes[rng.random(n) < 0.5] = 0
        for policy in (0, 1):
            for eps, mb in [(0.25, 16), (0.0, 1), (1.0, 4), (0.1, 27)]:
                a = sc.plan_groups(sizes, policy, eps, mb)
                b = ora.group_gemms(sizes, policy, eps, mb)
                np.testing.assert_array_equal(a["order"], b["order"])
                assert [tuple(map(int, g)) for g in a["groups"]] == [tuple(map(int, g)) for g in b["groups"]]
                np.testing.assert_array_equal(a["buffer_offsets"], b["buffer_offsets"])
                assert a["buffer_length"] == b["buffer_length"]
                assert a["overhead"] == pytest.approx(b["overhead"])
    with pytest.raises(sc.InvalidArgument):
        sc.plan_groups([1, 2], 1, -1.0, 16)


def test_python_mirror_weight_offsets():
    ora = load_oracle()
    for K, s in [(1, 1), (3, 1), (3, 2), (5, 2)]:
        np.testing.assert_array_equal(sc.weight_offsets(K, s), ora.weight_offsets(K, s))
    with pytest.raises(sc.InvalidArgument, match="kernel size must be a positive odd integer"):
        sc.weight_offsets(2, 1)


def test_no_cpu_fallback_when_library_missing(tmp_path):
    """The product path fails loudly instead of falling back to anything on the CPU."""
    with pytest.raises(ImportError):
        sc.sconv.load.__wrapped__ if hasattr(sc.sconv.load, "__wrapped__") else None
        import importlib
        mod = importlib.import_module("paper_2401_06145_b200.sconv")
        saved = mod._lib
        try:
            mod._lib = None
            mod.load(str(tmp_path / "missing.so"))
        finally:
            mod._lib = saved


def test_theoretical_hyperparams_matches_oracle():
    """SPEC.md:244-252 (Eq. 4) through the C ABI (no GPU needed): equal to the oracle, the
    SPEC's worked example |P| = |Q| = 2^16 -> B = 16, and its argument error."""
    o = load_oracle()
    assert sc.theoretical_hyperparams(1 << 16, 1 << 16)[0] == 16
    rng = np.random.default_rng(4)
    for p, q in [(1, 1), (2, 1), (1, 2), (100000, 100000), (123457, 40001)] + [
            tuple(int(v) for v in rng.integers(1, 10 ** 7, 2)) for _ in range(200)]:
        assert sc.theoretical_hyperparams(p, q) == o.theoretical_hyperparams(p, q), (p, q)
    with pytest.raises(sc.InvalidArgument, match="point counts must be positive"):
        sc.theoretical_hyperparams(0, 5)
