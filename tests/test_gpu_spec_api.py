"""The SPEC-signature boundary on the GPU, against the oracle.

* build_kernel_map_sorted(P, Q, offsets, B, C) -> (KernelMap, SearchCounters) for an arbitrary
  sorted query list and offset list: every backend's canonical map equals the
  oracle's exactly; the SORTED_SPEC backend (the SPEC's own work decomposition, incl.
  balance_blocks' ceil(L/C) ranges) reproduces the oracle's SearchCounters exactly.
* Acceptance #3 asserted on the GPU's counters: <= 10 mean comparisons per query
  at |P| = |Q| = 1e5, K = 3, B = 256, C = 512, and the SPEC's two comparison bounds.
* Acceptance #7: sort counts of map chains and of forward_network.
* forward_network(spec, cloud, cfg, seed) vs the oracle's.
"""
import numpy as np
import pytest

import paper_2401_06145_b200 as sc
from paper_2401_06145_b200 import network as N
from parity import elementwise_errors

pytestmark = pytest.mark.gpu

BACKENDS = [sc.MAP_SORTED, sc.MAP_HASH, sc.MAP_SORTED_SPEC]


def cloud(rng, n, extent, lo=0):
    xyz = np.unique(rng.integers(lo, lo + extent, (n, 3)).astype(np.int32), axis=0)
    return xyz[rng.permutation(len(xyz))]


def sorted_unique(xyz):
    xyz = np.unique(xyz, axis=0)  # lexicographic (x, y, z) = packed-key order
    return xyz.astype(np.int32)


def offsets_of(kind, rng):
    if kind == "k3":
        return np.array([(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)], np.int32)
    if kind == "k5s2":
        r = range(-4, 5, 2)
        return np.array([(a, b, c) for a in r for b in r for c in r], np.int32)
    if kind == "k2":
        return np.array([(a, b, c) for a in (0, 1) for b in (0, 1) for c in (0, 1)], np.int32)
    # a random sorted offset set (SPEC: offsets sorted once per layer)
    return sorted_unique(rng.integers(-3, 4, (12, 3)))


def read_lists(m):
    q, sizes, j, i = m.read()
    return q, sizes, j, i


@pytest.mark.parametrize("n,extent,p_sorted,okind,B,Cq", [
    (3000, 20, False, "k3", 256, 512),
    (5000, 30, True, "k5s2", 64, 100),
    (2000, 12, False, "rand", 16, 7),
    (4000, 40, False, "k2", 256, 1),
    (1, 5, False, "k3", 4, 512),
])
def test_explicit_map_all_backends_vs_oracle(ctx, oracle, n, extent, p_sorted, okind, B, Cq):
    rng = np.random.default_rng(n + extent)
    P = cloud(rng, n, extent)
    if p_sorted:
        P = sorted_unique(P)
    # queries: half drawn from P, half fresh points (some outside P's extent)
    Q = sorted_unique(np.concatenate([P[: max(1, len(P) // 2)], cloud(rng, max(1, n // 2), extent + 6, -3)]))
    offs = offsets_of(okind, rng)
    oq, osz, oj, oi, ocnt = oracle.map_build(P, p_sorted, Q, offs, 0, B, Cq)
    for be in BACKENDS:
        m = sc.KernelMap.build_explicit(ctx, P, p_sorted, Q, offs, B, Cq, be)
        q, sizes, j, i = read_lists(m)
        np.testing.assert_array_equal(q, oq)
        np.testing.assert_array_equal(sizes, osz)
        np.testing.assert_array_equal(j, oj)
        np.testing.assert_array_equal(i, oi)
        c = m.search_counters()
        assert c["sorts"] == (0 if p_sorted else 1), (be, c)
        if be == sc.MAP_SORTED_SPEC:
            assert c["counted"] == 1
            got = [c["backward_comparisons"], c["forward_comparisons"], c["source_elements_loaded"],
                   c["queries_executed"], c["sorts"]]
            assert got == [int(v) for v in ocnt], (got, ocnt.tolist())
        m.free()


def test_explicit_map_errors(ctx):
    P = np.array([[0, 0, 0], [1, 0, 0]], np.int32)
    with pytest.raises(sc.InvalidArgument, match="query coordinates must be sorted and unique"):
        sc.KernelMap.build_explicit(ctx, P, False, np.array([[1, 0, 0], [0, 0, 0]], np.int32), [[0, 0, 0]])
    with pytest.raises(sc.OutOfRange, match="coordinate x out of range: 1048576"):
        sc.KernelMap.build_explicit(ctx, P, False, np.array([[1 << 20, 0, 0]], np.int32), [[0, 0, 0]])
    with pytest.raises(sc.InvalidArgument):
        sc.KernelMap.build_explicit(ctx, P, False, P, np.zeros((0, 3), np.int32))


@pytest.mark.parametrize("Cq", [1, 7, 64, 512, 4096])
def test_balance_blocks_C_vs_oracle(ctx, oracle, Cq):
    """C splits every query block longer than C into ceil(L/C) near-equal ranges
    (SPEC.md:217-225): the map is unchanged, source_elements_loaded grows with the range count,
    and every counter equals the oracle's."""
    rng = np.random.default_rng(11)
    P = sorted_unique(cloud(rng, 20000, 40))
    offs = offsets_of("k3", rng)
    oq, osz, oj, oi, ocnt = oracle.map_build(P, True, P, offs, 0, 256, Cq)
    m = sc.KernelMap.build_explicit(ctx, P, True, P, offs, 256, Cq, sc.MAP_SORTED_SPEC)
    _, sizes, j, i = read_lists(m)
    np.testing.assert_array_equal(sizes, osz)
    np.testing.assert_array_equal(j, oj)
    np.testing.assert_array_equal(i, oi)
    c = m.search_counters()
    assert [c["backward_comparisons"], c["forward_comparisons"], c["source_elements_loaded"],
            c["queries_executed"]] == [int(v) for v in ocnt[:4]]


def test_acceptance3_on_gpu_counters(ctx, oracle):
    """SPEC acceptance #3: |P| = |Q| = 1e5 (uniform in 400^3, generate_synthetic seed 1), K = 3,
    B = 256, C = 512: mean comparisons per query (backward amortised + forward) <= 10, the naive
    per-query search needs 17; counters exact (equal to the oracle's)."""
    xyz, _ = sc.generate_synthetic(100000, 400, 0, 1)
    m = sc.KernelMap.build(ctx, xyz, False, 3, 1, 1, B=256, Cq=512, backend=sc.MAP_SORTED_SPEC)
    c = m.search_counters()
    _, _, _, _, ocnt = oracle.layer_map(xyz, False, 3, 1, 1, backend=0, B=256, Cq=512)
    got = [c["backward_comparisons"], c["forward_comparisons"], c["source_elements_loaded"], c["queries_executed"],
           c["sorts"]]
    assert got == [int(v) for v in ocnt], (got, ocnt.tolist())
    per_query = (c["backward_comparisons"] + c["forward_comparisons"]) / c["queries_executed"]
    print(f"acceptance3 (GPU counters): {per_query:.3f} comparisons per query, {c}")
    assert per_query <= 10.0
    nb = -(-100000 // 256)
    assert c["backward_comparisons"] <= 27 * nb * 17  # K^3 ceil(|P|/B) ceil(log2(|Q|+1))
    assert c["forward_comparisons"] <= c["queries_executed"] * 9  # ceil(log2(B+1))
    assert c["sorts"] == 1
    # the default (redesigned) backend gives the identical map
    m2 = sc.KernelMap.build(ctx, xyz, False, 3, 1, 1, B=256, Cq=512)
    a, b = m.read(), m2.read()
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_acceptance7_map_chain_sorts(ctx):
    """Sort reuse: an unsorted input sorts once; chained stride-1 maps reuse
    the sorted keys (0 sorts); a strided map performs its Eq. 1 sort."""
    xyz, _ = sc.generate_synthetic(20000, 40, 0, 3)
    first = sc.KernelMap.build(ctx, xyz, False, 3, 1, 1)
    chain = [first]
    for _ in range(4):
        chain.append(sc.KernelMap.chained(ctx, chain[-1], 3, 1, 1))
    assert [m.search_counters()["sorts"] for m in chain] == [1, 0, 0, 0, 0]
    strided = [first]
    for s in [2, 1, 2, 1]:
        strided.append(sc.KernelMap.chained(ctx, strided[-1], 3, s, s))
    assert sum(m.search_counters()["sorts"] for m in strided) == 3


@pytest.mark.parametrize("layers", [
    [(3, 1, 4, 16), (3, 1, 16, 16), (3, 1, 16, 16), (3, 1, 16, 16), (3, 1, 16, 16)],
    [(3, 1, 4, 16), (3, 2, 16, 32), (3, 1, 32, 32), (3, 2, 32, 64), (3, 1, 64, 64)],
    N.PRESETS["unet_like"],
])
def test_forward_network_vs_oracle(ctx, oracle, layers):
    """SPEC forward_network: weights Rng(stream_seed(seed, l+1)) U[-0.1, 0.1], sorted output,
    sort counts (acceptance #7: 1 for the stride-1 chain, 3 for strides [1,2,1,2,1])."""
    xyz, F = sc.generate_synthetic(20000, 40, 4, 9)
    out, sorts = N.forward_network(ctx, layers, sc.PointCloud(xyz, F, False), seed=9)
    oq, of, osorts = oracle.forward_network(layers, xyz, False, F, 9, workers=8)
    np.testing.assert_array_equal(out.coords, oq)
    assert sorts == osorts == 1 + sum(1 for L in layers if L[1] > 1)
    mx, mean, fro = elementwise_errors(out.features, of)
    print(f"forward_network {len(layers)} layers: fro {fro:.2e} max rel_e {mx:.2e} mean {mean:.2e}")
    assert fro <= 2e-3, (mx, mean, fro)  # f16 operands over 5-7 chained layers


def test_theoretical_hyperparams_gpu_build(ctx):
    """The advisory (B, C) of Eq. 4 are valid build parameters (B rounded to the multiple of 4
    the staged copies need) and give the same map."""
    xyz, _ = sc.generate_synthetic(30000, 60, 0, 5)
    B, Cq = sc.theoretical_hyperparams(30000, 30000)
    B4 = max(4, (B + 3) // 4 * 4)
    a = sc.KernelMap.build(ctx, xyz, False, 3, 1, 1, B=B4, Cq=Cq, backend=sc.MAP_SORTED_SPEC).read()
    b = sc.KernelMap.build(ctx, xyz, False, 3, 1, 1).read()
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
