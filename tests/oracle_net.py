"""TEST INFRASTRUCTURE — the CPU oracle run over a network graph, and the pure-Python
workload modules loaded WITHOUT the engine package.

Used by the GPU parity tests (the checker) and by bench.py's CPU legs (cpu_baseline and
`--impl reference`). Nothing here imports `paper_2401_06145_b200` as a package: the scene
generators (datasets.py) and graph definitions (graphs.py) are pure numpy/Python files that
are loaded by path, so a process that uses only this module never loads libsconv_b200.so.
"""
import importlib.util
import os
import sys

import numpy as np

from oracle_lib import load_oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2401_06145_b200")


def load_pure(name):
    """paper_2401_06145_b200/<name>.py as a stand-alone module (no package __init__)."""
    key = f"_sconv_pure_{name}"
    if key in sys.modules:
        return sys.modules[key]
    spec = importlib.util.spec_from_file_location(key, os.path.join(PKG, f"{name}.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[key] = mod
    spec.loader.exec_module(mod)
    return mod


def oracle_weights(g, seed):
    """graphs.init_weights with the oracle's SPEC PRNG (bit-identical to the engine's)."""
    ora = load_oracle()
    return load_pure("graphs").init_weights(g, seed, ora.generate_weights)


def oracle_graph(g, weights, coords, feats, workers=None, tensors=False):
    """Whole graph on the CPU oracle (fp32 features, fp64 accumulation): SPEC sc_layer_forward
    per CONV, ADD / CONCAT in fp32. Returns the output tensor's
    (coords, feats), or every tensor when tensors=True."""
    ora = load_oracle()
    workers = workers or os.cpu_count() or 1
    CONV, ADD = 1, 2
    T = {g.input: (coords, feats)}
    for o in g.ops:
        xin, fin = T[o.a]
        if o.kind == CONV:
            tgt = T[o.b][0] if o.transposed else None
            q, f, _ = ora.layer_forward(xin, True, fin, weights[o.weight], o.K, o.offset_scale, o.out_stride,
                                        bool(o.transposed), tgt, workers=workers)
            T[o.out] = (q, np.maximum(f, 0) if o.relu else f)
        elif o.kind == ADD:
            s = fin + T[o.b][1]
            T[o.out] = (xin, np.maximum(s, 0) if o.relu else s)
        else:
            T[o.out] = (xin, np.concatenate([fin, T[o.b][1]], 1))
    return T if tensors else T[g.output]
