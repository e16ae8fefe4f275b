"""Network graphs for BASELINE configs 2-5 (pure Python: no engine import, so the CPU
reference arm and the tests can build the same graphs without loading libsconv_b200.so).

The reference gives only the SC layer and a sequential netdef; the
backbones it cites (MinkUNet42, SparseResNet21D) are not specified there,
so the topologies below are this builder's definitions, with BN folded away
(inference) and ReLU fused into the conv epilogues:

  MinkUNet42      stem 2 x conv3 | 4 x [down K=2 s=2, 2 residual blocks] | 4 x [transposed
                  K=2 s=2, concat skip, 2 residual blocks]  -> 42 SC convs + 7 1x1 shortcuts
  SparseResNet21D stem conv3 | stage1 2 residual blocks | 4 x [conv3 s=2, 2 residual blocks]
                  with the last stage a single strided conv  -> 21 SC convs (x2 width "wide")
  UNetPair        K=2 s=2 down 32->64, transposed K=2 s=2 64->32 onto the input coordinates

Weights: U[-a, a] from Rng(stream_seed(seed, weight_id + 1)) (SPEC.md:528 draws U[-0.1, 0.1];
here a = sqrt(3 / (nbr * c_in)) with nbr the expected neighbours per voxel, so activations
neither explode nor vanish through 42 layers with random weights — the SPEC scale is the
special case nbr * c_in = 300).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List

import numpy as np

CONV, ADD, CONCAT = 1, 2, 3


@dataclass
class Op:
    kind: int
    out: int
    a: int
    b: int = -1  # second operand (ADD/CONCAT) or target tensor (transposed CONV)
    K: int = 3
    offset_scale: int = 1
    out_stride: int = 1
    transposed: int = 0
    c_in: int = 0
    c_out: int = 0
    weight: int = -1
    relu: int = 0

    def row(self):
        return [self.kind, self.out, self.a, self.b, self.K, self.offset_scale, self.out_stride, self.transposed,
                self.c_in, self.c_out, self.weight, self.relu]


@dataclass
class Graph:
    ops: List[Op] = field(default_factory=list)
    n_tensors: int = 0
    input: int = 0
    output: int = 0
    in_channels: int = 0
    channels: dict = field(default_factory=dict)
    stride: dict = field(default_factory=dict)  # tensor stride per tensor (for docs / checks)
    nbr: dict = field(default_factory=dict)     # expected neighbours used for the weight scale

    def tensor(self, c, ts):
        t = self.n_tensors
        self.n_tensors += 1
        self.channels[t], self.stride[t] = c, ts
        return t

    def conv(self, x, c_out, K=3, out_stride=None, relu=True, nbr=9.0):
        """out_stride = the output TENSOR stride; the op's Eq. 1 stride is 1 when it equals the
        input's (submanifold: Q = P) and the new tensor stride otherwise (floor to it)."""
        ts = self.stride[x]
        out_ts = ts if out_stride is None else out_stride
        y = self.tensor(c_out, out_ts)
        w = len([o for o in self.ops if o.kind == CONV])
        eq1 = 1 if out_ts == ts else out_ts
        self.ops.append(Op(CONV, y, x, -1, K, ts, eq1, 0, self.channels[x], c_out, w, int(relu)))
        self.nbr[w] = nbr
        return y

    def down(self, x, c_out, relu=True):  # K=2 s=2 (offsets {0, ts}^3, Q = floor(P / 2ts) * 2ts)
        return self.conv(x, c_out, K=2, out_stride=2 * self.stride[x], relu=relu, nbr=4.0)

    def up(self, x, target, c_out, relu=True):  # transposed K=2 s=2 onto `target`'s coordinates
        ts = self.stride[target]
        y = self.tensor(c_out, ts)
        w = len([o for o in self.ops if o.kind == CONV])
        self.ops.append(Op(CONV, y, x, target, 2, ts, ts, 1, self.channels[x], c_out, w, int(relu)))
        self.nbr[w] = 1.0
        return y

    def add(self, a, b, relu=True):
        y = self.tensor(self.channels[a], self.stride[a])
        self.ops.append(Op(ADD, y, a, b, relu=int(relu)))
        return y

    def concat(self, a, b):
        y = self.tensor(self.channels[a] + self.channels[b], self.stride[a])
        self.ops.append(Op(CONCAT, y, a, b))
        return y

    def residual(self, x, c_out):
        h = self.conv(x, c_out)
        h = self.conv(h, c_out, relu=False)
        sc = x if self.channels[x] == c_out else self.conv(x, c_out, K=1, relu=False, nbr=1.0)
        return self.add(h, sc)

    def convs(self):
        return [o for o in self.ops if o.kind == CONV]


def minkunet42(in_ch=4, cs=(32, 32, 64, 128, 256, 256, 128, 96, 96)) -> Graph:
    g = Graph(in_channels=in_ch)
    x = g.tensor(in_ch, 1)
    g.input = x
    x = g.conv(x, cs[0])
    x0 = g.conv(x, cs[0])
    enc, h = [x0], x0
    for i in range(4):
        h = g.down(h, cs[i])
        h = g.residual(h, cs[i + 1])
        h = g.residual(h, cs[i + 1])
        enc.append(h)
    for i in range(4):
        skip = enc[3 - i]
        h = g.up(h, skip, cs[5 + i])
        h = g.concat(h, skip)
        h = g.residual(h, cs[5 + i])
        h = g.residual(h, cs[5 + i])
    g.output = h
    return g


def sparse_resnet21d(in_ch=6, width=2) -> Graph:
    c = [16 * width, 32 * width, 64 * width, 128 * width]
    g = Graph(in_channels=in_ch)
    x = g.tensor(in_ch, 1)
    g.input = x
    h = g.conv(x, c[0])
    h = g.residual(h, c[0])
    h = g.residual(h, c[0])
    for i in range(1, 4):
        h = g.conv(h, c[i], K=3, out_stride=2 * g.stride[h], nbr=3.0)  # conv3 stride 2
        h = g.residual(h, c[i])
        h = g.residual(h, c[i])
    h = g.conv(h, c[3], K=3, out_stride=2 * g.stride[h], nbr=3.0)  # last stage: one strided conv
    g.output = h
    return g


def unet_pair(c_in=32, c_mid=64) -> Graph:
    g = Graph(in_channels=c_in)
    x = g.tensor(c_in, 1)
    g.input = x
    d = g.down(x, c_mid, relu=False)
    g.output = g.up(d, x, c_in, relu=False)
    return g


# SPEC netdef presets (oracle preset_network): (K, s, c_in, c_out) per layer
PRESETS = {
    "resnet_like": [(3, 1, 4, 16), (3, 1, 16, 16), (3, 2, 16, 32), (3, 1, 32, 32), (3, 2, 32, 64), (3, 1, 64, 64),
                    (3, 2, 64, 128), (3, 1, 128, 128)],
    "unet_like": [(3, 1, 4, 32), (3, 2, 32, 64), (3, 1, 64, 64), (3, 2, 64, 128), (3, 1, 128, 128), (3, 1, 128, 64),
                  (3, 1, 64, 32)],
}


def spec_chain(layers) -> Graph:
    """SPEC NetworkSpec: a sequential chain of SPEC-literal SC layers (K, s,
    c_in, c_out) — offsets weight_offsets(K, s), Eq. 1 stride s, no nonlinearity — where layer
    l+1's input coordinates are layer l's sorted output (sort reuse). Weight id l."""
    layers = [tuple(int(v) for v in L) for L in layers]
    if not layers:
        raise ValueError("empty network")
    for a, b in zip(layers, layers[1:]):
        if a[3] != b[2]:
            raise ValueError("network layers are not channel compatible")
    g = Graph(in_channels=layers[0][2])
    x = g.tensor(layers[0][2], 1)
    g.input = x
    for w, (K, s, ci, co) in enumerate(layers):
        y = g.tensor(co, 1)
        g.ops.append(Op(CONV, y, x, -1, K, s, s, 0, ci, co, w, 0))
        x = y
    g.output = x
    return g


def spec_weights(g: Graph, seed: int, generate: Callable) -> dict:
    """layer l's WeightSet from Rng(stream_seed(seed, l + 1)), U[-0.1, 0.1]."""
    return {o.weight: generate(seed, o.weight + 1, o.K ** 3, o.c_in, o.c_out) for o in g.convs()}


def weight_scale(g: Graph, o: Op) -> float:
    """Factor applied to the SPEC's U[-0.1, 0.1] draw: a / 0.1 with a = sqrt(3 / (nbr * c_in))."""
    return float(np.sqrt(3.0 / (g.nbr[o.weight] * o.c_in)) / 0.1)


def init_weights(g: Graph, seed: int, generate: Callable) -> dict:
    """Per conv weight id: U[-a, a] with a = sqrt(3 / (nbr * c_in)) (see module docstring).
    `generate(seed, stream, K3, c_in, c_out)` draws the SPEC's U[-0.1, 0.1] WeightSet
    (SPEC.md:528); the engine's sconv_generate_weights and the oracle's generator give the
    same bits (tests/test_capi.py)."""
    out = {}
    for o in g.convs():
        w = generate(seed, o.weight + 1, o.K ** 3, o.c_in, o.c_out)
        out[o.weight] = (w * np.float32(weight_scale(g, o))).astype(np.float32)
    return out
