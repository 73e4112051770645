"""Seeded/synthetic layer tables shaped like the paper's workloads (Table 4).

This module is an INPUT GENERATOR shared by the CUDA product's tests/bench and the
CPU oracle.  It contains none of the cost model's arithmetic (no Table 2 terms, no
halo volumes, no collective costs): it only turns an architecture description into
the per-row element counts, weights and FLOP counts that the paper takes as inputs
(P:167-181 tensors x, y, w, bi; P:519 FW_l, BW_l, WU_l).

Conventions (readings recorded in DESIGN.md):
  * One row per weighted layer for ResNets; BN/ReLU/add/pools folded; the projection
    shortcut 1x1 conv is folded into the block's last 1x1 row (flag FOLDED).  Keeps
    Table 4's G = 50 / 152.
  * VGG16 rows = 13x(Conv+ReLU), 5 Pool, FC, ReLU, Dropout, FC, ReLU, Dropout, FC = 38
    (P:678).  Pooling uses ceil mode (Chainer cover_all) so that 3x226^2 gives the
    "~169M" parameters of Table 4 (floor mode would give 138M).
  * CosmoFlow-like 3D net: 5x(Conv3d k3 p1 + ReLU + Pool) + FC,ReLU,FC,ReLU,FC = 20 rows,
    ~2M parameters, 4-channel N^3 input.  Our synthetic stand-in.
  * FLOPs (paper: FW/BW/WU are empirical; "FLOP counts" in theory):
    conv/FC fw = 2*C*F*prod(K)*prod(Y) per sample, bw = 2*fw; pool fw = y*prod(K);
    element-wise / norm fw = y; weightless bw = fw; wu = 2*(w+bi) per iteration.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from math import prod

# Row kinds (conv, FC-as-conv, channel-wise pool/norm, element-wise)
CONV, FC, POOL, ELEM, NORM = 0, 1, 2, 3, 4
KIND_NAMES = {CONV: "conv", FC: "fc", POOL: "pool", ELEM: "elem", NORM: "norm"}

# Row flags
FLAG_COMM = 1      # filter/channel communication point (Conv/FC rows, Table 3)
FLAG_FOLDED = 4    # w / fw include folded layers, so w != C*F*prod(K) is allowed

IMAGENET_D = 1_281_167   # "1.28M" samples (Table 4)
COSMOFLOW_D = 1584       # Table 4


@dataclass
class Layer:
    name: str
    kind: int
    ndim: int
    C: int
    F: int
    X: tuple
    Y: tuple
    K: tuple
    x: int
    y: int
    w: int
    bi: int
    fw: int
    bw: int
    wu: int
    flags: int = 0


@dataclass
class Model:
    name: str
    layers: list
    D: int                 # dataset size (samples)
    default_Ls: int        # default spatial prefix length (rows) -- P:608
    meta: dict = field(default_factory=dict)

    @property
    def G(self) -> int:
        return len(self.layers)


def _pad3(t):
    t = tuple(int(v) for v in t)
    return t + (1,) * (3 - len(t))


def _conv_out(n, k, s, p, ceil_mode=False):
    num = n + 2 * p - k
    if num < 0:
        raise ValueError("kernel larger than padded input")
    q = -(-num // s) if ceil_mode else num // s
    return q + 1


def make_conv(name, C, F, X, K, stride=1, pad=0, bias=True):
    nd = len(X)
    Ks = (K,) * nd if isinstance(K, int) else tuple(K)
    Y = tuple(_conv_out(X[i], Ks[i], stride, pad) for i in range(nd))
    w = C * F * prod(Ks)
    bi = F if bias else 0
    fw = 2 * C * F * prod(Ks) * prod(Y)
    return Layer(name, CONV, nd, C, F, _pad3(X), _pad3(Y), _pad3(Ks),
                 C * prod(X), F * prod(Y), w, bi, fw, 2 * fw, 2 * (w + bi), FLAG_COMM)


def make_fc(name, C, F, X, bias=True):
    # FC over x[N,C,WxH] == conv with K = input extent, output 1x1.
    nd = len(X)
    Ks = tuple(X)
    Y = (1,) * nd
    w = C * F * prod(Ks)
    bi = F if bias else 0
    fw = 2 * C * F * prod(Ks)
    return Layer(name, FC, nd, C, F, _pad3(X), _pad3(Y), _pad3(Ks),
                 C * prod(X), F, w, bi, fw, 2 * fw, 2 * (w + bi), FLAG_COMM)


def make_pool(name, C, X, K, stride, pad=0, ceil_mode=False):
    nd = len(X)
    Ks = (K,) * nd if isinstance(K, int) else tuple(K)
    Y = tuple(_conv_out(X[i], Ks[i], stride, pad, ceil_mode) for i in range(nd))
    y = C * prod(Y)
    fw = y * prod(Ks)
    return Layer(name, POOL, nd, C, C, _pad3(X), _pad3(Y), _pad3(Ks),
                 C * prod(X), y, 0, 0, fw, fw, 0, 0)


def make_elem(name, C, X, kind=ELEM):
    nd = len(X)
    n = C * prod(X)
    # element-wise F = C, weight w[C,F,0] -> K = 0
    return Layer(name, kind, nd, C, C, _pad3(X), _pad3(X), (0, 0, 0),
                 n, n, 0, 0, n, n, 0, 0)


# --------------------------------------------------------------------------- ResNet
def resnet(depth: int, res: int = 226) -> Model:
    blocks = {50: [3, 4, 6, 3], 101: [3, 4, 23, 3], 152: [3, 8, 36, 3]}[depth]
    rows = []
    conv1 = make_conv("conv1", 3, 64, (res, res), 7, stride=2, pad=3, bias=False)
    rows.append(conv1)
    s = conv1.Y[0]
    s = _conv_out(s, 3, 2, 1)          # max pool 3x3/2 (folded into conv1's row)
    cin = 64
    for si, nb in enumerate(blocks):
        mid = 64 * 2 ** si
        out = 4 * mid
        for bi_ in range(nb):
            stride = 2 if (si > 0 and bi_ == 0) else 1
            a = make_conv(f"s{si+1}b{bi_+1}a", cin, mid, (s, s), 1, bias=False)
            b = make_conv(f"s{si+1}b{bi_+1}b", mid, mid, (s, s), 3, stride=stride, pad=1, bias=False)
            s2 = b.Y[0]
            c = make_conv(f"s{si+1}b{bi_+1}c", mid, out, (s2, s2), 1, bias=False)
            if bi_ == 0:
                # projection shortcut 1x1/stride folded into the block's last 1x1 row (Q25)
                pw = cin * out
                pf = 2 * cin * out * s2 * s2
                c.w += pw
                c.fw += pf
                c.bw += 2 * pf
                c.wu += 2 * pw
                c.flags |= FLAG_FOLDED
            rows += [a, b, c]
            cin = out
            s = s2
    rows.append(make_fc("fc", cin, 1000, (1, 1)))   # global avg pool folded
    assert len(rows) == depth
    return Model(f"resnet{depth}", rows, IMAGENET_D, default_Ls=len(rows) - 1,
                 meta={"res": res})


# --------------------------------------------------------------------------- VGG16
def vgg16(res: int = 226) -> Model:
    cfg = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]
    rows = []
    c, s = 3, res
    ci = 0
    for v in cfg:
        if v == "M":
            p = make_pool(f"pool{len([r for r in rows if r.kind == POOL]) + 1}", c, (s, s), 2, 2,
                          ceil_mode=True)
            rows.append(p)
            s = p.Y[0]
        else:
            ci += 1
            cv = make_conv(f"conv{ci}", c, v, (s, s), 3, stride=1, pad=1)
            rows.append(cv)
            rows.append(make_elem(f"relu{ci}", v, (s, s)))
            c = v
    first_fc = len(rows)
    rows.append(make_fc("fc6", c, 4096, (s, s)))
    rows.append(make_elem("relu6", 4096, (1, 1)))
    rows.append(make_elem("drop6", 4096, (1, 1)))
    rows.append(make_fc("fc7", 4096, 4096, (1, 1)))
    rows.append(make_elem("relu7", 4096, (1, 1)))
    rows.append(make_elem("drop7", 4096, (1, 1)))
    rows.append(make_fc("fc8", 4096, 1000, (1, 1)))
    assert len(rows) == 38
    return Model("vgg16", rows, IMAGENET_D, default_Ls=first_fc, meta={"res": res})


# --------------------------------------------------------------------------- CosmoFlow-like
def cosmoflow(n: int = 256) -> Model:
    chans = [4, 16, 32, 64, 128, 256]
    rows = []
    s = n
    for i in range(5):
        cv = make_conv(f"conv{i+1}", chans[i], chans[i + 1], (s, s, s), 3, stride=1, pad=1)
        rows.append(cv)
        rows.append(make_elem(f"relu{i+1}", chans[i + 1], (s, s, s)))
        if i < 4:
            p = make_pool(f"pool{i+1}", chans[i + 1], (s, s, s), 2, 2)
        else:
            p = make_pool(f"pool{i+1}", chans[i + 1], (s, s, s), s, s)   # global pool
        rows.append(p)
        s = p.Y[0]
    rows.append(make_fc("fc1", 256, 2048, (1, 1, 1)))
    rows.append(make_elem("relu_fc1", 2048, (1, 1, 1)))
    rows.append(make_fc("fc2", 2048, 128, (1, 1, 1)))
    rows.append(make_elem("relu_fc2", 128, (1, 1, 1)))
    rows.append(make_fc("fc3", 128, 4, (1, 1, 1)))
    assert len(rows) == 20
    # "For CosmoFlow, we aggregate after the second convolution/pooling layer"
    return Model(f"cosmoflow{n}", rows, COSMOFLOW_D, default_Ls=6, meta={"res": n})


def by_name(name: str) -> Model:
    if name == "resnet50":
        return resnet(50)
    if name == "resnet152":
        return resnet(152)
    if name == "vgg16":
        return vgg16()
    if name.startswith("cosmoflow"):
        return cosmoflow(int(name[len("cosmoflow"):] or 256))
    raise KeyError(name)


def param_count(m: Model) -> int:
    """Plain input bookkeeping: total weights + biases (Table 4 "# Param")."""
    return sum(r.w + r.bi for r in m.layers)
