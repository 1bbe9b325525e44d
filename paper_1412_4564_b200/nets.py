"""The BASELINE.json networks as layer lists for the DAG engine.

Each network is built from the reference's blocks exactly as SURVEY.md
§8d / Appendix A specifies (LeNet, CIFAR-10 quick + LRN, imagenet-caffe-alex,
VGG-VD-16 + bnorm), with the reference's synthetic-input recipe:
data U[-1,1) seed 1, weights 0.01 N(0,1) seed 2 in network order, zero
biases, bnorm w=1 b=0, labels 1 + below(C) seed 3.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import lib


@dataclass
class Net:
    name: str
    batch: int
    classes: int
    inputs: dict = field(default_factory=dict)       # name -> HWCN shape
    params: list = field(default_factory=list)       # (name, shape, init)
    layers: list = field(default_factory=list)       # (kind, name, inputs, outputs, params)

    def conv(self, name, x, out, fh, fw, cin, cout, stride=1, pad=(0, 0, 0, 0), groups=1,
             bias=True):
        f = f"{name}f"
        self.params.append((f, (fh, fw, cin // groups, cout), "normal"))
        ins = [x, f]
        if bias:
            b = f"{name}b"
            self.params.append((b, (1, 1, cout, 1), "zeros"))
            ins.append(b)
        self.layers.append(("conv", name, ins, [out],
                            [stride, stride, pad[0], pad[1], pad[2], pad[3], groups]))
        return out

    def relu(self, name, x, out):
        self.layers.append(("relu", name, [x], [out], []))
        return out

    def lrn(self, name, x, out, n, kappa, alpha, beta):
        self.layers.append(("lrn", name, [x], [out], [n, kappa, alpha, beta]))
        return out

    def pool(self, name, x, out, win, stride, pad=(0, 0, 0, 0), mode="max"):
        self.layers.append(("pool", name, [x], [out],
                            [win, win, stride, stride, pad[0], pad[1], pad[2], pad[3],
                             0 if mode == "max" else 1]))
        return out

    def bnorm(self, name, x, out, channels, eps=1e-5):
        w, b = f"{name}w", f"{name}b"
        self.params.append((w, (1, 1, channels, 1), "ones"))
        self.params.append((b, (1, 1, channels, 1), "zeros"))
        self.layers.append(("bnorm", name, [x, w, b], [out], [eps]))
        return out

    def loss(self, x, label="label", out="objective"):
        self.layers.append(("loss", "loss", [x, label], [out], []))
        return out

    # -- synthetic inputs ---------------------------------------------------
    def init_params(self, seed=2, rng=None):
        """rng: the generator class (default: libck's host xoshiro256**; the
        oracle's restatement oracle.Rng yields the identical stream)."""
        r = (rng or Rng)(seed)
        out = {}
        for name, shape, init in self.params:
            n = int(np.prod(shape))
            if init == "normal":
                out[name] = r.normal(n, 0.01)
            elif init == "ones":
                out[name] = np.ones(n, np.float32)
            else:
                out[name] = np.zeros(n, np.float32)
        return out

    def init_inputs(self, data_seed=1, label_seed=3, rng=None):
        ds = self.inputs["data"]
        ls = self.inputs["label"]
        R = rng or Rng
        return {"data": R(data_seed).uniform(int(np.prod(ds))),
                "label": R(label_seed).labels(int(np.prod(ls)), self.classes)}

    def build(self, target):
        """Emit into any object with the graph.hpp construction API."""
        for name, shape in self.inputs.items():
            target.add_input(name, shape)
        for name, shape, _ in self.params:
            target.add_param(name, shape)
        for kind, name, ins, outs, p in self.layers:
            target.add_layer(kind, name, ins, outs, p)
        return target

    def conv_layers(self):
        """(name, x shape, f shape, geom) for every conv layer, shapes inferred."""
        shapes = dict(self.inputs)
        for name, shape, _ in self.params:
            shapes[name] = shape
        out = []
        for kind, name, ins, outs, p in self.layers:
            xs = shapes[ins[0]]
            if kind == "conv":
                fs = shapes[ins[1]]
                s, pt, pb, pl, pr = p[0], p[2], p[3], p[4], p[5]
                ys = ((xs[0] + pt + pb - fs[0]) // s + 1, (xs[1] + pl + pr - fs[1]) // s + 1,
                      fs[3], xs[3])
                out.append((name, xs, fs, p))
            elif kind == "pool":
                w, s, pt, pb, pl, pr = p[0], p[2], p[4], p[5], p[6], p[7]
                ys = ((xs[0] + pt + pb - w) // s + 1, (xs[1] + pl + pr - w) // s + 1, xs[2], xs[3])
            elif kind == "loss":
                ys = (1, 1, 1, 1)
            elif kind == "bilinear":
                gs = shapes[ins[1]]
                ys = (gs[1], gs[2], xs[2], xs[3])
            elif kind == "pdist":
                ys = (xs[0], xs[1], 1, xs[3])
            else:
                ys = xs
            for o in outs:  # (split: every output)
                shapes[o] = ys
        return out

    def conv_flops(self):
        """Algorithmic conv FLOP per fwd+bwd step, dgrad of the
        first layer included because the reference computes it."""
        total = 0
        shapes = {}
        for name, xs, fs, p in self.conv_layers():
            s, pt, pb, pl, pr = p[0], p[2], p[3], p[4], p[5]
            oh = (xs[0] + pt + pb - fs[0]) // s + 1
            ow = (xs[1] + pl + pr - fs[1]) // s + 1
            macs = xs[3] * oh * ow * fs[3] * fs[0] * fs[1] * fs[2]
            total += 3 * 2 * macs
        return total


class Rng:
    """The reference generator (rng.cpp) via libck's host helper."""

    def __init__(self, seed):
        self.h = C.c_void_p(lib().ck_rng_create(seed))

    def __del__(self):
        if getattr(self, "h", None):
            lib().ck_rng_destroy(self.h)
            self.h = None

    def uniform(self, n, lo=-1.0, hi=1.0):
        out = np.empty(n, np.float32)
        lib().ck_rng_uniform(self.h, out.ctypes.data, n, lo, hi)
        return out

    def normal(self, n, scale=1.0):
        out = np.empty(n, np.float32)
        lib().ck_rng_normal(self.h, out.ctypes.data, n, scale)
        return out

    def labels(self, n, classes):
        out = np.empty(n, np.float32)
        lib().ck_rng_labels(self.h, out.ctypes.data, n, classes)
        return out


def lenet(batch=100) -> Net:
    """cnn_mnist LeNet."""
    n = Net("lenet", batch, 10)
    n.inputs = {"data": (28, 28, 1, batch), "label": (1, 1, 1, batch)}
    x = n.conv("conv1", "data", "x1", 5, 5, 1, 20)
    x = n.pool("pool1", x, "x2", 2, 2)
    x = n.conv("conv2", x, "x3", 5, 5, 20, 50)
    x = n.pool("pool2", x, "x4", 2, 2)
    x = n.conv("conv3", x, "x5", 4, 4, 50, 500)
    x = n.relu("relu3", x, "x6")
    x = n.conv("conv4", x, "x7", 1, 1, 500, 10)
    n.loss(x)
    return n


def cifar(batch=128) -> Net:
    """CIFAR-10 quick with LRN and max/avg pooling.  LRN
    parameters (3, 1, 5e-5/3, 0.75) are this build's choice, as documented."""
    n = Net("cifar", batch, 10)
    n.inputs = {"data": (32, 32, 3, batch), "label": (1, 1, 1, batch)}
    pad = (0, 1, 0, 1)
    lrn = (3, 1.0, 5e-5 / 3, 0.75)
    x = n.conv("conv1", "data", "x1", 5, 5, 3, 32, pad=(2, 2, 2, 2))
    x = n.pool("pool1", x, "x2", 3, 2, pad, "max")
    x = n.relu("relu1", x, "x3")
    x = n.lrn("norm1", x, "x4", *lrn)
    x = n.conv("conv2", x, "x5", 5, 5, 32, 32, pad=(2, 2, 2, 2))
    x = n.relu("relu2", x, "x6")
    x = n.pool("pool2", x, "x7", 3, 2, pad, "avg")
    x = n.lrn("norm2", x, "x8", *lrn)
    x = n.conv("conv3", x, "x9", 5, 5, 32, 64, pad=(2, 2, 2, 2))
    x = n.relu("relu3", x, "x10")
    x = n.pool("pool3", x, "x11", 3, 2, pad, "avg")
    x = n.conv("conv4", x, "x12", 4, 4, 64, 64)
    x = n.relu("relu4", x, "x13")
    x = n.conv("conv5", x, "x14", 1, 1, 64, 10)
    n.loss(x)
    return n


def alexnet(batch=256) -> Net:
    """imagenet-caffe-alex (bvlc order; pool pads [0 1 0 1] from
    caffe_pool_equiv, geometry.cpp:97-118), no dropout (not a block)."""
    n = Net("alexnet", batch, 1000)
    n.inputs = {"data": (227, 227, 3, batch), "label": (1, 1, 1, batch)}
    pad = (0, 1, 0, 1)
    lrn = (5, 1.0, 2e-5, 0.75)
    x = n.conv("conv1", "data", "c1", 11, 11, 3, 96, stride=4)
    x = n.relu("relu1", x, "r1")
    x = n.lrn("norm1", x, "n1", *lrn)
    x = n.pool("pool1", x, "p1", 3, 2, pad)
    x = n.conv("conv2", x, "c2", 5, 5, 96, 256, pad=(2, 2, 2, 2), groups=2)
    x = n.relu("relu2", x, "r2")
    x = n.lrn("norm2", x, "n2", *lrn)
    x = n.pool("pool2", x, "p2", 3, 2, pad)
    x = n.conv("conv3", x, "c3", 3, 3, 256, 384, pad=(1, 1, 1, 1))
    x = n.relu("relu3", x, "r3")
    x = n.conv("conv4", x, "c4", 3, 3, 384, 384, pad=(1, 1, 1, 1), groups=2)
    x = n.relu("relu4", x, "r4")
    x = n.conv("conv5", x, "c5", 3, 3, 384, 256, pad=(1, 1, 1, 1), groups=2)
    x = n.relu("relu5", x, "r5")
    x = n.pool("pool5", x, "p5", 3, 2, pad)
    x = n.conv("fc6", x, "f6", 6, 6, 256, 4096)
    x = n.relu("relu6", x, "r6")
    x = n.conv("fc7", x, "f7", 1, 1, 4096, 4096)
    x = n.relu("relu7", x, "r7")
    x = n.conv("fc8", x, "f8", 1, 1, 4096, 1000)
    n.loss(x)
    return n


def vgg16_bn(batch=64, image=224) -> Net:
    """VGG-VD-16 with batch norm after every conv."""
    n = Net("vgg16bn", batch, 1000)
    n.inputs = {"data": (image, image, 3, batch), "label": (1, 1, 1, batch)}
    cfg = [[64, 64], [128, 128], [256, 256, 256], [512, 512, 512], [512, 512, 512]]
    x, cin, k = "data", 3, 0
    for gi, group in enumerate(cfg):
        for cout in group:
            k += 1
            x = n.conv(f"conv{k}", x, f"c{k}", 3, 3, cin, cout, pad=(1, 1, 1, 1))
            x = n.bnorm(f"bn{k}", x, f"b{k}", cout)
            x = n.relu(f"relu{k}", x, f"r{k}")
            cin = cout
        x = n.pool(f"pool{gi + 1}", x, f"p{gi + 1}", 2, 2)
    side = image // 32
    x = n.conv("fc6", x, "f6", side, side, 512, 4096)
    x = n.relu("relu_fc6", x, "rf6")
    x = n.conv("fc7", x, "f7", 1, 1, 4096, 4096)
    x = n.relu("relu_fc7", x, "rf7")
    x = n.conv("fc8", x, "f8", 1, 1, 4096, 1000)
    n.loss(x)
    return n


NETS = {"lenet": lenet, "cifar": cifar, "alexnet": alexnet, "vgg16bn": vgg16_bn}
# BASELINE.json configs: the batch each network is quoted at
DEFAULT_BATCH = {"lenet": 100, "cifar": 128, "alexnet": 256, "vgg16bn": 64}
