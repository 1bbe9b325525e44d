"""Host mirror of the reference DAG API (graph.hpp:93-190) over the device
engine in libck.so (engine.cu).

``Graph`` keeps the reference's vocabulary -- add_input / add_param /
add_layer(kind, name, inputs, outputs, hyper) / finalize / forward /
backward -- and the device engine keeps every value and derivative resident
in HBM.  Tensors cross the boundary only through ``set`` / ``get`` copies.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import ck_shape, ck_tensor, lib, raise_for
from .blocks import MATH, handle


def _u64x4(values=None):
    arr = (C.c_uint64 * 4)()
    if values is not None:
        for k, v in enumerate(values):
            arr[k] = int(v)
    return arr


class Graph:
    def __init__(self, math: str = "tf32", device: int | None = None):
        self.hd = handle(device)
        g = C.c_void_p()
        raise_for(lib().ck_graph_create(self.hd.h, C.byref(g)), self.hd.h)
        self.g = g
        self.math = math
        self.shapes = {}
        self.params = []
        self.inputs = []
        self.layers = []

    def __del__(self):
        if getattr(self, "g", None) and _lib._lib is not None:
            _lib._lib.ck_graph_destroy(self.g)
            self.g = None

    def _check(self, code):
        raise_for(code, self.hd.h)

    # -- construction (graph.hpp:96-102) --
    def add_input(self, name, shape):
        self._check(lib().ck_graph_add_input(self.g, name.encode(), ck_shape(*shape)))
        self.shapes[name] = tuple(shape)
        self.inputs.append(name)

    def add_param(self, name, shape):
        self._check(lib().ck_graph_add_param(self.g, name.encode(), ck_shape(*shape)))
        self.shapes[name] = tuple(shape)
        self.params.append(name)

    def add_layer(self, kind, name, inputs, outputs, params=()):
        self.layers.append((kind, name, list(inputs), list(outputs), list(params)))
        p = (C.c_double * max(1, len(params)))(*[float(v) for v in params])
        self._check(lib().ck_graph_add_layer(self.g, kind.encode(), name.encode(),
                                             ",".join(inputs).encode(), ",".join(outputs).encode(),
                                             p, len(params)))

    def finalize(self):
        self._check(lib().ck_graph_finalize(self.g, MATH[self.math]))

    # -- tensors --
    def view(self, name, deriv=False) -> ck_tensor:
        t = ck_tensor()
        self._check(lib().ck_graph_var(self.g, name.encode(), int(deriv), C.byref(t)))
        return t

    def shape(self, name):
        s = self.view(name).shape
        return (s.h, s.w, s.c, s.n)

    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def set(self, name, data):
        """Copy host (numpy) or device (torch) data into a variable."""
        t = self.view(name)
        n = t.shape.h * t.shape.w * t.shape.c * t.shape.n
        if isinstance(data, torch.Tensor):
            src = data.contiguous().float()
            assert src.numel() == n, (name, src.numel(), n)
            self._check(lib().ck_memcpy(self.hd.h, t.data, src.data_ptr(), 4 * n, self._stream()))
            torch.cuda.current_stream().synchronize()
        else:
            arr = np.ascontiguousarray(data, dtype=np.float32)
            assert arr.size == n, (name, arr.size, n)
            self._check(lib().ck_memcpy(self.hd.h, t.data, arr.ctypes.data, 4 * n, self._stream()))
            torch.cuda.current_stream().synchronize()

    def get(self, name, deriv=False) -> np.ndarray:
        t = self.view(name, deriv)
        n = t.shape.h * t.shape.w * t.shape.c * t.shape.n
        out = np.empty(n, np.float32)
        self._check(lib().ck_memcpy(self.hd.h, out.ctypes.data, t.data, 4 * n, self._stream()))
        torch.cuda.current_stream().synchronize()
        return out

    # -- evaluation (graph.cpp:494, :548) --
    def forward(self):
        self._check(lib().ck_graph_forward(self.g, self._stream()))

    def backward(self, objective="objective"):
        self._check(lib().ck_graph_backward(self.g, objective.encode(), self._stream()))

    @property
    def last_launches(self) -> int:
        return lib().ck_graph_last_launches(self.g)

    # -- model files (manifest + blobs, ck_graph_save / ck_graph_load) --
    def save(self, path):
        """Write the model directory: manifest.txt + one blob per parameter."""
        self._check(lib().ck_graph_save(self.g, str(path).encode()))

    @classmethod
    def load(cls, path, math="tf32", device=None):
        """Build, finalize and fill a graph from a model directory."""
        self = cls.__new__(cls)
        self.hd = handle(device)
        self.math = math
        g = C.c_void_p()
        raise_for(lib().ck_graph_load(self.hd.h, str(path).encode(), MATH[math], C.byref(g)),
                  self.hd.h)
        self.g = g
        self.shapes, self.params, self.inputs, self.layers = {}, [], [], []
        for ln in open(f"{path}/manifest.txt"):
            t = ln.split()
            if t and t[0] == "var":
                shape = tuple(int(v) for v in t[3:7])
                self.shapes[t[1]] = shape
                (self.inputs if t[2] == "input" else self.params).append(t[1])
            elif t and t[0] == "layer":
                p = [float(v) for v in t[5][2:].split(",") if v]
                self.layers.append((t[1], t[2], t[3][3:].split(","), t[4][4:].split(","), p))
        return self

    def set_meta(self, key, value):
        self._check(lib().ck_graph_set_meta(self.g, key.encode(), str(value).encode()))

    def get_meta(self, key):
        v = lib().ck_graph_get_meta(self.g, key.encode())
        return None if v is None else v.decode()

    def set_option(self, name: str, value):
        """Engine option (ck_graph_set_option), e.g. ``lrn_grid``."""
        self._check(lib().ck_graph_set_option(self.g, name.encode(), int(value)))

    def set_profiling(self, on: bool):
        self._check(lib().ck_graph_set_profiling(self.g, int(on)))

    def layer_times(self):
        """[(layer, fwd_ms, bwd_ms)] of the last profiled evaluation."""
        torch.cuda.synchronize()
        out = []
        for i in range(lib().ck_graph_layer_count(self.g)):
            f, b = C.c_float(), C.c_float()
            self._check(lib().ck_graph_layer_ms(self.g, i, C.byref(f), C.byref(b)))
            out.append((lib().ck_graph_layer_name(self.g, i).decode(), f.value, b.value))
        return out


class Feeder:
    """cnn_train's batch prefetch (cnn_train.m ``opts.prefetch``) for a
    device-resident graph: two device buffers per input, alternated.  ``put``
    copies the next batch's pinned host tensors into the free buffer on a copy
    stream while the current step computes; ``take`` (on the compute stream)
    waits for that copy and binds the graph's inputs to the buffer
    (``ck_graph_bind_input``: no device-to-device copy; a trainer replays one
    captured graph per binding).  ``result`` queues an asynchronous device->host
    read of a variable (e.g. the objective) into pinned memory, read back by
    ``collect``."""

    def __init__(self, graph: Graph, names, stream):
        self.g, self.names, self.stream = graph, list(names), stream
        self.copy = torch.cuda.Stream(device=stream.device)
        self.bufs = []
        for _ in range(2):
            bset = {}
            for n in self.names:
                s = graph.view(n).shape
                bset[n] = torch.empty(s.h * s.w * s.c * s.n, dtype=torch.float32,
                                      device=stream.device)
            self.bufs.append(bset)
        self.ready = [torch.cuda.Event(), torch.cuda.Event()]
        self.free = [torch.cuda.Event(), torch.cuda.Event()]
        for e in self.free:
            e.record(stream)
        self.fill = 0        # buffer the next put() fills
        self.queued = []     # filled buffers, oldest first
        self.cur = None      # buffer bound to the graph now
        self.pending = []
        self.h2d_bytes = sum(4 * t.numel() for t in self.bufs[0].values())

    def put(self, host: dict):
        """Queue the H2D copy of one batch (pinned host tensors by name)."""
        k = self.fill
        self.copy.wait_event(self.free[k])  # the step that read buffer k is done
        cs = C.c_void_p(self.copy.cuda_stream)
        for n in self.names:
            src = host[n]
            assert src.is_pinned() and src.numel() == self.bufs[k][n].numel(), n
            self.g._check(lib().ck_memcpy(self.g.hd.h, self.bufs[k][n].data_ptr(), src.data_ptr(),
                                          4 * src.numel(), cs))
        self.ready[k].record(self.copy)
        self.queued.append(k)
        self.fill ^= 1

    def take(self):
        """On the compute stream: wait for the oldest filled buffer and bind the
        graph's inputs to it; the previously bound buffer becomes free once the
        work queued so far (the step that read it) completes."""
        if self.cur is not None:
            self.free[self.cur].record(self.stream)
        k = self.queued.pop(0)
        self.stream.wait_event(self.ready[k])
        for n in self.names:
            self.g._check(lib().ck_graph_bind_input(self.g.g, n.encode(),
                                                    self.bufs[k][n].data_ptr()))
        self.cur = k

    def unbind(self):
        """Restore the graph's own input buffers."""
        for n in self.names:
            self.g._check(lib().ck_graph_bind_input(self.g.g, n.encode(), None))
        if self.cur is not None:
            self.free[self.cur].record(self.stream)
            self.cur = None

    def result(self, name="objective"):
        v = self.g.view(name)
        out = torch.empty(v.shape.h * v.shape.w * v.shape.c * v.shape.n, dtype=torch.float32,
                          pin_memory=True)
        self.g._check(lib().ck_memcpy(self.g.hd.h, out.data_ptr(), v.data, 4 * out.numel(),
                                      C.c_void_p(self.stream.cuda_stream)))
        self.pending.append(out)
        return out

    def collect(self):
        self.stream.synchronize()
        out, self.pending = [t.numpy().copy() for t in self.pending], []
        return out


class Trainer:
    """cnn_train's SGD step with optional NCCL data parallelism."""

    def __init__(self, graph: Graph, objective="objective", lr=0.01, momentum=0.9,
                 weight_decay=5e-4):
        self.graph = graph
        t = C.c_void_p()
        graph._check(lib().ck_trainer_create(graph.g, objective.encode(), lr, momentum,
                                             weight_decay, C.byref(t)))
        self.t = t

    def __del__(self):
        if getattr(self, "t", None) and _lib._lib is not None:
            _lib._lib.ck_trainer_destroy(self.t)
            self.t = None

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        raise_for(lib().ck_nccl_unique_id(buf), None)
        return buf.raw

    def init_dp(self, uid: bytes, rank: int, world: int):
        self.graph._check(lib().ck_trainer_init_dp(self.t, uid, rank, world))

    def set_update_stream(self, on: bool):
        self.graph._check(lib().ck_trainer_set_update_stream(self.t, int(on)))

    def last_timing(self):
        """(fwd_ms, bwd_ms, exchange_tail_ms) of the last profiled step."""
        f, b, c = C.c_float(), C.c_float(), C.c_float()
        self.graph._check(lib().ck_trainer_last_timing(self.t, C.byref(f), C.byref(b), C.byref(c)))
        return f.value, b.value, c.value

    @property
    def allreduces(self) -> int:
        return lib().ck_trainer_allreduce_count(self.t)

    # -- checkpoints (ck_trainer_save / ck_trainer_load) --
    def save(self, path, rng_state=None, epoch=0):
        self.graph._check(lib().ck_trainer_save(self.t, str(path).encode(), _u64x4(rng_state),
                                                int(epoch)))

    def load(self, path):
        """Restore parameters + momentum; returns (rng_state, epoch)."""
        st, ep = _u64x4(), C.c_int64()
        self.graph._check(lib().ck_trainer_load(self.t, str(path).encode(), st, C.byref(ep)))
        return [int(v) for v in st], ep.value

    def fit(self, images, labels, epochs, seed=0, data="data", label="label", checkpoint=None,
            start_epoch=0, rng_state=None, log=None, top_k=5):
        """cnn_train: epochs x ceil(N / batch) SGD steps over
        batches drawn by a per-epoch permutation of the reference generator
        (rng.cpp:51-59, seeded with `seed`); per-epoch records (loss, top-1,
        top-5, sec, images/sec); a checkpoint (parameters, momentum, epoch,
        generator state) after every epoch when `checkpoint` is a directory;
        a non-finite loss aborts with NumericError.  The last
        batch of an epoch is padded with label-0 (ignored, loss.cpp:100)
        samples: exact for networks without batch norm.  Resume with
        (rng_state, epoch) from Trainer.load."""
        import time

        from .nets import Rng
        g = self.graph
        xs, ls = g.shapes[data], g.shapes[label]
        B = xs[3]
        per_x, per_l = xs[0] * xs[1] * xs[2], ls[0] * ls[1] * ls[2]
        images = np.ascontiguousarray(images, np.float32).reshape(-1, per_x)
        labels = np.ascontiguousarray(labels, np.float32).reshape(-1, per_l)
        N = images.shape[0]
        loss_layer = next(l for l in g.layers if l[0] == "loss")
        pred = loss_layer[2][0]
        from . import blocks as _B
        rng = Rng(seed)
        if rng_state is not None:
            lib().ck_rng_set_state(rng.h, _u64x4(rng_state))
        records = []
        xb = np.empty((B, per_x), np.float32)
        lb = np.empty((B, per_l), np.float32)
        for epoch in range(start_epoch, epochs):
            t0 = time.perf_counter()
            perm = np.empty(N, np.int64)
            lib().ck_rng_permutation(rng.h, N, perm.ctypes.data)
            tot_loss = tot1 = totk = 0.0
            for b0 in range(0, N, B):
                idx = perm[b0:b0 + B]
                xb[: len(idx)] = images[idx]
                lb[: len(idx)] = labels[idx]
                xb[len(idx):] = 0.0
                lb[len(idx):] = 0.0  # ignored samples
                g.set(data, xb)
                g.set(label, lb)
                tot_loss += self.step()
                m = _B.loss_metrics(_as_torch(g, pred), _as_torch(g, label), None, top_k)
                m = m.cpu().numpy()
                tot1 += float(m[0])
                totk += float(m[1])
            sec = time.perf_counter() - t0
            rec = {"epoch": epoch + 1, "split": "train", "loss": tot_loss / N, "top1": tot1 / N,
                   "top5": totk / N, "sec": sec, "images_per_sec": N / sec}
            records.append(rec)
            if log:
                log(rec)
            if checkpoint:
                st = _u64x4()
                lib().ck_rng_get_state(rng.h, st)
                self.save(checkpoint, [int(v) for v in st], epoch + 1)
        return records

    def set_graph(self, on: bool):
        """Replay each step as one CUDA graph (ck_trainer_set_graph)."""
        self.graph._check(lib().ck_trainer_set_graph(self.t, int(on)))

    def step(self, want_loss=True, stream=None):
        s = C.c_void_p(stream if stream is not None else torch.cuda.current_stream().cuda_stream)
        if want_loss:
            v = C.c_float()
            self.graph._check(lib().ck_trainer_step(self.t, C.byref(v), s))
            return v.value
        self.graph._check(lib().ck_trainer_step(self.t, None, s))
        return None


def _as_torch(g: Graph, name):
    """A device copy (N, C, W, H) of a graph variable's value, in stream order."""
    t = g.view(name)
    s = t.shape
    n = s.h * s.w * s.c * s.n
    u = torch.empty(n, device="cuda")
    g._check(lib().ck_memcpy(g.hd.h, u.data_ptr(), t.data, 4 * n, g._stream()))
    return u.reshape(s.n, s.c, s.w, s.h)
