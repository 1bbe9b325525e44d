"""The cnn_train loop around the device step and the model
files: lossless model round trip, checkpoint resume
equal to straight-through training bitwise, the NaN abort, the no-op and
learning properties."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


def lenet_graph(math="tf32", batch=16):
    from paper_1412_4564_b200 import nets
    from paper_1412_4564_b200.graph import Graph
    net = nets.lenet(batch=batch)
    g = Graph(math=math)
    net.build(g)
    g.finalize()
    for k, v in net.init_params().items():
        g.set(k, v)
    return net, g


def toy_data(n=80, seed=5):
    """Two classes separable by the sign of the mean brightness of the left
    half of the image (a LeNet-shaped synthetic set)."""
    r = O.Rng(seed)
    x = r.uniform(n * 28 * 28, 0.0, 1.0).reshape(n, 28, 28)
    y = (np.arange(n) % 2).astype(np.float32)
    x[y == 1, :14, :] += 0.5
    return x.astype(np.float32).ravel(), (y + 1).astype(np.float32)


def test_model_round_trip(tmp_path):
    from paper_1412_4564_b200.graph import Graph
    net, g = lenet_graph()
    g.set_meta("averageImage", "0.1307")
    g.set_meta("inputSize", "28 28 1")
    g.save(tmp_path / "m1")
    g2 = Graph.load(tmp_path / "m1", math="tf32")
    g2.save(tmp_path / "m2")
    for f in sorted(p.name for p in (tmp_path / "m1").iterdir()):
        assert (tmp_path / "m1" / f).read_bytes() == (tmp_path / "m2" / f).read_bytes(), f
    assert g2.get_meta("averageImage") == "0.1307" and g2.get_meta("inputSize") == "28 28 1"
    x = O.Rng(1).uniform(28 * 28 * 16)
    lab = O.Rng(2).labels(16, 10)
    outs = []
    for gg in (g, g2):
        gg.set("data", x)
        gg.set("label", lab)
        gg.forward()
        outs.append(gg.get("x7"))
    assert np.array_equal(outs[0], outs[1])  # loaded model forward == pre-save, exactly


def test_model_load_errors(tmp_path):
    from paper_1412_4564_b200._lib import DataError
    from paper_1412_4564_b200.graph import Graph
    _, g = lenet_graph()
    g.save(tmp_path / "m")
    (tmp_path / "m" / "conv2f.blob").unlink()
    with pytest.raises(DataError, match="missing blob 'conv2f.blob'"):
        Graph.load(tmp_path / "m")
    g.save(tmp_path / "v")
    m = (tmp_path / "v" / "manifest.txt").read_text().replace("ck-manifest 1", "ck-manifest 9")
    (tmp_path / "v" / "manifest.txt").write_text(m)
    with pytest.raises(DataError, match="version 9 not supported"):
        Graph.load(tmp_path / "v")


def test_checkpoint_resume_is_bitwise(tmp_path):
    """2 epochs then resume 3 == 5 straight, bitwise."""
    from paper_1412_4564_b200.graph import Trainer
    x, y = toy_data()
    net, g = lenet_graph()
    t = Trainer(g, lr=0.002, momentum=0.9, weight_decay=5e-4)
    straight = t.fit(x, y, epochs=5, seed=11)
    want = {p: g.get(p) for p, _, _ in net.params}
    net, g = lenet_graph()
    t = Trainer(g, lr=0.002, momentum=0.9, weight_decay=5e-4)
    first = t.fit(x, y, epochs=2, seed=11, checkpoint=str(tmp_path / "ck"))
    del t, g
    net, g = lenet_graph()
    g.set("conv1f", np.zeros(5 * 5 * 20, np.float32))  # clobbered: the checkpoint restores it
    t = Trainer(g, lr=0.002, momentum=0.9, weight_decay=5e-4)
    state, epoch = t.load(str(tmp_path / "ck"))
    assert epoch == 2
    rest = t.fit(x, y, epochs=5, seed=11, start_epoch=epoch, rng_state=state)
    for p in want:
        assert np.array_equal(g.get(p), want[p]), p
    assert [r["loss"] for r in first + rest] == [r["loss"] for r in straight]
    # learning on the separable toy set: mean loss of epoch 5 < epoch 1
    assert straight[-1]["loss"] < straight[0]["loss"]
    assert set(straight[0]) >= {"epoch", "loss", "top1", "top5", "sec", "images_per_sec"}


def test_lr_zero_is_noop():
    """learning-rate 0 -> final params identical to initial."""
    from paper_1412_4564_b200.graph import Trainer
    x, y = toy_data(32)
    net, g = lenet_graph()
    before = {p: g.get(p) for p, _, _ in net.params}
    Trainer(g, lr=0.0, momentum=0.9, weight_decay=0.0).fit(x, y, epochs=2, seed=3)
    for p in before:
        assert np.array_equal(g.get(p), before[p]), p


@pytest.mark.parametrize("graph_mode", [False, True])
def test_nan_loss_aborts(graph_mode):
    """a NaN loss aborts training with a diagnostic (NumericError,
    exit code 3 of the CLI), eager or from a replayed CUDA graph."""
    from paper_1412_4564_b200._lib import NumericError
    from paper_1412_4564_b200.graph import Trainer
    net, g = lenet_graph()
    x, y = toy_data(16)
    g.set("data", x)
    g.set("label", y)
    t = Trainer(g, lr=0.01)
    t.set_graph(graph_mode)
    stream = torch.cuda.Stream()
    for _ in range(3):
        t.step(stream=stream.cuda_stream)
    # (a NaN pixel alone may vanish: max pooling's `v > best` drops NaN
    # unless it is a window's first element, as in pool.cpp:59-64)
    g.set("conv4b", np.full(10, np.nan, np.float32))
    with pytest.raises(NumericError, match="non-finite loss"):
        t.step(stream=stream.cuda_stream)
