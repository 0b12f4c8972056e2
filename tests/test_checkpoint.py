"""QQQ1 checkpoint container and GPU layer loader, against a
checkpoint written by the reference itself (tests/golden/make_golden_checkpoint.py)
and the reference's own validation cases (pkg/tests/test_checkpoint.py)."""

import json
import os
import struct

import numpy as np
import pytest

from paper_2406_09904_b200.checkpoint import (ALIGN, MAGIC, Checkpoint, TensorRecord, load_layers,
                                              read_checkpoint, store_layer, write_checkpoint)
from paper_2406_09904_b200.errors import CheckpointFormatError

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CKPT = os.path.join(GOLD, "layers.qqq")


def _sample():
    rng = np.random.default_rng(3)
    ck = Checkpoint(metadata={"v": 1, "note": "sample"})
    ck.add("w.f32", "f32", rng.standard_normal((6, 4)).astype(np.float32))
    ck.add("a.q", "i8", rng.integers(-127, 128, (5, 7)).astype(np.int8))
    ck.add("h.f16", "f16", rng.standard_normal(9).astype(np.float16))
    ck.add("w.q4", "i4p", rng.integers(0, 256, (5, 3)).astype(np.uint8), rows=9)
    return ck


def test_reference_checkpoint_reads_and_rewrites_byte_identical(tmp_path):
    ck = read_checkpoint(CKPT)
    assert set(ck.metadata["layers"]) == {"blk0.qkv", "blk0.down"}
    assert ck.tensors["blk0.qkv.q4"].dtype == "i4p" and ck.tensors["blk0.qkv.q4"].rows == 256
    p = str(tmp_path / "re.qqq")
    write_checkpoint(ck, p)
    assert open(p, "rb").read() == open(CKPT, "rb").read()


def test_round_trip_and_canonical_bytes(tmp_path):
    ck = _sample()
    p1, p2 = str(tmp_path / "a.qqq"), str(tmp_path / "b.qqq")
    write_checkpoint(ck, p1)
    assert read_checkpoint(p1) == ck
    flipped = Checkpoint(metadata=dict(ck.metadata), tensors=dict(reversed(list(ck.tensors.items()))))
    write_checkpoint(flipped, p2)
    assert open(p1, "rb").read() == open(p2, "rb").read()  # insertion order does not matter
    blob = open(p1, "rb").read()
    assert blob[:4] == MAGIC
    (hlen,) = struct.unpack("<Q", blob[4:12])
    for e in json.loads(blob[12:12 + hlen])["tensors"].values():
        assert e["offset"] % ALIGN == 0


def test_empty_checkpoint(tmp_path):
    p = str(tmp_path / "e.qqq")
    write_checkpoint(Checkpoint(metadata={"v": 1}), p)
    back = read_checkpoint(p)
    assert back.tensors == {} and back.metadata == {"v": 1}


def test_record_validation():
    with pytest.raises(CheckpointFormatError, match="dtype"):
        TensorRecord("f64", np.zeros(3))
    with pytest.raises(CheckpointFormatError, match="row count"):
        TensorRecord("i4p", np.zeros(3, np.uint8))


def _write(tmp_path):
    p = str(tmp_path / "a.qqq")
    write_checkpoint(_sample(), p)
    return p


def _patch(path, mutate):
    blob = open(path, "rb").read()
    (hlen,) = struct.unpack("<Q", blob[4:12])
    header = json.loads(blob[12:12 + hlen])
    data = blob[(12 + hlen + ALIGN - 1) // ALIGN * ALIGN:]
    mutate(header)
    raw = json.dumps(header, sort_keys=True).encode()
    out = MAGIC + struct.pack("<Q", len(raw)) + raw
    out += b"\0" * ((len(out) + ALIGN - 1) // ALIGN * ALIGN - len(out)) + data
    open(path, "wb").write(out)


def _bump(h):
    for e in h["tensors"].values():
        e["offset"] += 1


def _collide(h):
    names = sorted(h["tensors"])
    h["tensors"][names[1]]["offset"] = h["tensors"][names[0]]["offset"]


@pytest.mark.parametrize("defect,match", [
    (lambda p, b: open(p, "wb").write(b"NOPE" + b[4:]), "magic"),
    (lambda p, b: open(p, "wb").write(b[:20]), "truncated"),
    (lambda p, b: open(p, "wb").write(b[:-40]), "past end"),
    (lambda p, b: open(p, "wb").write(b[:12] + b"\xff\xff\xff\xff" + b[16:]), "JSON"),
    (lambda p, b: _patch(p, lambda h: h["tensors"]["a.q"].update(dtype="f64")), "dtype"),
    (lambda p, b: _patch(p, _bump), "aligned"),
    (lambda p, b: _patch(p, lambda h: h["tensors"]["w.f32"].update(shape=[7, 4])), "nbytes"),
    (lambda p, b: _patch(p, _collide), "overlap"),
    (lambda p, b: open(p, "wb").write(MAGIC + struct.pack("<Q", 16) + b'{"metadata": {}}'), "index"),
    (lambda p, b: _patch(p, lambda h: h["tensors"][sorted(h["tensors"])[-1]].update(dtype="xx")), "dtype"),
])
def test_validation(tmp_path, defect, match):  # pkg/tests/test_checkpoint.py TestValidation
    p = _write(tmp_path)
    defect(p, open(p, "rb").read())
    with pytest.raises(CheckpointFormatError, match=match):
        read_checkpoint(p)
    with pytest.raises(CheckpointFormatError, match=match):
        load_layers(p, names=[], device="cpu", prepare=False)  # the loader validates the whole index too


def test_missing_layer_and_tensor(tmp_path):
    p = _write(tmp_path)
    with pytest.raises(CheckpointFormatError, match="no layer"):
        load_layers(p, names=["nope"], device="cpu", prepare=False)


@pytest.mark.gpu
def test_gpu_load_reference_layers_bit_exact(tmp_path):
    """Layers written by the reference, loaded straight to the GPU (weights
    repacked on the GPU at load time): apply_quant_linear equals the
    reference's output on the layers it loads back, bit for bit."""
    import torch

    import paper_2406_09904_b200 as Q

    exp = np.load(os.path.join(GOLD, "layers_expected.npz"))
    layers = load_layers(CKPT)
    assert set(layers) == {"blk0.qkv", "blk0.down"}
    for name, layer in layers.items():
        assert layer.qweights.packed.is_cuda and layer._cache.get("fused") is not None  # (key, FusedScales)
        y = Q.apply_quant_linear(torch.from_numpy(exp[f"{name}.x"]).cuda(), layer)
        assert np.array_equal(y.cpu().numpy().view(np.uint64), exp[f"{name}.y"].view(np.uint64)), name
    # store -> write -> read: the same bytes as the reference wrote
    ck = Checkpoint(metadata={"layers": {}, "model": "golden"})
    for name in sorted(layers, key=lambda n: list(read_checkpoint(CKPT).metadata["layers"]).index(n)):
        store_layer(ck, layers[name])
    p = str(tmp_path / "again.qqq")
    write_checkpoint(ck, p)
    assert open(p, "rb").read() == open(CKPT, "rb").read()
