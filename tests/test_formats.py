"""Host formats and generators against the reference's (model.cpp:361-427,
patching.cpp:16-62, proj/tests/support.hpp:19-76)."""
import os

import numpy as np
import pytest

from paper_2510_23264_b200 import formats, synth
from helpers import SMALL, TINY, TOY, bits


def test_weights_round_trip_and_errors(tmp_path):
    w = synth.random_weights(TINY, 9)
    p = str(tmp_path / "w.bin")
    formats.save_weights(w, p)
    r = formats.load_weights(p)
    assert r.cfg == TINY
    assert all(np.array_equal(bits(a), bits(b)) for a, b in zip(w.mats, r.mats))
    raw = open(p, "rb").read()
    bad = bytearray(raw)
    bad[0] = ord("X")
    open(p, "wb").write(bad)
    with pytest.raises(formats.BadMagicError):
        formats.load_weights(p)
    bad = bytearray(raw)
    bad[100] ^= 1
    open(p, "wb").write(bad)
    with pytest.raises(formats.BadChecksumError):
        formats.load_weights(p)
    open(p, "wb").write(raw[:-20])
    with pytest.raises(formats.TruncatedError):
        formats.load_weights(p)
    open(p, "wb").write(raw + b"\0")
    with pytest.raises(formats.BadShapeError):
        formats.load_weights(p)
    bad = bytearray(raw)
    bad[4] = 2
    open(p, "wb").write(bad)
    with pytest.raises(formats.BadVersionError):
        formats.load_weights(p)


@pytest.mark.parametrize("cfg,seed", [(TINY, 101), (TOY, 1), (SMALL, 7)])
def test_generators_equal_reference_bytes(ref, cfg, seed, tmp_path):
    wp, dp = str(tmp_path / "w.bin"), str(tmp_path / "d.jsonl")
    ref.gen_random(cfg.fields8(), seed, 5, seed + 1, wp, dp)
    w = synth.random_weights(cfg, seed)
    p2 = str(tmp_path / "w2.bin")
    formats.save_weights(w, p2)
    assert open(wp, "rb").read() == open(p2, "rb").read()
    a = formats.load_dataset_jsonl(dp)
    b = synth.random_dataset(cfg, 5, seed + 1)
    for f in ("clean", "corrupt", "answer", "distractor"):
        assert np.array_equal(getattr(a, f), getattr(b, f))


def test_dataset_jsonl_round_trip(tmp_path):
    ds = synth.random_dataset(TOY, 4, 3)
    p = str(tmp_path / "d.jsonl")
    formats.save_dataset_jsonl(ds, p)
    r = formats.load_dataset_jsonl(p)
    assert np.array_equal(r.clean, ds.clean) and np.array_equal(r.answer, ds.answer)
    formats.validate_dataset(r, TOY)
    bad = formats.Dataset(ds.clean.copy(), ds.corrupt, ds.answer, ds.answer.copy())
    with pytest.raises(ValueError):
        formats.validate_dataset(bad, TOY)


@pytest.mark.parametrize("gen", [synth.ioi_dataset, synth.greater_than_dataset,
                                 synth.docstring_dataset])
def test_task_shaped_generators_are_valid(gen):
    from helpers import GPT2S
    ds = gen(GPT2S, 64, 1)
    formats.validate_dataset(ds, GPT2S)
    assert len(ds) == 64 and not np.array_equal(ds.clean, ds.corrupt)
