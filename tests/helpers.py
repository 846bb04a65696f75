"""Shared test fixtures: model configs of the parity suite and generators.

Weights/datasets come from paper_2510_23264_b200.synth, whose bytes equal
the reference's portable generators (proj/tests/support.hpp:19-76), pinned in
tests/test_formats.py.
"""
import os

import numpy as np

from paper_2510_23264_b200 import formats, synth

# proj/tests/test_patching.cpp:23-33 / test_acdc.cpp:25-35
TINY = formats.ModelConfig(2, 2, 12, 6, 9, 5, 1, 1)
# BASELINE config 1: 2-layer attention-only toy, 4 heads, d=128 (V=512, S=16 proposed)
TOY = formats.ModelConfig(2, 4, 128, 32, 512, 16, 1, 0)
# a small MLP model that exercises every node kind and multi-tile GEMMs
SMALL = formats.ModelConfig(3, 4, 64, 16, 97, 8, 1, 1)
# GPT-2-small shape (BASELINE configs 2-3)
GPT2S = formats.ModelConfig(12, 12, 768, 64, 50257, 16, 1, 1)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def make(cfg, wseed=1, items=3, dseed=2):
    return synth.random_weights(cfg, wseed), synth.random_dataset(cfg, items, dseed)


def write(tmpdir, w, ds):
    wp, dp = os.path.join(tmpdir, "weights.bin"), os.path.join(tmpdir, "dataset.jsonl")
    formats.save_weights(w, wp)
    formats.save_dataset_jsonl(ds, dp)
    return wp, dp


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def random_mask(n_edges, seed, keep=0.6):
    return np.random.RandomState(seed).rand(n_edges) < keep
