"""Synthetic inputs in the reference's formats.

``random_weights`` / ``random_dataset`` restate the reference's portable test
generators (proj/tests/support.hpp:19-76): raw ``std::mt19937`` draws (numpy's
MT19937 with legacy seeding is the same engine), mapped exactly as the C++
does, so the bytes equal what the reference writes (pinned by
tests/test_synth.py against oracle/_ref).

``ioi_dataset`` / ``greater_than_dataset`` / ``docstring_dataset`` are the
IOI/Greater-Than/docstring-*shaped* prompt generators BASELINE.json configs
2-5 name. The reference has no such generators (SURVEY.md §7 hard part 6), so
these are builder restatements: fixed-template token sequences with seeded
name/number slots. They only shape the token statistics; the forward pass and
scoring semantics are unaffected.
"""
from __future__ import annotations

import numpy as np

from .formats import Dataset, ModelConfig, WeightSet


class _Mt:
    """std::mt19937 stream (support.hpp uses raw draws only)."""

    def __init__(self, seed: int):
        self.bg = np.random.MT19937()
        self.bg._legacy_seeding(int(seed) & 0xFFFFFFFF)

    def raw(self, n: int) -> np.ndarray:
        return self.bg.random_raw(n).astype(np.uint64)

    def rnd(self, n: int) -> np.ndarray:
        # support.hpp:21-23: float((rng() >> 8) * 0x1p-24) - 0.5f
        r = (self.raw(n) >> np.uint64(8)).astype(np.float64) * 2.0 ** -24
        return r.astype(np.float32) - np.float32(0.5)


def random_weights(cfg: ModelConfig, seed: int, weight_scale: float = 0.0) -> WeightSet:
    """support.hpp:27-54."""
    cfg.validate()
    rng = _Mt(seed)
    f32 = np.float32
    ws = f32(weight_scale) if weight_scale > 0.0 else f32(0.8) / np.sqrt(f32(cfg.d_model))

    def fill(shape, scale):
        n = int(np.prod(shape))
        return (f32(scale) * rng.rnd(n)).astype(np.float32).reshape(shape)

    def gain(n):
        return (f32(1.0) + f32(0.2) * rng.rnd(n)).astype(np.float32)

    d, v, s = cfg.d_model, cfg.vocab, cfg.seq_len
    mats = [fill((v, d), 1.0), fill((s, d), 0.5)]
    for _ in range(cfg.n_layers):
        mats += [gain(d), fill((d,), 0.1), fill((d, d), ws), fill((d, d), ws),
                 fill((d, d), ws), fill((d, d), ws)]
        if cfg.has_mlp:
            mats += [gain(d), fill((d,), 0.1), fill((d, 4 * d), ws), fill((4 * d, d), ws)]
    mats += [gain(d), fill((d,), 0.1), fill((d, v), 1.0)]
    return WeightSet(cfg, mats)


def random_dataset(cfg: ModelConfig, items: int, seed: int) -> Dataset:
    """support.hpp:56-76 (rng() % vocab draws, distractor redrawn until != answer)."""
    rng = _Mt(seed)
    S, V = cfg.seq_len, np.uint64(cfg.vocab)
    clean = np.zeros((items, S), np.int32)
    corrupt = np.zeros((items, S), np.int32)
    ans = np.zeros(items, np.int32)
    dis = np.zeros(items, np.int32)
    for i in range(items):
        clean[i] = (rng.raw(S) % V).astype(np.int32)
        corrupt[i] = (rng.raw(S) % V).astype(np.int32)
        ans[i] = int(rng.raw(1)[0] % V)
        while True:
            dis[i] = int(rng.raw(1)[0] % V)
            if dis[i] != ans[i]:
                break
    return Dataset(clean, corrupt, ans, dis)


def _template_tokens(rng: np.random.Generator, vocab: int, n: int, avoid) -> np.ndarray:
    pool = np.setdiff1d(np.arange(vocab, dtype=np.int32), np.asarray(sorted(avoid), np.int32))
    return rng.choice(pool, size=n, replace=False).astype(np.int32)


def ioi_dataset(cfg: ModelConfig, items: int, seed: int) -> Dataset:
    """IOI-shaped prompts (SURVEY.md §8(d) proposal): BOS When A and B went to
    the <place>, B gave a <obj> to -> answer A (indirect object), distractor B.
    Corrupt replaces both names with fresh names C, D. Filler words are
    fixed per seed; names are drawn per item. Pads/truncates to seq_len."""
    S, V = cfg.seq_len, cfg.vocab
    rng = np.random.default_rng(seed)
    n_names = max(8, min(200, V // 8))
    names = _template_tokens(rng, V, n_names, avoid=[])
    words = _template_tokens(rng, V, 16, avoid=names)
    bos, when, and_, went, to, the, gave, a = words[:8]
    places, objs = words[8:12], words[12:16]
    clean = np.zeros((items, S), np.int32)
    corrupt = np.zeros((items, S), np.int32)
    ans = np.zeros(items, np.int32)
    dis = np.zeros(items, np.int32)
    for i in range(items):
        A, B, C, D = rng.choice(names, 4, replace=False)
        place, obj = rng.choice(places), rng.choice(objs)

        def prompt(x, y):
            seq = [bos, when, x, and_, y, went, to, the, place, y, gave, a, obj, to]
            seq = [bos] * max(0, S - len(seq)) + seq
            return np.asarray(seq[-S:], np.int32)

        clean[i], corrupt[i] = prompt(A, B), prompt(C, D)
        ans[i], dis[i] = A, B
    return Dataset(clean, corrupt, ans, dis)


def greater_than_dataset(cfg: ModelConfig, items: int, seed: int) -> Dataset:
    """Greater-Than-shaped prompts: "The <noun> lasted from the year 17YY to the
    year 17" -> answer any two-digit token > YY; corrupt uses YY = 01. We
    use the answer (YY+1 .. ) / distractor (YY-1) pair."""
    S, V = cfg.seq_len, cfg.vocab
    rng = np.random.default_rng(seed + 7)
    digits = _template_tokens(rng, V, 100, avoid=[])  # tokens "00".."99"
    words = _template_tokens(rng, V, 8, avoid=digits)
    the, lasted, from_, year, to, century = words[:6]
    nouns = words[6:8]
    clean = np.zeros((items, S), np.int32)
    corrupt = np.zeros((items, S), np.int32)
    ans = np.zeros(items, np.int32)
    dis = np.zeros(items, np.int32)
    for i in range(items):
        yy = int(rng.integers(2, 98))
        noun = rng.choice(nouns)

        def prompt(y):
            seq = [the, noun, lasted, from_, the, year, century, digits[y], to, the, year, century]
            seq = [the] * max(0, S - len(seq)) + seq
            return np.asarray(seq[-S:], np.int32)

        clean[i], corrupt[i] = prompt(yy), prompt(1)
        ans[i], dis[i] = digits[yy + 1], digits[yy - 1]
    return Dataset(clean, corrupt, ans, dis)


def docstring_dataset(cfg: ModelConfig, items: int, seed: int) -> Dataset:
    """Docstring-shaped prompts: def f(<a>, <b>, <c>): \"\"\" ... :param <a>: ...
    :param <b>: ... :param -> answer <c>; corrupt renames the def arguments."""
    S, V = cfg.seq_len, cfg.vocab
    rng = np.random.default_rng(seed + 13)
    idents = _template_tokens(rng, V, max(16, min(400, V // 4)), avoid=[])
    words = _template_tokens(rng, V, 10, avoid=idents)
    def_, lpar, comma, rpar, quote, param, colon, desc = words[:8]
    clean = np.zeros((items, S), np.int32)
    corrupt = np.zeros((items, S), np.int32)
    ans = np.zeros(items, np.int32)
    dis = np.zeros(items, np.int32)
    for i in range(items):
        f, a, b, c, x, y, z = rng.choice(idents, 7, replace=False)

        def prompt(p, q, r):
            seq = [def_, f, lpar, p, comma, q, comma, r, rpar, colon, quote, desc, desc,
                   param, a, colon, desc, desc, param, b, colon, desc, desc, param]
            if len(seq) > S:  # compact form for short contexts
                seq = [def_, p, q, r, quote, param, a, desc, param, b, desc, param]
            seq = [quote] * max(0, S - len(seq)) + seq
            return np.asarray(seq[-S:], np.int32)

        clean[i], corrupt[i] = prompt(a, b, c), prompt(x, y, z)
        ans[i], dis[i] = c, (b if b != c else a)
    return Dataset(clean, corrupt, ans, dis)
