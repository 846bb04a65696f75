"""Host-side readers/writers for the reference's on-disk formats.

* ``weights.bin`` — proj/src/model.cpp:361-427: magic "PAHQ", u32 version 1,
  eight u32 ModelConfig fields, every matrix as row-major FP32 in canonical
  ``for_each_matrix`` order (model.cpp:285-308), then a u64 FNV-1a-64 of all
  preceding bytes.
* ``dataset.jsonl`` — proj/src/patching.cpp:16-62: one
  ``{"clean":[..],"corrupt":[..],"answer":a,"distractor":d}`` per line.

Errors mirror the reference's ``WeightIoError`` hierarchy
(proj/include/circuitquant/model.hpp:123-130).
"""
from __future__ import annotations

import json
import struct
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

MAGIC = b"PAHQ"
VERSION = 1
HEADER_BYTES = 4 + 4 + 8 * 4


class WeightIoError(RuntimeError):
    pass


class BadMagicError(WeightIoError):
    pass


class BadVersionError(WeightIoError):
    pass


class BadShapeError(WeightIoError):
    pass


class TruncatedError(WeightIoError):
    pass


class BadChecksumError(WeightIoError):
    pass


@dataclass(frozen=True)
class ModelConfig:
    """ModelConfig (proj/include/circuitquant/model.hpp:31-48)."""

    n_layers: int = 1
    n_heads: int = 1
    d_model: int = 8
    d_k: int = 8
    vocab: int = 16
    seq_len: int = 8
    batch: int = 1
    has_mlp: int = 0

    def validate(self) -> None:  # model.cpp:144-155
        if self.n_layers < 1:
            raise ValueError("ModelConfig: n_layers must be >= 1")
        if self.n_heads < 1:
            raise ValueError("ModelConfig: n_heads must be >= 1")
        if self.d_model < 1 or self.d_k < 1:
            raise ValueError("ModelConfig: d_model and d_k must be >= 1")
        if self.n_heads * self.d_k != self.d_model:
            raise ValueError("ModelConfig: n_heads * d_k must equal d_model")
        if self.vocab < 2:
            raise ValueError("ModelConfig: vocab must be >= 2")
        if self.seq_len < 1:
            raise ValueError("ModelConfig: seq_len must be >= 1")
        if self.batch != 1:
            raise ValueError("ModelConfig: batch must be 1")
        if self.has_mlp > 1:
            raise ValueError("ModelConfig: has_mlp must be 0 or 1")

    def fields8(self) -> List[int]:
        return [self.n_layers, self.n_heads, self.d_model, self.d_k, self.vocab,
                self.seq_len, self.batch, self.has_mlp]

    def matrix_specs(self):
        """(name, shape) in canonical order (model.cpp:285-308)."""
        d, v, s = self.d_model, self.vocab, self.seq_len
        out = [("w_e", (v, d)), ("w_pos", (s, d))]
        for l in range(self.n_layers):
            p = f"l{l}."
            out += [(p + "ln1_g", (d,)), (p + "ln1_b", (d,)), (p + "w_q", (d, d)),
                    (p + "w_k", (d, d)), (p + "w_v", (d, d)), (p + "w_o", (d, d))]
            if self.has_mlp:
                out += [(p + "ln2_g", (d,)), (p + "ln2_b", (d,)), (p + "w_in", (d, 4 * d)),
                        (p + "w_out", (4 * d, d))]
        out += [("ln_f_g", (d,)), ("ln_f_b", (d,)), ("w_u", (d, v))]
        return out


def fnv1a64(data: bytes, seed: int = 14695981039346656037) -> int:
    """FNV-1a-64 (model.cpp:324-332), pure Python (small files only)."""
    h = seed
    for b in data:
        h = ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def _fnv_fast(data: bytes) -> int:
    """Same hash via libcqg.so's host helper when available (large files)."""
    if len(data) > (1 << 20):
        try:
            from .engine import fnv1a64 as native
            return native(data)
        except Exception:
            pass
    return fnv1a64(data)


@dataclass
class WeightSet:
    cfg: ModelConfig
    mats: List[np.ndarray] = field(default_factory=list)  # canonical order, float32

    def named(self):
        return {n: m for (n, _), m in zip(self.cfg.matrix_specs(), self.mats)}


def save_weights(w: WeightSet, path: str) -> None:
    w.cfg.validate()
    buf = bytearray(MAGIC)
    buf += struct.pack("<I", VERSION)
    buf += struct.pack("<8I", *w.cfg.fields8())
    for (name, shape), m in zip(w.cfg.matrix_specs(), w.mats):
        a = np.ascontiguousarray(m, dtype=np.float32)
        if a.shape != shape:
            raise BadShapeError(f"save_weights: {name} has shape {a.shape}, want {shape}")
        buf += a.tobytes()
    buf += struct.pack("<Q", _fnv_fast(bytes(buf)))
    with open(path, "wb") as f:
        f.write(buf)


def load_weights(path: str, verify_checksum: bool = True) -> WeightSet:
    try:
        with open(path, "rb") as f:
            buf = f.read()
    except OSError as e:
        raise WeightIoError(f"load_weights: cannot open {path}") from e
    if len(buf) < 4 or buf[:4] != MAGIC:
        raise BadMagicError(f"load_weights: bad magic in {path}")
    if len(buf) < HEADER_BYTES:
        raise TruncatedError(f"load_weights: truncated header in {path}")
    (version,) = struct.unpack_from("<I", buf, 4)
    if version != VERSION:
        raise BadVersionError(f"load_weights: unsupported version {version}")
    cfg = ModelConfig(*struct.unpack_from("<8I", buf, 8))
    try:
        cfg.validate()
    except ValueError as e:
        raise BadShapeError(f"load_weights: {e}") from e
    specs = cfg.matrix_specs()
    payload = sum(int(np.prod(s)) * 4 for _, s in specs)
    expect = HEADER_BYTES + payload + 8
    if len(buf) < expect:
        raise TruncatedError(f"load_weights: file shorter than header implies in {path}")
    if len(buf) > expect:
        raise BadShapeError(f"load_weights: trailing bytes after checksum in {path}")
    if verify_checksum:
        (stored,) = struct.unpack_from("<Q", buf, len(buf) - 8)
        if _fnv_fast(buf[:-8]) != stored:
            raise BadChecksumError(f"load_weights: checksum mismatch in {path}")
    mats = []
    off = HEADER_BYTES
    for _, shape in specs:
        n = int(np.prod(shape))
        mats.append(np.frombuffer(buf, dtype="<f4", count=n, offset=off).reshape(shape).copy())
        off += 4 * n
    return WeightSet(cfg, mats)


@dataclass
class Dataset:
    """ContrastPair list (proj/include/circuitquant/patching.hpp:21-28) as arrays."""

    clean: np.ndarray       # [B][S] int32
    corrupt: np.ndarray     # [B][S] int32
    answer: np.ndarray      # [B] int32
    distractor: np.ndarray  # [B] int32

    def __len__(self) -> int:
        return int(self.clean.shape[0])

    def subset(self, idx) -> "Dataset":
        return Dataset(self.clean[idx].copy(), self.corrupt[idx].copy(),
                       self.answer[idx].copy(), self.distractor[idx].copy())


def load_dataset_jsonl(path: str) -> Dataset:
    clean, corrupt, ans, dis = [], [], [], []
    with open(path) as f:
        for line_no, line in enumerate(f, 1):
            if not line.strip():
                continue
            try:
                j = json.loads(line)
            except json.JSONDecodeError as e:
                raise RuntimeError(f"load_dataset_jsonl: line {line_no}: {e}") from e
            for k in ("clean", "corrupt", "answer", "distractor"):
                if k not in j:
                    raise RuntimeError(f"load_dataset_jsonl: line {line_no}: missing field")
            clean.append(j["clean"])
            corrupt.append(j["corrupt"])
            ans.append(j["answer"])
            dis.append(j["distractor"])
    return Dataset(np.asarray(clean, np.int32).reshape(len(clean), -1),
                   np.asarray(corrupt, np.int32).reshape(len(corrupt), -1),
                   np.asarray(ans, np.int32), np.asarray(dis, np.int32))


def save_dataset_jsonl(ds: Dataset, path: str) -> None:
    with open(path, "w") as f:
        for i in range(len(ds)):
            f.write(json.dumps({"answer": int(ds.answer[i]), "clean": [int(t) for t in ds.clean[i]],
                                "corrupt": [int(t) for t in ds.corrupt[i]],
                                "distractor": int(ds.distractor[i])}, separators=(",", ":")) + "\n")


def validate_dataset(ds: Dataset, cfg: ModelConfig) -> None:
    """patching.cpp:64-81"""
    if len(ds) == 0:
        raise ValueError("validate_dataset: empty dataset")
    v = cfg.vocab
    for i in range(len(ds)):
        at = f"validate_dataset: item {i}"
        if ds.clean.shape[1] != cfg.seq_len or ds.corrupt.shape[1] != cfg.seq_len:
            raise ValueError(at + ": prompt length must equal seq_len")
        if ds.clean[i].min() < 0 or ds.clean[i].max() >= v:
            raise ValueError(at + ": clean token out of range")
        if ds.corrupt[i].min() < 0 or ds.corrupt[i].max() >= v:
            raise ValueError(at + ": corrupt token out of range")
        if not (0 <= ds.answer[i] < v and 0 <= ds.distractor[i] < v):
            raise ValueError(at + ": answer tokens out of range")
        if ds.answer[i] == ds.distractor[i]:
            raise ValueError(at + ": answer equals distractor")
