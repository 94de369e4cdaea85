"""Checkpoint and metrics interop with the reference.

TBST1 is beastpipe's checkpoint container (pipeline.py:994-1073): the magic b"TBST1", then
per field a little-endian u32 name length, the ASCII name, a u8 dtype code (0 u8, 1 i64,
2 f32, 3 f64), a u8 ndim, ndim u32 dims and the little-endian data, and finally a u64
version.  The reference writes the MLP fields PARAM_FIELDS = (W1, b1, Wp, bp, Wv, bv)
(model.py:14); here the same container carries any ordered set of named arrays:
  * `save_params` / `load_params`: beastpipe MLP parameter sets, byte-identical to
    beastpipe.pipeline.checkpoint / restore (pinned by tests/golden/beastpipe_mlp.tbst1);
  * `checkpoint` / `restore`: an AtariNet state_dict in the upstream torch layout, so
    GPU-trained parameters leave the device in the reference's file format.
`MetricsWriter` appends learn() stats to logs.csv with the reference's columns and number
formats (pipeline.py:55-64, :191-229).
"""
from __future__ import annotations

import csv
import os
import struct
import threading
from dataclasses import dataclass

import numpy as np

MAGIC = b"TBST1"
DTYPE_BY_CODE = {0: np.dtype(np.uint8), 1: np.dtype(np.int64), 2: np.dtype(np.float32),
                 3: np.dtype(np.float64)}
CODE_BY_DTYPE = {v: k for k, v in DTYPE_BY_CODE.items()}
PARAM_FIELDS = ("W1", "b1", "Wp", "bp", "Wv", "bv")  # beastpipe model.py:14


class CheckpointError(ValueError):
    """Bad checkpoint file or shape mismatch (beastpipe pipeline.py:90-91)."""


def write_tbst1(path: str, fields, version: int) -> None:
    """fields: iterable of (name, array); written in order, then the u64 version."""
    with open(path, "wb") as f:
        f.write(MAGIC)
        for name, arr in fields:
            arr = np.asarray(arr)
            dtype = np.dtype(arr.dtype)
            if dtype not in CODE_BY_DTYPE:
                raise CheckpointError(f"{name}: dtype {dtype} not storable")
            raw = name.encode("ascii")
            f.write(struct.pack("<I", len(raw)))
            f.write(raw)
            f.write(struct.pack("<BB", CODE_BY_DTYPE[dtype], arr.ndim))
            f.write(struct.pack(f"<{arr.ndim}I", *arr.shape))
            f.write(np.ascontiguousarray(arr).astype(dtype.newbyteorder("<")).tobytes())
        f.write(struct.pack("<Q", int(version)))


def read_tbst1(path: str, expected_fields=None):
    """-> (dict name -> array in file order, version).  expected_fields pins the names and
    their order (the reference's restore() requires PARAM_FIELDS)."""
    with open(path, "rb") as f:
        data = f.read()
    if data[:5] != MAGIC:
        raise CheckpointError(f"bad magic {data[:5]!r}, expected {MAGIC!r}")
    off = 5
    arrays: dict[str, np.ndarray] = {}
    try:
        while len(data) - off > 8:
            (nlen,) = struct.unpack_from("<I", data, off)
            off += 4
            name = data[off:off + nlen].decode("ascii")
            off += nlen
            if expected_fields is not None:
                k = len(arrays)
                if k >= len(expected_fields) or name != expected_fields[k]:
                    want = expected_fields[k] if k < len(expected_fields) else "<end>"
                    raise CheckpointError(f"unexpected field '{name}', expected '{want}'")
            code, ndim = struct.unpack_from("<BB", data, off)
            off += 2
            if code not in DTYPE_BY_CODE:
                raise CheckpointError(f"{name}: unknown dtype code {code}")
            dims = struct.unpack_from(f"<{ndim}I", data, off)
            off += 4 * ndim
            dtype = DTYPE_BY_CODE[code]
            count = int(np.prod(dims)) if ndim else 1
            arrays[name] = np.frombuffer(data, dtype=dtype.newbyteorder("<"), count=count,
                                         offset=off).astype(dtype).reshape(dims)
            off += count * dtype.itemsize
        (version,) = struct.unpack_from("<Q", data, off)
        off += 8
    except (struct.error, ValueError, UnicodeDecodeError) as exc:
        if isinstance(exc, CheckpointError):
            raise
        raise CheckpointError(f"truncated or corrupt checkpoint: {exc}") from exc
    if off != len(data):
        raise CheckpointError(f"{len(data) - off} trailing bytes in checkpoint")
    if expected_fields is not None and len(arrays) != len(expected_fields):
        raise CheckpointError(f"checkpoint has {len(arrays)} fields, expected {len(expected_fields)}")
    return arrays, int(version)


def save_params(params, path: str) -> None:
    """beastpipe MLP parameters (ModelParams-like: attributes W1..bv, version) -> TBST1."""
    write_tbst1(path, [(n, getattr(params, n)) for n in PARAM_FIELDS], getattr(params, "version", 0))


def load_params(path: str):
    """TBST1 MLP checkpoint -> ({W1..bv}, version), field order checked like restore()."""
    return read_tbst1(path, expected_fields=PARAM_FIELDS)


def checkpoint(model, path: str, version: int = 0) -> None:
    """AtariNet (or any nn.Module) -> TBST1 with its state_dict in the upstream torch layout
    (f32 arrays, state_dict order)."""
    sd = model.state_dict()
    write_tbst1(path, [(k, v.detach().float().cpu().numpy()) for k, v in sd.items()], version)


def restore(path: str, model=None, expected_num_actions: int | None = None):
    """TBST1 -> (state dict of numpy arrays, version); loads it into `model` if given
    (shape mismatches raise CheckpointError like the reference's config checks)."""
    import torch

    arrays, version = read_tbst1(path)
    if expected_num_actions is not None:
        pol = arrays.get("policy.weight")
        if pol is None or pol.shape[0] != expected_num_actions:
            got = None if pol is None else pol.shape[0]
            raise CheckpointError(f"policy.weight: checkpoint has num_actions {got}, "
                                  f"expected {expected_num_actions}")
    if model is not None:
        want = model.state_dict()
        if list(want.keys()) != list(arrays.keys()):
            raise CheckpointError(f"fields {list(arrays)} do not match the model's {list(want)}")
        for k, v in want.items():
            if tuple(v.shape) != arrays[k].shape:
                raise CheckpointError(f"{k}: shape {arrays[k].shape}, expected {tuple(v.shape)}")
        model.load_state_dict({k: torch.from_numpy(np.ascontiguousarray(a)) for k, a in arrays.items()})
    return arrays, version


# ---------------------------------------------------------------------------------- logs.csv
LOG_COLUMNS = ("step", "frames", "mean_episode_return", "pg_loss", "baseline_loss",
               "entropy_loss", "total_loss", "fps")  # pipeline.py:55-64


@dataclass
class MetricsRecord:
    step: int
    frames: int
    mean_episode_return: float
    pg_loss: float
    baseline_loss: float
    entropy_loss: float
    total_loss: float
    fps: float

    @classmethod
    def from_stats(cls, step: int, frames: int, stats: dict, fps: float) -> "MetricsRecord":
        """From the upstream learn() stats dict (learner.learn)."""
        return cls(step, frames, float(stats.get("mean_episode_return", float("nan"))),
                   float(stats["pg_loss"]), float(stats["baseline_loss"]),
                   float(stats["entropy_loss"]), float(stats["total_loss"]), float(fps))


class MetricsWriter:
    """Appends MetricsRecords to <logdir>/logs.csv in the reference's format (pipeline.py:191-229)."""

    def __init__(self, logdir: str | None):
        self._lock = threading.Lock()
        self.records: list[MetricsRecord] = []
        self._file = None
        self._csv = None
        if logdir is not None:
            os.makedirs(logdir, exist_ok=True)
            self._file = open(os.path.join(logdir, "logs.csv"), "w", newline="")
            self._csv = csv.writer(self._file)
            self._csv.writerow(LOG_COLUMNS)
            self._file.flush()

    def append(self, r: MetricsRecord) -> None:
        with self._lock:
            self.records.append(r)
            if self._csv is not None:
                self._csv.writerow([r.step, r.frames, f"{r.mean_episode_return:.6f}", f"{r.pg_loss:.6f}",
                                    f"{r.baseline_loss:.6f}", f"{r.entropy_loss:.6f}",
                                    f"{r.total_loss:.6f}", f"{r.fps:.2f}"])
                self._file.flush()

    def close(self) -> None:
        with self._lock:
            if self._file is not None:
                self._file.close()
                self._file = None
                self._csv = None
