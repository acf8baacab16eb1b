"""Trained-artifact storage: ODM1 records + JSON-lines meta.

Same files, byte for byte, as the reference's store.py (dictionary: store.py:53-94;
SBO codes: store.py:99-133) and its record container (data.py:210-258).  Codes
held on the device (``DeviceCode``, from ``sbo.represent_device``) are streamed:
per record, signal chunks are packed into the column-major float64 payload on the
GPU (``sbo_codes_pack``), copied into pinned host buffers on a copy stream and
written while the next chunk is packed and copied — the host never materializes
the k x m matrices (2.4 GB at m = 2^24, s0 = 8).
"""
from __future__ import annotations

import itertools
import json
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _lib as L
from .sbo import SparseCode, UnionDictionary

ODM_MAGIC = b"ODM1"
ODM_HEADER = struct.Struct("<QQ")

DICT_FILE = "dict.odm"
DICT_META_FILE = "dict.meta.json"
CODES_FILE = "codes.odm"
CODES_META_FILE = "codes.meta.json"


class MatrixFormatError(ValueError):
    """Malformed ODM1 matrix container (data.py:33-34)."""


# ---------------------------------------------------------------- records
# An ODM1 record (data.py:210-258 defines the container): 4 magic bytes, the
# shape as two little-endian uint64, then the float64 payload in column-major
# order.  Files are plain concatenations of records.
_SHAPE = np.dtype("<u8")
_PREFIX = len(ODM_MAGIC) + ODM_HEADER.size


def _frame(rows: int, cols: int) -> bytes:
    """The fixed-size part of a record of the given shape."""
    return ODM_MAGIC + np.array([rows, cols], dtype=_SHAPE).tobytes()


def _encode(a) -> bytes:
    m = np.asarray(a, dtype=np.float64)
    if m.ndim != 2:
        raise ValueError(f"ODM1 stores 2-D matrices, got shape {m.shape}")
    return _frame(*m.shape) + np.asfortranarray(m).astype("<f8", copy=False).tobytes(order="F")


def write_record(f, a: np.ndarray) -> int:
    """Append one record to a binary stream; returns its size in bytes (data.py:228-237)."""
    blob = _encode(a)
    f.write(blob)
    return len(blob)


def read_record(buf: bytes, pos: int) -> tuple[np.ndarray, int]:
    """Decode the record starting at byte ``pos`` of ``buf``; returns (matrix, end
    offset).  Malformed input raises MatrixFormatError (data.py:240-258)."""
    view = memoryview(buf)
    magic = bytes(view[pos:pos + len(ODM_MAGIC)])
    if magic != ODM_MAGIC:
        raise MatrixFormatError(f"bad magic {magic!r} at offset {pos}, expected {ODM_MAGIC!r}")
    body = pos + len(ODM_MAGIC)
    if len(view) - body < ODM_HEADER.size:
        raise MatrixFormatError(f"truncated header at offset {body}")
    rows, cols = (int(v) for v in np.frombuffer(view, dtype=_SHAPE, count=2, offset=body))
    start = pos + _PREFIX
    nbytes = 8 * rows * cols
    if len(view) - start < nbytes:
        raise MatrixFormatError(
            f"truncated payload: expected {nbytes} bytes, got {len(view) - start}")
    flat = np.frombuffer(view, dtype="<f8", count=rows * cols, offset=start)
    return np.array(flat.reshape((cols, rows)).T, order="F"), start + nbytes


def _scan(path: Path):
    """Every record of a file, in order."""
    buf = path.read_bytes()
    pos = 0
    while pos < len(buf):
        a, pos = read_record(buf, pos)
        yield a


def _save_records(path: Path, matrices) -> list[int]:
    """Write the matrices as consecutive records; returns each record's offset."""
    blobs = [_encode(a) for a in matrices]
    path.write_bytes(b"".join(blobs))
    return list(itertools.accumulate((len(b) for b in blobs[:-1]), initial=0)) if blobs else []


def _meta_text(header: dict, offsets: list[int], label: str) -> str:
    """JSON-lines meta: the header, then one {label: i, "offset": o} line per record."""
    rows = [header] + [{label: i, "offset": o} for i, o in enumerate(offsets)]
    return "".join(json.dumps(r, sort_keys=True) + "\n" for r in rows)


def _load_meta(path: Path) -> tuple[dict, list[dict]]:
    parsed = [json.loads(t) for t in path.read_text().splitlines() if t.strip()]
    if not parsed:
        raise MatrixFormatError(f"empty meta file {path}")
    return parsed[0], parsed[1:]


# ------------------------------------------------------------- dictionary
def save_dictionary(out_dir, dictionary, extra_meta: dict | None = None) -> None:
    """Write ``dictionary`` (a union of blocks or one dense atom matrix) and its
    meta file; the files the reference's store.py:53-69 writes."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    union = isinstance(dictionary, UnionDictionary)
    mats = list(dictionary.blocks) if union else [np.asarray(dictionary, dtype=np.float64)]
    header = ({"format": "union-onb", "p": dictionary.p, "blocks": dictionary.num_blocks}
              if union else {"format": "dense", "p": mats[0].shape[0], "atoms": mats[0].shape[1]})
    header.update(extra_meta or {})
    offsets = _save_records(out / DICT_FILE, mats)
    (out / DICT_META_FILE).write_text(_meta_text(header, offsets, "block"))


def load_dictionary(out_dir):
    """Read what save_dictionary wrote: (dictionary, header) (store.py:72-96)."""
    out = Path(out_dir)
    header, entries = _load_meta(out / DICT_META_FILE)
    mats = list(_scan(out / DICT_FILE))
    if entries and len(entries) != len(mats):
        raise MatrixFormatError(f"meta lists {len(entries)} records, file holds {len(mats)}")
    kind = header["format"]
    if kind == "union-onb":
        if len(mats) != header["blocks"]:
            raise MatrixFormatError(
                f"dictionary holds {len(mats)} blocks, meta says {header['blocks']}")
        return UnionDictionary(mats), header
    if kind == "dense":
        if len(mats) != 1:
            raise MatrixFormatError("dense dictionary file must hold one record")
        return mats[0], header
    raise MatrixFormatError(f"unknown dictionary format {kind!r}")


# ------------------------------------------------------------------ codes
@dataclass
class DeviceCode:
    """A SparseCode resident on the device (sbo.represent_device): block int32 (m,),
    indices int16 and values float64 as k rows of stride ld, energy and
    residual_sq float64 (m,)."""

    block: torch.Tensor
    indices: torch.Tensor
    values: torch.Tensor
    energy: torch.Tensor
    residual_sq: torch.Tensor

    @property
    def m(self) -> int:
        return int(self.block.shape[0])

    @property
    def k(self) -> int:
        return int(self.indices.shape[0])

    def to_host(self) -> SparseCode:
        m = self.m
        return SparseCode(self.block.cpu().numpy().astype(np.int64),
                          self.indices[:, :m].cpu().numpy().astype(np.int64),
                          self.values[:, :m].cpu().numpy(), self.energy.cpu().numpy(),
                          self.residual_sq.cpu().numpy())


def _codes_header(m: int, k: int) -> dict:
    return {"format": "sbo-codes", "signals": m, "nnz_per_signal": k}


def save_sbo_codes(out_dir, code, chunk: int = 1 << 20) -> None:
    """store.py:99-115.  ``code`` is a host SparseCode or a DeviceCode (streamed)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    if isinstance(code, DeviceCode):
        offsets = _stream_device_codes(out / CODES_FILE, code, chunk)
        header = _codes_header(code.m, code.k)
    else:
        rows = (code.block[None, :], code.indices, code.values, code.energy[None, :],
                code.residual_sq[None, :])
        offsets = _save_records(out / CODES_FILE, [np.asarray(r, np.float64) for r in rows])
        header = _codes_header(int(code.block.shape[0]), int(code.indices.shape[0]))
    (out / CODES_META_FILE).write_text(_meta_text(header, offsets, "record"))


def load_sbo_codes(out_dir) -> SparseCode:
    """store.py:118-133."""
    out = Path(out_dir)
    header, _ = _load_meta(out / CODES_META_FILE)
    if header.get("format") != "sbo-codes":
        raise MatrixFormatError(f"not an sbo codes file: {header!r}")
    block, indices, values, energy, residual_sq = _scan(out / CODES_FILE)
    return SparseCode(block=block.ravel().astype(np.int64), indices=indices.astype(np.int64),
                      values=values, energy=energy.ravel(), residual_sq=residual_sq.ravel())


def _stream_device_codes(path: Path, code: DeviceCode, chunk: int) -> list[int]:
    """The five records of save_sbo_codes from device arrays, chunk by chunk: pack
    (compute stream) -> pinned host buffer (copy stream) -> file, double-buffered."""
    dev = code.block.device
    m, k = code.m, code.k
    ld = int(code.indices.stride(0))
    width = max(k, 1)
    chunk = max(1, min(chunk, m))
    stage = [torch.empty(chunk * width, dtype=torch.float64, device=dev) for _ in range(2)]
    host = [torch.empty(chunk * width, dtype=torch.float64).pin_memory() for _ in range(2)]
    packed = [torch.cuda.Event() for _ in range(2)]
    landed = [torch.cuda.Event() for _ in range(2)]
    copier = torch.cuda.Stream(dev)
    compute = torch.cuda.current_stream(dev)
    st = compute.cuda_stream
    shapes = [(1, m), (k, m), (k, m), (1, m), (1, m)]
    offsets, pos = [], 0
    with open(path, "wb") as f:
        for rec, (rows, cols) in enumerate(shapes):
            offsets.append(pos)
            f.write(_frame(rows, cols))
            pos += _PREFIX + 8 * rows * cols
            per = rows  # float64 values per signal in this record
            spans = [(j0, min(chunk, m - j0)) for j0 in range(0, m, chunk)]

            def issue(i):
                j0, n = spans[i]
                b = i % 2
                if rec in (0, 1, 2):
                    L.call("sbo_codes_pack", rec, code.block.data_ptr(), code.indices.data_ptr(),
                           code.values.data_ptr(), ld, k, j0, n, stage[b].data_ptr(), st)
                    src = stage[b][: n * per]
                else:
                    src = (code.energy if rec == 3 else code.residual_sq)[j0: j0 + n]
                packed[b].record(compute)
                with torch.cuda.stream(copier):
                    copier.wait_event(packed[b])
                    host[b][: n * per].copy_(src, non_blocking=True)
                    landed[b].record(copier)

            if spans:
                issue(0)
            for i, (j0, n) in enumerate(spans):
                if i + 1 < len(spans):
                    # buffer (i+1)%2 was written to the file in step i-1 (synchronous)
                    issue(i + 1)
                landed[i % 2].synchronize()
                f.write(memoryview(host[i % 2].numpy()[: n * per]).cast("B"))
            # the next record's issue(0) reuses buffer 0: the file write above that
            # read it has completed (f.write is synchronous)
    return offsets
