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
def write_record(f, a: np.ndarray) -> int:
    """data.py:228-237 — append one ODM1 record; returns the bytes written."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"ODM1 stores 2-D matrices, got shape {a.shape}")
    payload = a.tobytes(order="F")
    f.write(ODM_MAGIC)
    f.write(ODM_HEADER.pack(a.shape[0], a.shape[1]))
    f.write(payload)
    return len(ODM_MAGIC) + ODM_HEADER.size + len(payload)


def read_record(buf: bytes, pos: int) -> tuple[np.ndarray, int]:
    """data.py:240-258 — one ODM1 record at ``pos``; returns (matrix, next pos)."""
    if buf[pos: pos + 4] != ODM_MAGIC:
        raise MatrixFormatError(
            f"bad magic {buf[pos:pos + 4]!r} at offset {pos}, expected {ODM_MAGIC!r}")
    pos += 4
    if len(buf) - pos < ODM_HEADER.size:
        raise MatrixFormatError(f"truncated header at offset {pos}")
    rows, cols = ODM_HEADER.unpack_from(buf, pos)
    pos += ODM_HEADER.size
    need = rows * cols * 8
    have = len(buf) - pos
    if have < need:
        raise MatrixFormatError(f"truncated payload: expected {need} bytes, got {have}")
    a = np.frombuffer(buf, dtype="<f8", count=rows * cols, offset=pos)
    return a.reshape(rows, cols, order="F").copy(order="F"), pos + need


def _write_records(path: Path, matrices) -> list[int]:
    offsets, pos = [], 0
    with open(path, "wb") as f:
        for a in matrices:
            offsets.append(pos)
            pos += write_record(f, a)
    return offsets


def _write_meta(path: Path, header: dict, offsets: list[int], label: str) -> None:
    lines = [json.dumps(header, sort_keys=True)]
    lines += [json.dumps({label: i, "offset": off}, sort_keys=True) for i, off in enumerate(offsets)]
    path.write_text("\n".join(lines) + "\n")


def _read_meta(path: Path) -> tuple[dict, list[dict]]:
    lines = [ln for ln in path.read_text().splitlines() if ln.strip()]
    if not lines:
        raise MatrixFormatError(f"empty meta file {path}")
    return json.loads(lines[0]), [json.loads(ln) for ln in lines[1:]]


def _read_all(path: Path) -> list[np.ndarray]:
    buf = path.read_bytes()
    out, pos = [], 0
    while pos < len(buf):
        a, pos = read_record(buf, pos)
        out.append(a)
    return out


# ------------------------------------------------------------- dictionary
def save_dictionary(out_dir, dictionary, extra_meta: dict | None = None) -> None:
    """store.py:53-69 — a union of blocks, or a dense atom dictionary."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    if isinstance(dictionary, UnionDictionary):
        offsets = _write_records(out / DICT_FILE, dictionary.blocks)
        header = {"format": "union-onb", "p": dictionary.p, "blocks": dictionary.num_blocks}
    else:
        d = np.asarray(dictionary, dtype=np.float64)
        offsets = _write_records(out / DICT_FILE, [d])
        header = {"format": "dense", "p": d.shape[0], "atoms": d.shape[1]}
    header.update(extra_meta or {})
    _write_meta(out / DICT_META_FILE, header, offsets, "block")


def load_dictionary(out_dir):
    """store.py:72-96 — (dictionary, header)."""
    out = Path(out_dir)
    header, entries = _read_meta(out / DICT_META_FILE)
    matrices = _read_all(out / DICT_FILE)
    if len(entries) not in (0, len(matrices)):
        raise MatrixFormatError(f"meta lists {len(entries)} records, file holds {len(matrices)}")
    if header["format"] == "union-onb":
        if len(matrices) != header["blocks"]:
            raise MatrixFormatError(
                f"dictionary holds {len(matrices)} blocks, meta says {header['blocks']}")
        return UnionDictionary(matrices), header
    if header["format"] == "dense":
        if len(matrices) != 1:
            raise MatrixFormatError("dense dictionary file must hold one record")
        return matrices[0], header
    raise MatrixFormatError(f"unknown dictionary format {header['format']!r}")


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
        _write_meta(out / CODES_META_FILE, _codes_header(code.m, code.k), offsets, "record")
        return
    records = [code.block[None, :].astype(np.float64), code.indices.astype(np.float64),
               code.values, code.energy[None, :], code.residual_sq[None, :]]
    offsets = _write_records(out / CODES_FILE, records)
    _write_meta(out / CODES_META_FILE,
                _codes_header(int(code.block.shape[0]), int(code.indices.shape[0])), offsets,
                "record")


def load_sbo_codes(out_dir) -> SparseCode:
    """store.py:118-133."""
    out = Path(out_dir)
    header, _ = _read_meta(out / CODES_META_FILE)
    if header.get("format") != "sbo-codes":
        raise MatrixFormatError(f"not an sbo codes file: {header!r}")
    block, indices, values, energy, residual_sq = _read_all(out / CODES_FILE)
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
            f.write(ODM_MAGIC)
            f.write(ODM_HEADER.pack(rows, cols))
            pos += len(ODM_MAGIC) + ODM_HEADER.size + 8 * rows * cols
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
