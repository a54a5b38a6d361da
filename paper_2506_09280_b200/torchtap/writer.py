"""TTRC serialisation of captured records (byte-identical to the
reference writer, pkg/adapter/src/torchtap/writer.py:65-105).

Captures stay in HBM in their own dtype; the f32 little-endian bytes the
file format requires are produced only here, at flush time.
"""

from __future__ import annotations

import json
import struct
from dataclasses import dataclass

import numpy as np

from .errors import WriteError

MAGIC = b"TTRC"
END_MAGIC = b"CRTT"
VERSION = 1


def canonical_json(obj) -> bytes:
    return json.dumps(obj, sort_keys=True, separators=(",", ":")).encode("utf-8")


def encode_id(iteration: int, microbatch: int, kind: str, module: str) -> str:
    return f"iter={iteration}|mb={microbatch}|kind={kind}|mod={module}"


@dataclass(frozen=True)
class FlatRecord:
    """One captured tensor: canonical id, payload (a detached tensor, usually
    on the GPU), module class.  Optional shard annotation for tensor-parallel
    captures: mapping (ShardMapping), rank (6-tuple), replica size."""

    ident: str
    payload: object
    module_class: str
    mapping: object = None
    rank: tuple = (0, 0, 0, 0, 0, 0)
    replica: int = 1

    def host(self) -> np.ndarray:
        """float32 host copy of the payload (the file's carrier dtype)."""
        import torch
        p = self.payload
        if isinstance(p, torch.Tensor):
            return p.detach().to("cpu", torch.float32).contiguous().numpy()
        return np.ascontiguousarray(p, dtype=np.float32)


def _box(bounds) -> bytes:
    return struct.pack(f"<{2 * len(bounds)}Q", *[v for ab in bounds for v in ab])


def _record_bytes(rec: FlatRecord) -> bytes:
    ident = rec.ident.encode("utf-8")
    cls = rec.module_class.encode("utf-8")
    payload = rec.host()
    shape = payload.shape
    if rec.mapping is None:
        whole = tuple((0, n) for n in shape)
        pairs = [(whole, whole)]
    else:
        pairs = [(loc.bounds, glob.bounds) for loc, glob in rec.mapping.pairs]
    parts = [struct.pack("<BI", 1, len(ident)), ident,
             struct.pack("<7H", *rec.rank, rec.replica),
             struct.pack("<I", len(cls)), cls,
             struct.pack(f"<BB{len(shape)}Q", 0, len(shape), *shape),
             struct.pack("<H", len(pairs))]
    for loc, glob in pairs:
        parts.append(_box(glob))
        parts.append(_box(loc))
    data = payload.astype("<f4", copy=False).tobytes()
    parts.append(struct.pack("<Q", len(data)))
    parts.append(data)
    return b"".join(parts)


def serialize(header: dict, records: list) -> bytes:
    try:
        head = canonical_json(header)
    except (TypeError, ValueError) as exc:
        raise WriteError(f"header is not JSON-serializable: {exc}") from None
    out = [MAGIC, struct.pack("<HHI", VERSION, 0, len(head)), head]
    out.extend(_record_bytes(r) for r in records)
    out.append(END_MAGIC)
    return b"".join(out)


def write(header: dict, records: list, path) -> None:
    data = serialize(header, records)
    try:
        with open(path, "wb") as fh:
            fh.write(data)
    except OSError as exc:
        raise WriteError(f"cannot write trace to {path}: {exc}") from None
