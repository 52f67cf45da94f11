"""Binary frames (reference pkg/src/dvla/wire.py): kept for the host-side
planes and for interoperability with the reference's WIRE transport.

On B200 the weight plane never serialises parameters: snapshots travel as
raw device regions over NVLink with (version, count) carried out of band
(replicate.py).  This module reproduces the reference frame format byte for
byte for the message types that still cross a host boundary: weight
snapshots (wire.py:144-147, 161-163, 227-237), metadata (137-143, 211-224)
and acks (148-150).  Little-endian; header = magic "DVLA" | u16 version=1 |
u8 msg_type | u64 payload_len.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .core import ParamSnapshot, snapshot_from_params

MAGIC = b"DVLA"
FORMAT_VERSION = 1
HEADER_LEN = 15
MSG_TRAJECTORY_BATCH = 1
MSG_METADATA = 2
MSG_WEIGHT_SNAPSHOT = 3
MSG_ACK = 4
_MAX_REASONABLE_COUNT = 1 << 32


class DecodeError(ValueError):
    """Malformed frame; the message names the offending byte offset."""

    def __init__(self, offset: int, reason: str):
        super().__init__(f"{reason} at offset {offset}")
        self.offset = offset
        self.reason = reason


@dataclass(frozen=True)
class TrajectoryBatchMsg:
    policy_version: int
    groups: tuple


@dataclass(frozen=True)
class MetadataMsg:
    entries: tuple


@dataclass(frozen=True)
class AckMsg:
    epoch_id: int


def weight_frame_size(param_count: int) -> int:
    """Header + (version, count) + 4 bytes per parameter (wire.py:161-163)."""
    return HEADER_LEN + 16 + 4 * param_count


def _host_f32(params) -> np.ndarray:
    if type(params).__module__.startswith("torch"):
        params = params.detach().float().cpu().numpy()
    return np.ascontiguousarray(params, dtype="<f4").ravel()


def encode(msg) -> bytes:
    if isinstance(msg, ParamSnapshot):
        flat = _host_f32(msg.params)
        payload = struct.pack("<QQ", msg.version, flat.size) + flat.tobytes()
        mtype = MSG_WEIGHT_SNAPSHOT
    elif isinstance(msg, MetadataMsg):
        parts = [struct.pack("<I", len(msg.entries))]
        for key, val in msg.entries:
            kb = key.encode("utf-8")
            parts.append(struct.pack("<H", len(kb)) + kb + struct.pack("<I", len(val)) + bytes(val))
        payload = b"".join(parts)
        mtype = MSG_METADATA
    elif isinstance(msg, AckMsg):
        payload = struct.pack("<Q", msg.epoch_id)
        mtype = MSG_ACK
    elif isinstance(msg, TrajectoryBatchMsg):
        raise TypeError("trajectory frames stay device-resident on B200 (see planes.Channel)")
    else:
        raise TypeError(f"cannot encode {type(msg)!r}")
    return MAGIC + struct.pack("<HBQ", FORMAT_VERSION, mtype, len(payload)) + payload


def frame_size(msg) -> int:
    return len(encode(msg))


def _need(buf, pos, n, what):
    if pos + n > len(buf):
        raise DecodeError(pos, f"truncated {what}")


def decode(buf):
    buf = bytes(buf)
    _need(buf, 0, 4, "magic")
    if buf[:4] != MAGIC:
        raise DecodeError(0, "bad magic")
    _need(buf, 4, 2, "format_version")
    (ver,) = struct.unpack_from("<H", buf, 4)
    if ver != FORMAT_VERSION:
        raise DecodeError(4, f"unsupported format_version {ver}")
    _need(buf, 6, 1, "msg_type")
    mtype = buf[6]
    _need(buf, 7, 8, "payload_len")
    (plen,) = struct.unpack_from("<Q", buf, 7)
    if plen != len(buf) - HEADER_LEN:
        raise DecodeError(7, f"payload_len {plen} != actual {len(buf) - HEADER_LEN}")
    pos = HEADER_LEN
    if mtype == MSG_WEIGHT_SNAPSHOT:
        _need(buf, pos, 8, "version")
        (version,) = struct.unpack_from("<Q", buf, pos)
        pos += 8
        at = pos
        _need(buf, pos, 8, "param_count")
        (count,) = struct.unpack_from("<Q", buf, pos)
        pos += 8
        if count > _MAX_REASONABLE_COUNT:
            raise DecodeError(at, f"param_count {count} overflows the frame")
        _need(buf, pos, 4 * count, "parameter block")
        params = np.frombuffer(buf, dtype="<f4", count=count, offset=pos).copy()
        pos += 4 * count
        if not np.isfinite(params).all():
            bad = int(np.flatnonzero(~np.isfinite(params))[0])
            raise DecodeError(at + 8 + 4 * bad, "non-finite parameter")
        msg = snapshot_from_params(params, version)
    elif mtype == MSG_METADATA:
        _need(buf, pos, 4, "entry_count")
        (n,) = struct.unpack_from("<I", buf, pos)
        pos += 4
        entries = []
        for _ in range(n):
            _need(buf, pos, 2, "key_len")
            (kl,) = struct.unpack_from("<H", buf, pos)
            pos += 2
            _need(buf, pos, kl, "key bytes")
            kraw = buf[pos:pos + kl]
            try:
                key = kraw.decode("utf-8")
            except UnicodeDecodeError:
                raise DecodeError(pos, "key is not valid utf-8") from None
            pos += kl
            _need(buf, pos, 4, "val_len")
            (vl,) = struct.unpack_from("<I", buf, pos)
            pos += 4
            _need(buf, pos, vl, "value bytes")
            entries.append((key, buf[pos:pos + vl]))
            pos += vl
        msg = MetadataMsg(entries=tuple(entries))
    elif mtype == MSG_ACK:
        _need(buf, pos, 8, "epoch_id")
        msg = AckMsg(epoch_id=struct.unpack_from("<Q", buf, pos)[0])
        pos += 8
    elif mtype == MSG_TRAJECTORY_BATCH:
        raise DecodeError(6, "trajectory frames are not decoded on the B200 path")
    else:
        raise DecodeError(6, f"unknown msg_type {mtype}")
    if pos != len(buf):
        raise DecodeError(pos, f"{len(buf) - pos} trailing bytes")
    return msg


def messages_equal(a, b) -> bool:
    """Structural equality comparing parameter payloads bitwise."""
    if type(a) is not type(b):
        return False
    if isinstance(a, AckMsg):
        return a.epoch_id == b.epoch_id
    if isinstance(a, MetadataMsg):
        return a.entries == b.entries
    if isinstance(a, ParamSnapshot):
        return a.version == b.version and a.host_bytes() == b.host_bytes()
    raise TypeError(f"cannot compare {type(a)!r}")
