"""Planes and wire frames (host logic, CPU): the reference's plane and wire
contracts (reference tests/test_planes.py, tests/test_wire.py) on the B200
package, plus the weight frame pinned byte-for-byte to the reference's."""

import struct
import threading

import numpy as np
import pytest

from conftest import golden
from paper_2605_13276_b200 import wire
from paper_2605_13276_b200.core import ConfigError, Rng, UsageError, snapshot_from_params
from paper_2605_13276_b200.planes import (Channel, ChannelClosed, ControlPlane, LinkProfile,
                                           Plane, RunAborted, Transport, TransportMode,
                                           WeightMailbox)


def _snap(version=1, n=20):
    return snapshot_from_params(Rng(7).gaussian(n).astype(np.float32), version)


def test_weight_frame_bytes_match_reference():
    g = golden("wire")
    snap = snapshot_from_params(g["params"], int(g["version"]))
    assert wire.encode(snap) == g["frame"].tobytes()
    assert wire.encode(wire.MetadataMsg(entries=())) == g["meta"].tobytes()
    assert wire.encode(wire.AckMsg(epoch_id=77)) == g["ack"].tobytes()
    back = wire.decode(g["frame"].tobytes())
    assert wire.messages_equal(back, snap)


def test_weight_frame_size_formula():
    assert len(wire.encode(_snap(n=123))) == wire.weight_frame_size(123)
    assert wire.weight_frame_size(0) == wire.HEADER_LEN + 16


def test_decode_errors_name_offsets():
    buf = bytearray(wire.encode(_snap(n=5)))
    with pytest.raises(wire.DecodeError, match="bad magic") as e:
        wire.decode(b"XXXX" + bytes(buf[4:]))
    assert e.value.offset == 0
    with pytest.raises(wire.DecodeError, match="trailing|payload_len"):
        wire.decode(bytes(buf) + b"\x00")
    bad = bytearray(buf)
    struct.pack_into("<f", bad, 15 + 8 + 8 + 4 * 3, float("nan"))
    with pytest.raises(wire.DecodeError, match="non-finite parameter") as e:
        wire.decode(bytes(bad))
    assert e.value.offset == 15 + 8 + 8 + 4 * 3
    with pytest.raises(wire.DecodeError, match="truncated"):
        wire.decode(bytes(buf[:10]))


def test_plane_isolation():
    from paper_2605_13276_b200.grpo import GroupBatch
    gb = GroupBatch(group_id=0, horizon=4, chunk=4, obs=np.zeros((2, 1, 3)),
                    actions=np.zeros((2, 1, 8)), behavior_log_prob=np.zeros((2, 1)),
                    rewards=np.zeros(2), behavior_version=0)
    with pytest.raises(UsageError, match="not allowed on the data plane"):
        Transport(TransportMode.INPROC, Plane.DATA).outbound(_snap())
    with pytest.raises(UsageError, match="not allowed on the control plane"):
        Transport(TransportMode.INPROC, Plane.CONTROL).outbound(gb)
    with pytest.raises(UsageError, match="not a plane message"):
        Transport(TransportMode.INPROC, Plane.DATA).outbound(object())
    with pytest.raises(UsageError, match="control transport"):
        ControlPlane(Transport(TransportMode.INPROC, Plane.DATA))


def test_inproc_is_zero_copy_and_wire_counts_two_copies():
    t = Transport(TransportMode.INPROC, Plane.CONTROL)
    s = _snap()
    p, n, d = t.outbound(s)
    assert p is s and n == 0 and d == 0.0 and t.inbound(p) is s
    assert t.copy_counter == 0 and t.bytes_counter == 0
    w = Transport(TransportMode.WIRE, Plane.CONTROL)
    p, n, _ = w.outbound(s)
    back = w.inbound(p)
    assert wire.messages_equal(back, s) and w.copy_counter == 2 and w.bytes_counter == n


def test_link_profile():
    assert LinkProfile(100.0, 100e6).delay_s(1 << 20) == pytest.approx(100e-6 + (1 << 20) / 100e6)
    with pytest.raises(ConfigError, match="latency_us"):
        LinkProfile(latency_us=-1.0).validate()


def test_channel_fifo_backpressure_close_abort():
    ch = Channel(2, Transport(TransportMode.INPROC, Plane.DATA))
    ch.put(wire.AckMsg(0))
    ch.put(wire.AckMsg(1))
    with pytest.raises(TimeoutError, match="put timed out"):
        ch.put(wire.AckMsg(2), timeout=0.05)
    assert [ch.take().epoch_id for _ in range(2)] == [0, 1]
    with pytest.raises(TimeoutError, match="take timed out"):
        ch.take(timeout=0.05)
    ch.close()
    with pytest.raises(ChannelClosed):
        ch.put(wire.AckMsg(3))
    ab = threading.Event()
    ab.set()
    with pytest.raises(RunAborted):
        Channel(1, Transport(TransportMode.INPROC, Plane.DATA), abort_event=ab).take()


def test_mailbox_latest_wins_and_monotone():
    box = WeightMailbox(Transport(TransportMode.INPROC, Plane.CONTROL))
    box.deliver(_snap(1), 1)
    box.deliver(_snap(3), 3)
    box.deliver(_snap(2), 2)
    assert box.take_newest().version == 3
    box.deliver(_snap(2), 2)
    assert box.take_newest(timeout=0.05) is None


def test_broadcast_bytes_per_subscriber_and_regression_guard():
    t = Transport(TransportMode.WIRE, Plane.CONTROL)
    plane = ControlPlane(t)
    boxes = [plane.subscribe(name=f"s{i}") for i in range(4)]
    s = _snap(1, n=25)
    plane.broadcast(s)
    assert t.bytes_counter == 4 * wire.weight_frame_size(25) and t.copy_counter == 4
    assert all(b.take_newest().version == 1 for b in boxes)
    with pytest.raises(UsageError, match="version regression"):
        plane.broadcast(_snap(1))
    with pytest.raises(UsageError, match="ParamSnapshot only"):
        plane.broadcast(wire.AckMsg(0))
