"""Wire codec parity with the reference (golden bytes from
/root/reference/pkg/src/hrt/wire.py via tests/golden/make_golden_wire.py)
and the device-locator data frame.  CPU only."""

import pytest

from conftest import load_golden

from paper_2303_02543_b200.errors import ProtocolError
from paper_2303_02543_b200.wire import (HEADER_SIZE, DeviceLocator, MessageHeader, MsgKind,
                                        decode_header, should_inline)


def test_encode_matches_reference_bytes():
    g = load_golden("wire.json")
    assert g["header_size"] == HEADER_SIZE == 64
    for h in g["headers"]:
        f = h["fields"]
        ours = MessageHeader(MsgKind(f["msg_kind"]), f["handler_id"], f["target_rank"],
                             f["target_index"], f["payload_size"], f["inline_flag"],
                             f["correlation_id"], f["element_size"], tuple(f["dims"]),
                             f["source_device_type"])
        assert ours.encode().hex() == h["hex"]
        back = decode_header(bytes.fromhex(h["hex"]))
        assert back.encode() == ours.encode()


def test_malformed_verdicts_match_reference():
    for b in load_golden("wire.json")["malformed"]:
        buf = bytes.fromhex(b["hex"])
        if b["verdict"] == "ok":
            decode_header(buf)
        else:
            with pytest.raises(ProtocolError):
                decode_header(buf)


def test_inline_rule():
    for c in load_golden("wire.json")["inline"]:
        assert should_inline(c["n"]) == c["inline"]


def test_device_locator_roundtrip():
    loc = DeviceLocator(bytes(range(64)), 123456, 1 << 28, 3, 0x7F0000000000)
    back = DeviceLocator.decode(loc.encode())
    assert back == loc
    with pytest.raises(ProtocolError):
        DeviceLocator.decode(b"XXXX" + loc.encode()[4:])
