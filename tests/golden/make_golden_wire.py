"""Golden header bytes from the reference wire codec
(/root/reference/pkg/src/hrt/wire.py).  Usage (repo root):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_wire.py

Writes tests/golden/wire.json: seeded headers (fields + reference encoding,
hex) and malformed buffers with the reference's decode verdict."""

import json
import os
import random

from hrt.errors import ProtocolError
from hrt.wire import HEADER_SIZE, MessageHeader, MsgKind, decode_header, should_inline

HERE = os.path.dirname(os.path.abspath(__file__))
rnd = random.Random(20230302)
headers = []
for _ in range(300):
    f = dict(msg_kind=rnd.choice(list(MsgKind)).value, handler_id=rnd.randrange(1 << 32),
             target_rank=rnd.randrange(1 << 32), target_index=rnd.randrange(1 << 64),
             payload_size=rnd.randrange(1 << 64), inline_flag=rnd.random() < 0.5,
             correlation_id=rnd.randrange(1 << 64), element_size=rnd.randrange(1 << 32),
             dims=[rnd.randrange(1 << 32) for _ in range(3)],
             source_device_type=rnd.choice([0, 1, 0xFF]))
    h = MessageHeader(MsgKind(f["msg_kind"]), f["handler_id"], f["target_rank"], f["target_index"],
                      f["payload_size"], f["inline_flag"], f["correlation_id"], f["element_size"],
                      tuple(f["dims"]), f["source_device_type"])
    headers.append(dict(fields=f, hex=h.encode().hex()))
bad = []
base = MessageHeader(MsgKind.HANDLER, 1, 2, 3, 4).encode()
cases = {"truncated": base[:63], "magic": b"XRTM" + base[4:], "version": base[:4] + b"\x02" + base[5:],
         "kind0": base[:5] + b"\x00" + base[6:], "kind9": base[:5] + b"\x09" + base[6:],
         "inline2": base[:6] + b"\x02" + base[7:], "reserved": base[:63] + b"\x01",
         "ok_with_tail": base + b"payload"}
for name, buf in cases.items():
    try:
        decode_header(buf)
        verdict = "ok"
    except ProtocolError:
        verdict = "ProtocolError"
    bad.append(dict(name=name, hex=buf.hex(), verdict=verdict))
inline = [dict(n=n, inline=should_inline(n)) for n in (0, 447, 448, 449, 1 << 20)]
json.dump(dict(header_size=HEADER_SIZE, headers=headers, malformed=bad, inline=inline),
          open(os.path.join(HERE, "wire.json"), "w"))
print(len(headers), "headers;", [b["verdict"] for b in bad])
