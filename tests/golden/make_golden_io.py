"""Generate tests/golden/golden_io.json from the REFERENCE frame codecs.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_io.py

Each case is an in-memory PPM / PGM file (valid or malformed, built by
``io_cases()``, which the tests import); the reference's read_ppm /
read_mask_pgm outcome is recorded: the decoded array's shape and sha256, or
the FormatError's message and byte offset.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)


def io_cases():
    """(kind, bytes): kind 'ppm' or 'pgm'."""
    rng = np.random.default_rng(31)
    px = rng.integers(0, 256, size=(3, 4, 3), dtype=np.uint8).tobytes()     # 4 x 3 frame
    m = np.where(rng.random(12) < 0.5, 255, 0).astype(np.uint8).tobytes()  # 4 x 3 mask
    c = []
    ppm = lambda head: ("ppm", head + px)  # noqa: E731
    c += [ppm(b"P6\n4 3\n255\n"), ppm(b"P6 4 3 255 "), ppm(b"P6\t4\t3\t255\t"), ppm(b"P6\r\n4 3\r\n255\r"),
          ppm(b"P6\x0b4\x0c3\n255\n"), ppm(b"P6\n# comment\n4 3\n# more # text\n255\n"),
          ppm(b"P6#x\n4#y\n3#z\n255\n"), ppm(b"P6\n004 0003\n0255\n"), ppm(b"P6\n4 3\n255\n\n"[:-1]),
          ppm(b"P6\n4 3\n255 "), ("ppm", b"P6\n4 3\n255\n" + px[:-1]), ("ppm", b"P6\n4 3\n255\n" + px + b"\n"),
          ("ppm", b"P6\n4 3\n255\n"), ("ppm", b"P6\n4 3\n255"), ("ppm", b"P6\n4 3\n255#c\n" + px),
          ("ppm", b"P3\n4 3\n255\n" + px), ("ppm", b"P5\n4 3\n255\n" + px), ("ppm", b"P66\n4 3\n255\n" + px),
          ("ppm", b"\x00P6\n4 3\n255\n" + px), ("ppm", b"P'6 4 3 255\n" + px), ("ppm", b'P"6 4 3 255\n' + px),
          ("ppm", b"p6 4 3 255\n" + px), ("ppm", b"P6\n4x 3\n255\n" + px), ("ppm", b"P6\n4 -3\n255\n" + px),
          ("ppm", b"P6\n4 3.0\n255\n" + px), ("ppm", b"P6\n0 3\n255\n"), ("ppm", b"P6\n4 000\n255\n"),
          ("ppm", b"P6\n4 3\n65535\n" + px), ("ppm", b"P6\n4 3\n00\n" + px), ("ppm", b"P6\n4 3\nabc\n" + px),
          ("ppm", b"P6\n99999999999 1\n255\n" + px), ("ppm", b""), ("ppm", b"   \n\t"), ("ppm", b"# only"),
          ("ppm", b"P6"), ("ppm", b"P6\n4"), ("ppm", b"P6\n4 3"), ("ppm", b"P6\n4 3\n"),
          ("ppm", b"P6\n4 3\n255\xff" + px), ("ppm", b"P6\n\xe9 3\n255\n" + px)]
    pgm = lambda head, body=m: ("pgm", head + body)  # noqa: E731
    c += [pgm(b"P5\n4 3\n255\n"), pgm(b"P5 4 3 255 "), pgm(b"P5\n4 3\n255\n", m[:5] + b"\x80" + m[6:]),
          pgm(b"P5\n4 3\n255\n", b"\x01" + m[1:]), pgm(b"P5\n4 3\n255\n", m[:-1]), pgm(b"P5\n4 3\n255\n", m + b"x"),
          pgm(b"P6\n4 3\n255\n"), pgm(b"P5\n4 3\n1\n"), pgm(b"P5\n# c\n4 3 255\n"),
          pgm(b"P5\n4 3\n255\n", bytes(12)), pgm(b"P5\n4 3\n255\n", b"\xff" * 12)]
    return c


def main():
    from make_golden import ref
    out = []
    for kind, data in io_cases():
        fn = ref.read_ppm if kind == "ppm" else ref.read_mask_pgm
        try:
            a = fn(data)
            out.append({"kind": kind, "ok": True, "shape": list(a.shape),
                        "sha": hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()})
        except ref.FormatError as e:
            out.append({"kind": kind, "ok": False, "type": "FormatError", "msg": str(e), "offset": e.offset})
        except ValueError as e:
            out.append({"kind": kind, "ok": False, "type": "ValueError", "msg": str(e), "offset": None})
    path = os.path.join(HERE, "golden_io.json")
    with open(path, "w") as f:
        json.dump({"generator": "tests/golden/make_golden_io.py", "cases": out}, f, indent=0)
    print(f"wrote {path}: {sum(c['ok'] for c in out)} ok / {len(out)}")


if __name__ == "__main__":
    main()
