"""Rewrite committed version-1 map blobs (maps/**/*.pltmap) as version 2, which records the
input plane the map was trained on (the ray law's plane_z of its config).  Only the header
changes; weights, biases and normalisation are copied byte for byte.

    python tools/upgrade_maps.py
"""
import glob
import os
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from plt_inputs import configs as C  # noqa: E402

HDR = "<IIQII"


def config_of(path: str) -> str:
    rel = os.path.relpath(path, os.path.join(ROOT, "maps"))
    parts = rel.split(os.sep)
    return parts[1] if parts[0] == "flare" else os.path.basename(path)[:-7].rsplit("_", 1)[0]


def main():
    for path in sorted(glob.glob(os.path.join(ROOT, "maps", "**", "*.pltmap"), recursive=True)):
        blob = open(path, "rb").read()
        assert blob[:8] == b"PLTMAP01", path
        ver, direction, pid, ncl, nrl = struct.unpack_from(HDR, blob, 8)
        if ver != 1:
            continue
        plane = float(C.CONFIGS[config_of(path)]["law"]["plane_z"])
        off = 8 + struct.calcsize(HDR)
        new = blob[:8] + struct.pack(HDR, 2, direction, pid, ncl, nrl) + struct.pack("<d", plane) + blob[off:]
        with open(path, "wb") as f:
            f.write(new)
        print(os.path.relpath(path, ROOT), "-> v2, plane_z", plane)


if __name__ == "__main__":
    main()
