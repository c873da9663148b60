"""CPU restatement of the reference's frame / mesh I/O (TEST INFRASTRUCTURE).

Only tests/ may import this.  It restates, in plain Python over zlib:

  * the PNG format (ISO/IEC 15948: chunks, CRC, zlib stream, the five row
    filters, bit depths 1-16, colour types 0/2/3/4/6) — the reference links
    libpng (image_io.cpp:1-122), which is absent here; its read transforms
    (png_set_expand, png_set_strip_16, png_set_strip_alpha,
    png_set_gray_to_rgb; image_io.cpp:88-92) are restated from the libpng
    documentation: expansion scales a k-bit gray sample by 255/(2^k-1),
    strip_16 keeps the high byte;
  * mesh_io.cpp:104-145 write_ply and :147-218 read_ply byte for byte;
  * TexturedMesh::with_channels (texture.cpp:74-91).
"""
from __future__ import annotations

import struct
import zlib

import numpy as np

SIG = bytes([137, 80, 78, 71, 13, 10, 26, 10])
CHANNELS = {0: 1, 2: 3, 3: 1, 4: 2, 6: 4}


def _chunk(tag: bytes, data: bytes) -> bytes:
    return struct.pack(">I", len(data)) + tag + data + struct.pack(">I", zlib.crc32(tag + data) & 0xffffffff)


def _paeth(a, b, c):
    p = a + b - c
    pa, pb, pc = abs(p - a), abs(p - b), abs(p - c)
    return a if (pa <= pb and pa <= pc) else (b if pb <= pc else c)


def pack_samples(samples: np.ndarray, depth: int) -> bytes:
    """One row of integer samples -> packed big-endian bytes."""
    s = [int(v) for v in samples.ravel()]
    if depth == 16:
        return b"".join(struct.pack(">H", v) for v in s)
    if depth == 8:
        return bytes(s)
    per = 8 // depth
    out = bytearray((len(s) + per - 1) // per)
    for i, v in enumerate(s):
        out[i // per] |= v << (8 - depth * (1 + i % per))
    return bytes(out)


def encode_png(rows: list[bytes], width: int, height: int, depth: int, ctype: int, filters=None,
               palette: bytes | None = None, idat_split: int = 0) -> bytes:
    """rows: packed scanlines; filters: per-row filter type (0-4); idat_split: bytes per IDAT chunk."""
    bpp = max(1, CHANNELS[ctype] * depth // 8)
    raw = bytearray()
    prev = bytes(len(rows[0]))
    for y, row in enumerate(rows):
        f = 0 if filters is None else filters[y]
        out = bytearray(len(row))
        for i in range(len(row)):
            a = row[i - bpp] if i >= bpp else 0
            b = prev[i]
            c = prev[i - bpp] if i >= bpp else 0
            pred = [0, a, b, (a + b) >> 1, _paeth(a, b, c)][f]
            out[i] = (row[i] - pred) & 255
        raw += bytes([f]) + out
        prev = row
    z = zlib.compress(bytes(raw), 9)
    png = SIG + _chunk(b"IHDR", struct.pack(">IIBBBBB", width, height, depth, ctype, 0, 0, 0))
    if palette is not None:
        png += _chunk(b"PLTE", palette)
    step = idat_split or len(z)
    for i in range(0, len(z), step):
        png += _chunk(b"IDAT", z[i:i + step])
    return png + _chunk(b"IEND", b"")


def decode_png(data: bytes):
    """-> (header dict, list of unfiltered packed rows)."""
    assert data[:8] == SIG
    o, idat, hdr, plte = 8, b"", None, None
    while o < len(data):
        n = struct.unpack(">I", data[o:o + 4])[0]
        tag, body = data[o + 4:o + 8], data[o + 8:o + 8 + n]
        assert struct.unpack(">I", data[o + 8 + n:o + 12 + n])[0] == zlib.crc32(tag + body) & 0xffffffff
        if tag == b"IHDR":
            w, h, d, ct, _, _, il = struct.unpack(">IIBBBBB", body)
            hdr = dict(width=w, height=h, depth=d, ctype=ct, interlace=il)
        elif tag == b"PLTE":
            plte = body
        elif tag == b"IDAT":
            idat += body
        elif tag == b"IEND":
            break
        o += 12 + n
    raw = zlib.decompress(idat)
    ch = CHANNELS[hdr["ctype"]]
    stride = (hdr["width"] * ch * hdr["depth"] + 7) // 8
    bpp = max(1, ch * hdr["depth"] // 8)
    rows, prev = [], bytes(stride)
    for y in range(hdr["height"]):
        f = raw[y * (stride + 1)]
        s = raw[y * (stride + 1) + 1:(y + 1) * (stride + 1)]
        row = bytearray(stride)
        for i in range(stride):
            a = row[i - bpp] if i >= bpp else 0
            b = prev[i]
            c = prev[i - bpp] if i >= bpp else 0
            pred = [0, a, b, (a + b) >> 1, _paeth(a, b, c)][f]
            row[i] = (s[i] + pred) & 255
        rows.append(bytes(row))
        prev = bytes(row)
    hdr["palette"] = plte
    return hdr, rows


def unpack_samples(row: bytes, n: int, depth: int) -> np.ndarray:
    if depth == 16:
        return np.frombuffer(row, ">u2")[:n].astype(np.int64)
    if depth == 8:
        return np.frombuffer(row, np.uint8)[:n].astype(np.int64)
    per = 8 // depth
    return np.array([(row[i // per] >> (8 - depth * (1 + i % per))) & ((1 << depth) - 1) for i in range(n)])


def to_rgb8(hdr, rows) -> np.ndarray:
    """read_color_png transforms (image_io.cpp:88-92)."""
    w, h, d, ct = hdr["width"], hdr["height"], hdr["depth"], hdr["ctype"]
    ch = CHANNELS[ct]
    out = np.zeros((h, w, 3), np.uint8)
    for y, row in enumerate(rows):
        s = unpack_samples(row, w * ch, d).reshape(w, ch)
        if ct == 3:
            pal = np.frombuffer(hdr["palette"], np.uint8).reshape(-1, 3)
            out[y] = pal[s[:, 0]]
            continue
        v = s >> 8 if d == 16 else (s if d == 8 else s * 255 // ((1 << d) - 1))
        if ch <= 2:
            out[y] = np.repeat(v[:, :1], 3, axis=1)
        else:
            out[y] = v[:, :3]
    return out


def to_depth16(hdr, rows) -> np.ndarray:
    assert hdr["ctype"] == 0 and hdr["depth"] == 16
    return np.stack([np.frombuffer(r, ">u2").astype(np.uint16) for r in rows])


# ---------------------------------------------------------------- PLY
def write_ply(vertices, triangles, normals=None, channels=()) -> bytes:
    """mesh_io.cpp:104-145 (returns the file bytes)."""
    V, T = len(vertices), len(triangles)
    h = "ply\nformat binary_little_endian 1.0\n"
    h += f"element vertex {V}\n"
    h += "property float x\nproperty float y\nproperty float z\n"
    if normals is not None:
        h += "property float nx\nproperty float ny\nproperty float nz\n"
    for name, comps, _ in channels:
        for c in range(comps):
            h += f"property float {name}_{c}\n"
    h += f"element face {T}\n"
    h += "property list uchar int vertex_indices\n"
    for name, comps, _ in channels:
        h += f"comment channel {name} {comps}\n"
    h += "end_header\n"
    cols = [np.asarray(vertices, np.float64).astype(np.float32).reshape(V, 3)]
    if normals is not None:
        cols.append(np.asarray(normals, np.float64).astype(np.float32).reshape(V, 3))
    for _, comps, data in channels:
        cols.append(np.asarray(data, np.float32).reshape(V, comps))
    body = np.concatenate(cols, axis=1).astype("<f4").tobytes() if V else b""
    faces = b"".join(b"\x03" + np.asarray(t, "<i4").tobytes() for t in np.asarray(triangles).reshape(-1, 3))
    return h.encode() + body + faces


def read_ply(data: bytes):
    """mesh_io.cpp:147-218 -> (vertices, normals|None, channels [(name, comps, array)], triangles)."""
    end = data.index(b"end_header\n") + len(b"end_header\n")
    lines = data[:end].decode().split("\n")
    assert lines[0] == "ply"
    nv = nf = 0
    props, chdir = [], []
    for ln in lines[1:]:
        t = ln.split()
        if not t:
            continue
        if t[0] == "format":
            assert t[1] == "binary_little_endian"
        elif t[0] == "element":
            if t[1] == "vertex":
                nv = int(t[2])
            elif t[1] == "face":
                nf = int(t[2])
        elif t[0] == "property" and t[1] != "list":
            props.append(t[2])
        elif t[0] == "comment" and len(t) >= 4 and t[1] == "channel":
            chdir.append((t[2], int(t[3])))
    with_n = len(props) >= 6 and props[3] == "nx"
    per = len(props)
    vb = np.frombuffer(data[end:end + nv * per * 4], "<f4").reshape(nv, per)
    verts = vb[:, :3].astype(np.float64)
    nrm = vb[:, 3:6].astype(np.float64) if with_n else None
    o = 6 if with_n else 3
    chans = []
    for name, comps in chdir:
        chans.append((name, comps, vb[:, o:o + comps].copy()))
        o += comps
    assert o == per
    fo = end + nv * per * 4
    tris = np.zeros((nf, 3), np.int32)
    for f in range(nf):
        assert data[fo] == 3
        tris[f] = np.frombuffer(data[fo + 1:fo + 13], "<i4")
        fo += 13
    return verts, nrm, chans, tris


def with_channels(visible, uv, weight, untextured):
    """texture.cpp:74-91 channel list."""
    ch = []
    for k in range(len(visible)):
        ch.append((f"cam{k}_vis", 1, np.asarray(visible[k], np.float32)))
        ch.append((f"cam{k}_uv", 2, np.asarray(uv[k], np.float32)))
        ch.append((f"cam{k}_w", 1, np.asarray(weight[k], np.float32)))
    ch.append(("untextured", 1, np.asarray(untextured, np.float32)))
    return ch
