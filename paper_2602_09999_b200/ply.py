"""ParameterStore <-> PLY in the de-facto 3DGS vertex layout.

Properties: x y z, f_dc_0..2, f_rest_0..44 (channel-major: f_rest_{c*15+k} is
SH coefficient k+1 of channel c), opacity (logit), scale_0..2 (log),
rot_0..3 (raw quaternion, w first).  The in-memory flat 59*N store keeps
sh_rest coefficient-major [N][15][3], so the codec transposes.
Reads ascii and binary_little_endian with any scalar property types, order and
extra properties; writes float32 in the order above.  Mirrors
include/tilesplat/ply.hpp (the C++ codec) byte for byte.
"""
from __future__ import annotations

import numpy as np

from . import types as T

PROPERTIES = (["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2"] + [f"f_rest_{i}" for i in range(45)] + ["opacity"]
              + [f"scale_{i}" for i in range(3)] + [f"rot_{i}" for i in range(4)])

_TYPES = {"char": "i1", "int8": "i1", "uchar": "u1", "uint8": "u1", "short": "i2", "int16": "i2",
          "ushort": "u2", "uint16": "u2", "int": "i4", "int32": "i4", "uint": "u4", "uint32": "u4",
          "float": "f4", "float32": "f4", "double": "f8", "float64": "f8"}


class PlyError(ValueError):
    """Malformed or incomplete PLY (maps onto the reference's validation error)."""


def params_to_rows(flat: np.ndarray, n: int) -> np.ndarray:
    means, ls, q, op, dc, rest = T.unpack_params(np.asarray(flat, np.float32), n)
    rows = np.empty((n, 59), np.float32)
    rows[:, 0:3] = means
    rows[:, 3:6] = dc
    rows[:, 6:51] = rest.transpose(0, 2, 1).reshape(n, 45)   # [N][15][3] -> [N][3][15]
    rows[:, 51] = op
    rows[:, 52:55] = ls
    rows[:, 55:59] = q
    return rows


def rows_to_params(rows: np.ndarray) -> np.ndarray:
    n = rows.shape[0]
    rest = rows[:, 6:51].reshape(n, 3, 15).transpose(0, 2, 1)
    return T.pack_params(rows[:, 0:3], rows[:, 52:55], rows[:, 55:59], rows[:, 51], rows[:, 3:6], rest)


def write_ply(path, flat: np.ndarray, n: int, binary: bool = True) -> None:
    rows = params_to_rows(flat, n)
    head = ["ply", f"format {'binary_little_endian' if binary else 'ascii'} 1.0", f"element vertex {n}"]
    head += [f"property float {p}" for p in PROPERTIES] + ["end_header"]
    with open(path, "wb") as f:
        f.write(("\n".join(head) + "\n").encode())
        if binary:
            f.write(rows.astype("<f4").tobytes())
        else:
            for r in rows:
                f.write((" ".join("%.9g" % float(x) for x in r) + "\n").encode())


def read_ply(path):
    """-> (flat 59*N float32 params, N)."""
    with open(path, "rb") as f:
        if f.readline().rstrip(b"\r\n") != b"ply":
            raise PlyError(f"{path}: missing ply magic")
        fmt, n, props, in_vertex, seen = None, None, [], False, False
        while True:
            line = f.readline()
            if not line:
                raise PlyError(f"{path}: header without end_header")
            w = line.decode("ascii", "replace").split()
            if not w:
                continue
            if w[0] == "format":
                if w[1] not in ("ascii", "binary_little_endian"):
                    raise PlyError(f"unsupported PLY format {w[1]}")
                fmt = w[1]
            elif w[0] == "element":
                if seen and not in_vertex:
                    continue
                in_vertex = w[1] == "vertex"
                if in_vertex:
                    seen, n = True, int(w[2])
                elif not seen:
                    raise PlyError("element before vertex is unsupported")
            elif w[0] == "property":
                if in_vertex:
                    if w[1] == "list":
                        raise PlyError("list properties in vertex are unsupported")
                    if w[1] not in _TYPES:
                        raise PlyError(f"bad property type {w[1]}")
                    props.append((w[2], _TYPES[w[1]]))
            elif w[0] == "end_header":
                break
        if n is None:
            raise PlyError(f"{path}: no vertex element")
        names = [p for p, _ in props]
        missing = [p for p in PROPERTIES if p not in names]
        if missing:
            raise PlyError(f"missing property {missing[0]}")
        if fmt == "binary_little_endian":
            dt = np.dtype([(p, "<" + t) for p, t in props])
            buf = f.read(dt.itemsize * n)
            if len(buf) < dt.itemsize * n:
                raise PlyError("truncated vertex data")
            rec = np.frombuffer(buf, dtype=dt, count=n)
            rows = np.stack([rec[p].astype(np.float32) for p in PROPERTIES], axis=1) if n else np.zeros((0, 59), np.float32)
        else:
            vals = np.array(f.read().split()[: n * len(props)], dtype=np.float64)
            if vals.size < n * len(props):
                raise PlyError("truncated ascii vertex data")
            vals = vals.reshape(n, len(props))
            rows = np.stack([vals[:, names.index(p)] for p in PROPERTIES], axis=1).astype(np.float32)
    return rows_to_params(np.ascontiguousarray(rows, np.float32).reshape(n, 59)), n
