"""PSTR v1 reader for the tests (pathstore.cpp:410-516 layout; test infrastructure only)."""
import struct

import numpy as np

VERT = np.dtype([("pos", "<f8", 3), ("cos_theta", "<f8"), ("cos_in", "<f8"), ("cos_out", "<f8"),
                 ("span_begin", "<u4"), ("span_end", "<u4"), ("voxel", "<i4"), ("surface", "<i2"),
                 ("species", "i1"), ("kind", "u1")])
SPAN = np.dtype([("voxel", "<u4"), ("length", "<f8")])
EVENT = np.dtype([("vertex", "<u4"), ("detector", "<u2"), ("pixel", "<i4"), ("cos_le", "<f8"),
                  ("geom", "<f8"), ("span_begin", "<u4"), ("span_end", "<u4")])
assert VERT.itemsize == 64 and SPAN.itemsize == 12 and EVENT.itemsize == 34


def read(path):
    raw = open(path, "rb").read()
    assert raw[:4] == b"PSTR" and struct.unpack_from("<I", raw, 4)[0] == 1
    count, gen, seed = struct.unpack_from("<QQQ", raw, 8)
    sorted_flag = raw[32]
    nb = struct.unpack_from("<Q", raw, 33)[0]
    o = 41
    beta = np.frombuffer(raw, "<f8", nb, o)
    o += 8 * nb
    kappa, gamma = struct.unpack_from("<dd", raw, o)
    o += 16
    recs = []
    for _ in range(count):
        stream, trunc = struct.unpack_from("<QB", raw, o)
        o += 9
        dir0 = np.frombuffer(raw, "<f8", 3, o)
        o += 24
        nv = struct.unpack_from("<I", raw, o)[0]
        o += 4
        verts = np.frombuffer(raw, VERT, nv, o)
        o += 64 * nv
        ns = struct.unpack_from("<I", raw, o)[0]
        o += 4
        spans = np.frombuffer(raw, SPAN, ns, o)
        o += 12 * ns
        ne = struct.unpack_from("<I", raw, o)[0]
        o += 4
        events = np.frombuffer(raw, EVENT, ne, o)
        o += 34 * ne
        nl = struct.unpack_from("<I", raw, o)[0]
        o += 4
        le = np.frombuffer(raw, SPAN, nl, o)
        o += 12 * nl
        recs.append(dict(stream=stream, truncated=trunc, dir0=dir0, vertices=verts, spans=spans,
                         events=events, le_spans=le))
    assert o == len(raw)
    return dict(count=count, generation=gen, seed=seed, sorted=sorted_flag, ref_beta=beta, kappa=kappa,
                gamma=gamma, records=recs)


def segment_spans(rec):
    """Spans of segments b = 1..B of one record (list of structured arrays)."""
    v = rec["vertices"]
    return [rec["spans"][v[b]["span_begin"]:v[b]["span_end"]] for b in range(1, len(v))]


def event_spans(rec):
    return [rec["le_spans"][e["span_begin"]:e["span_end"]] for e in rec["events"]]
