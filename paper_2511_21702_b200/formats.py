"""CSVD / CSVH / CSVI binary formats -> device-ready objects.

Readers and writers for the reference's on-disk artefacts, byte-compatible
with `csvd.tensor_io` (tensor_io.py:42-46, 136-189) and
`csvd.cluster_index.save_index / load_index` (cluster_index.py:398-479):

* CSVD table:  header "<4sIQQB7x" (magic, version 1, V, d, dtype 0), then
               V*d little-endian f32 weights and V f32 biases;
* CSVH queries: header "<4sIQQ" (magic, version 1, count, d), count*d f32;
* CSVI index:  header "<4sIBQQQH32s" (magic, version 1, mode code, C, V, d,
               bias depth m, 32-byte fingerprint), per cluster: centroid
               (d or d+1 f64), six f64 stats + u16 top-m count, top-m
               (f64 value, u64 token) pairs, u64 start / end; then V u64 perm.

Differences from the reference readers are deliberate and B200-motivated:
the table is memory-mapped and kept as float32 (the values are identical;
the reference widens to a float64 copy, 2x the host memory), and
`prepare_files` uploads straight from the mapping with the fingerprint
checked once, so a serving process goes from files to a resident device
table without a second host copy.
"""

from __future__ import annotations

import struct

import numpy as np

from .types import ClusterIndex, ClusterMeta, EmbeddingTable, NonFiniteEntryError

MODES = ("euclidean", "spherical", "bias_augmented")
_CSVD = (b"CSVD", struct.Struct("<4sIQQB7x"))
_CSVH = (b"CSVH", struct.Struct("<4sIQQ"))
_CSVI = (b"CSVI", struct.Struct("<4sIBQQQH32s"))
_REC = struct.Struct("<ddddddH")
_TOPM = struct.Struct("<dQ")
_RANGE = struct.Struct("<QQ")


class FormatError(Exception):
    """Base class for binary-format failures (tensor_io.py:49-62)."""


class BadMagicError(FormatError):
    pass


class VersionMismatchError(FormatError):
    pass


class TruncatedPayloadError(FormatError):
    pass


def _header(buf: memoryview, kind, what: str):
    magic, st = kind
    if len(buf) < st.size:
        raise TruncatedPayloadError(f"expected {st.size} bytes for {what} header, got {len(buf)}")
    fields = st.unpack_from(buf, 0)
    if fields[0] != magic:
        raise BadMagicError(f"bad magic {fields[0]!r}, expected {magic!r}")
    if fields[1] != 1:
        raise VersionMismatchError(f"unsupported version {fields[1]}")
    return fields


def _exact_size(total: int, need: int, what: str):
    if total < need:
        raise TruncatedPayloadError(f"expected {need} bytes for {what}, got {total}")
    if total > need:
        raise TruncatedPayloadError("trailing bytes after payload")


def _finite(a: np.ndarray, chunk: int = 1 << 24) -> bool:
    flat = a.reshape(-1)
    return all(np.isfinite(flat[i:i + chunk]).all() for i in range(0, flat.size, chunk))


def load_table(path, mmap: bool = True) -> EmbeddingTable:
    """tensor_io.load_embedding_table (tensor_io.py:136-163), float32, mapped."""
    raw = np.memmap(path, dtype=np.uint8, mode="r") if mmap else np.fromfile(path, dtype=np.uint8)
    _, _, V, d, dtype = _header(memoryview(raw), _CSVD, "table")
    if dtype != 0:
        raise VersionMismatchError(f"unsupported dtype code {dtype}")
    if V < 1 or d < 1:
        raise FormatError(f"invalid dims V={V}, d={d}")
    off = _CSVD[1].size
    _exact_size(raw.size, off + 4 * V * d + 4 * V, "weights and bias")
    w = raw[off:off + 4 * V * d].view("<f4").reshape(V, d)
    b = raw[off + 4 * V * d:].view("<f4")
    if not _finite(w) or not _finite(b):
        raise NonFiniteEntryError("file contains non-finite entries")
    return EmbeddingTable(weights=w, bias=b)


def save_table(table: EmbeddingTable, path) -> None:
    """tensor_io.save_embedding_table (tensor_io.py:166-172)."""
    w = table.weights_f64().astype("<f4") if table.weights.dtype != np.float32 else table.weights.astype("<f4")
    with open(path, "wb") as f:
        f.write(_CSVD[1].pack(_CSVD[0], 1, table.vocab_size, table.hidden_dim, 0))
        f.write(np.ascontiguousarray(w).tobytes())
        f.write(np.asarray(table.bias).astype("<f4").tobytes())


def load_queries(path) -> np.ndarray:
    """tensor_io.load_query_batch (tensor_io.py:175-189): [count, d] float64."""
    raw = np.fromfile(path, dtype=np.uint8)
    _, _, n, d = _header(memoryview(raw), _CSVH, "query batch")
    off = _CSVH[1].size
    _exact_size(raw.size, off + 4 * n * d, "vectors")
    v = raw[off:].view("<f4").reshape(n, d)
    if not _finite(v):
        raise NonFiniteEntryError("file contains non-finite entries")
    return v.astype(np.float64)


def save_queries(vectors: np.ndarray, path) -> None:
    v = np.asarray(vectors)
    with open(path, "wb") as f:
        f.write(_CSVH[1].pack(_CSVH[0], 1, v.shape[0], v.shape[1]))
        f.write(v.astype("<f4").tobytes())


def load_index(path) -> ClusterIndex:
    """cluster_index.load_index (cluster_index.py:432-479)."""
    raw = np.fromfile(path, dtype=np.uint8)
    buf = memoryview(raw)
    _, _, mode_code, C, V, d, m, fp = _header(buf, _CSVI, "index")
    if mode_code >= len(MODES):
        raise VersionMismatchError(f"unknown mode code {mode_code}")
    mode = MODES[mode_code]
    dg = d + 1 if mode == "bias_augmented" else d
    off = _CSVI[1].size
    clusters = []

    def need(n, what):
        if off + n > len(buf):
            raise TruncatedPayloadError(f"expected {n} bytes for {what}, got {len(buf) - off}")

    for _ in range(C):
        need(8 * dg + _REC.size, "cluster record")
        centroid = raw[off:off + 8 * dg].view("<f8").copy()
        off += 8 * dg
        cn, radius, ang, maxb, maxn, minn, n_top = _REC.unpack_from(buf, off)
        off += _REC.size
        need(_TOPM.size * n_top + _RANGE.size, "bias entries and range")
        topm = tuple((v, int(t)) for v, t in (_TOPM.unpack_from(buf, off + _TOPM.size * j) for j in range(n_top)))
        off += _TOPM.size * n_top
        start, end = _RANGE.unpack_from(buf, off)
        off += _RANGE.size
        clusters.append(ClusterMeta(centroid=centroid, centroid_norm=cn, radius=radius, angular=ang,
                                    max_bias=maxb, max_norm=maxn, min_norm=minn, bias_topm=topm,
                                    start=int(start), end=int(end)))
    _exact_size(len(buf) - off, 8 * V, "permutation")
    perm = raw[off:].view("<u8").astype(np.int64)
    return ClusterIndex(clusters=clusters, perm=perm, mode=mode, vocab_size=int(V), hidden_dim=int(d),
                        bias_depth=int(m), fingerprint=fp)


def save_index(index: ClusterIndex, path) -> None:
    """cluster_index.save_index (cluster_index.py:398-429)."""
    with open(path, "wb") as f:
        f.write(_CSVI[1].pack(_CSVI[0], 1, MODES.index(index.mode), index.n_clusters, index.vocab_size,
                              index.hidden_dim, index.bias_depth, index.fingerprint))
        for c in index.clusters:
            f.write(np.asarray(c.centroid, dtype="<f8").tobytes())
            f.write(_REC.pack(c.centroid_norm, c.radius, c.angular, c.max_bias, c.max_norm, c.min_norm,
                              len(c.bias_topm)))
            for value, token in c.bias_topm:
                f.write(_TOPM.pack(value, token))
            f.write(_RANGE.pack(c.start, c.end))
        f.write(np.asarray(index.perm).astype("<u8").tobytes())


def prepare_files(table_path, index_path, device: int | None = None):
    """Files -> resident B200 context: map the table, parse the index, check
    the fingerprint once (instead of per step, decode.py:142-144) and upload.
    Returns (table, index, DeviceIndex); the step API reuses the context."""
    from . import engine
    table = load_table(table_path)
    index = load_index(index_path)
    ctx = engine.prepare(table, index, device)
    return table, index, ctx
