"""Dataset and store file IO (storage.py:1-194 of the reference).

Host side, same API and errors as the reference: ``.fvecs`` / ``.ivecs``
records and the ``.pdx`` container as numpy ``BlockStore`` objects
(``read_pdx`` / ``write_pdx``).  Device side: ``load_index`` streams a
``.pdx`` file straight into an HBM store (``pdx_file_load``: pinned staging,
GPU transposition into the tile layout) and ``save_index`` writes an HBM
index back (``pdx_file_save``); a loaded store saves to the identical bytes.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .layout import Block, VectorCollection

MAGIC = b"PDXv1\x00\x00\x00"
VERSION = 1
FLAG_TRANSFORM = 1
FLAG_IVF = 2

_HEADER = struct.Struct("<8sIIQIIII")  # magic, version, flags, n, d, block_size, block_count, reserved


class FormatError(ValueError):
    """A file does not follow the expected byte layout (storage.py:29)."""


# ------------------------------------------------------------ fvecs / ivecs
def read_fvecs(path) -> VectorCollection:
    return VectorCollection.from_array(_read_vecs(path, np.float32))


def write_fvecs(collection: VectorCollection, path):
    _write_vecs(path, np.ascontiguousarray(collection.data, dtype=np.float32))


def read_ivecs(path) -> np.ndarray:
    """Integer records, e.g. ground-truth neighbour ids."""
    return _read_vecs(path, np.int32)


def write_ivecs(matrix: np.ndarray, path):
    _write_vecs(path, np.ascontiguousarray(matrix, dtype=np.int32))


def _read_vecs(path, dtype) -> np.ndarray:
    """Records of a little-endian u32 dimensionality then that many values
    (storage.py:50-69, same FormatError messages)."""
    raw = np.fromfile(path, dtype=np.uint8)
    if raw.size == 0:
        raise FormatError(f"{path}: no records (dimensionality is indeterminate)")
    if raw.size < 4:
        raise FormatError(f"{path}: truncated record at byte offset 0")
    d = int(raw[:4].view("<u4")[0])
    if d < 1:
        raise FormatError(f"{path}: invalid dimensionality {d} at byte offset 0")
    rec = 4 + 4 * d
    if raw.size % rec:
        raise FormatError(f"{path}: truncated record at byte offset {(raw.size // rec) * rec}")
    recs = raw.reshape(-1, rec)
    dims = recs[:, :4].copy().view("<u4")[:, 0]
    bad = np.flatnonzero(dims != d)
    if bad.size:
        raise FormatError(f"{path}: inconsistent dimensionality {int(dims[bad[0]])} "
                          f"at record {int(bad[0])}, expected {d}")
    return recs[:, 4:].copy().view(np.dtype(dtype).newbyteorder("<")).astype(dtype)


def _write_vecs(path, matrix: np.ndarray):
    n, d = matrix.shape
    out = np.empty((n, 4 + 4 * d), dtype=np.uint8)
    out[:, :4] = np.frombuffer(struct.pack("<I", d), dtype=np.uint8)
    out[:, 4:] = matrix.astype(matrix.dtype.newbyteorder("<"), copy=False).view(np.uint8) \
        .reshape(n, 4 * d)
    try:
        out.tofile(path)
    except OSError as exc:
        raise OSError(f"{path}: {exc}") from exc


# ------------------------------------------------------------- host .pdx
@dataclass
class IvfSection:
    """Bucket-index extension (storage.py:99-107)."""

    nlist: int
    training_seed: int
    centroids: np.ndarray  # (nlist, d) float32
    bucket_offsets: np.ndarray  # (nlist + 1,) uint32 into the block list
    bucket_means: np.ndarray  # (nlist, d) float64


@dataclass
class BlockStore:
    """A persisted collection in dimension-major blocks (storage.py:80-96)."""

    blocks: list
    global_means: np.ndarray  # (d,) float64
    block_size: int
    transform_seed: int | None = None
    transform_matrix: np.ndarray | None = None  # (d, d) float32
    ivf: IvfSection | None = None

    @property
    def n(self) -> int:
        return sum(b.m for b in self.blocks)

    @property
    def d(self) -> int:
        return self.blocks[0].d if self.blocks else self.global_means.shape[0]


def write_pdx(store: BlockStore, path):
    """storage.py:110-140 (host objects)."""
    flags = (FLAG_TRANSFORM if store.transform_matrix is not None else 0) | \
        (FLAG_IVF if store.ivf is not None else 0)
    try:
        with open(path, "wb") as f:
            f.write(_HEADER.pack(MAGIC, VERSION, flags, store.n, store.d, store.block_size,
                                 len(store.blocks), 0))
            f.write(np.asarray(store.global_means, dtype="<f8").tobytes())
            if store.transform_matrix is not None:
                f.write(struct.pack("<Q", store.transform_seed))
                f.write(np.asarray(store.transform_matrix, dtype="<f4").tobytes())
            for b in store.blocks:
                f.write(struct.pack("<II", b.m, b.data.shape[1]))
                f.write(np.asarray(b.ids, dtype="<i8").tobytes())
                f.write(np.asarray(b.data, dtype="<f4").tobytes())
            if store.ivf is not None:
                v = store.ivf
                f.write(struct.pack("<IQ", v.nlist, v.training_seed))
                f.write(np.asarray(v.centroids, dtype="<f4").tobytes())
                f.write(np.asarray(v.bucket_offsets, dtype="<u4").tobytes())
                f.write(np.asarray(v.bucket_means, dtype="<f8").tobytes())
    except OSError as exc:
        raise OSError(f"{path}: {exc}") from exc


def read_pdx(path) -> BlockStore:
    """storage.py:162-194 (host objects); framing validated natively
    (pdx_file_probe), so both readers raise the same FormatErrors."""
    info = probe(path)
    buf = memoryview(open(path, "rb").read())
    d = info["d"]
    pos = _HEADER.size

    def arr(dtype, count):
        nonlocal pos
        dt = np.dtype(dtype)
        a = np.frombuffer(buf[pos:pos + dt.itemsize * count], dtype=dt).copy()
        pos += dt.itemsize * count
        return a

    means = arr("<f8", d)
    seed = matrix = None
    if info["flags"] & FLAG_TRANSFORM:
        seed = int(arr("<u8", 1)[0])
        matrix = arr("<f4", d * d).astype(np.float32).reshape(d, d)
    blocks = []
    for _ in range(info["nblocks"]):
        m, mp = (int(v) for v in arr("<u4", 2))
        ids = arr("<i8", m).astype(np.int64)
        data = arr("<f4", d * mp).astype(np.float32).reshape(d, mp)
        blocks.append(Block(data=data, ids=ids, m=m))
    ivf = None
    if info["flags"] & FLAG_IVF:
        nlist = int(arr("<u4", 1)[0])
        tseed = int(arr("<u8", 1)[0])
        ivf = IvfSection(nlist=nlist, training_seed=tseed,
                         centroids=arr("<f4", nlist * d).astype(np.float32).reshape(nlist, d),
                         bucket_offsets=arr("<u4", nlist + 1),
                         bucket_means=arr("<f8", nlist * d).reshape(nlist, d))
    return BlockStore(blocks=blocks, global_means=means, block_size=info["block_size"],
                      transform_seed=seed, transform_matrix=matrix, ivf=ivf)


# ----------------------------------------------------------- device .pdx
def probe(path) -> dict:
    """Sizes and framing of a .pdx file (pdx_file_probe; no GPU needed)."""
    info = _lib.PdxFileInfo()
    _lib.check(_lib.lib().pdx_file_probe(str(path).encode(), C.byref(info)))
    return {f: getattr(info, f) for f, _ in _lib.PdxFileInfo._fields_}


def load_index(path, group: int = 8):
    """Stream a .pdx file into HBM (pdx_file_load).

    Returns an ``IvfIndex`` when the file has an IVF section, else a
    ``FlatPartitioning`` over its blocks.  Either carries ``transform`` (an
    OrthogonalTransform, or None), ``global_means`` and ``block_mpad`` so
    ``save_index`` writes the same bytes back."""
    import torch
    from .index import FlatPartitioning, IvfIndex
    from .pruning import OrthogonalTransform
    from .store import DeviceStore, to_device
    info = _lib.PdxFileInfo()
    L = _lib.lib()
    _lib.check(L.pdx_file_probe(str(path).encode(), C.byref(info)))
    d, nb, nt, nlist = info.d, info.nblocks, info.ntiles, info.nlist
    d_pad = (d + 7) // 8 * 8 if group == 8 else d
    dev = torch.device("cuda", torch.cuda.current_device())
    tiles = torch.empty((max(nt, 1), d_pad // group, 64, group), dtype=torch.float32, device=dev)
    tile_ids = torch.empty((max(nt, 1), 64), dtype=torch.int64, device=dev)
    bm = np.zeros(max(nb, 1), np.int32)
    bmp = np.zeros(max(nb, 1), np.int32)
    means = np.zeros(d, np.float64)
    transform = np.zeros((d, d), np.float32) if info.flags & FLAG_TRANSFORM else None
    cent = np.zeros((max(nlist, 1), d), np.float32)
    boff = np.zeros(nlist + 1, np.int64)
    bmeans = np.zeros((max(nlist, 1), d), np.float64)
    _lib.check(L.pdx_file_load(str(path).encode(), C.byref(info), int(group), _lib.ptr(tiles),
                               _lib.ptr(tile_ids), _lib.ptr(bm), _lib.ptr(bmp), _lib.ptr(means),
                               _lib.ptr(transform), _lib.ptr(cent), _lib.ptr(boff),
                               _lib.ptr(bmeans), _lib.stream_handle()))
    bm, bmp = bm[:nb], bmp[:nb]
    ntl = (bm.astype(np.int64) + 63) // 64
    block_tile = np.concatenate([[0], np.cumsum(ntl)]).astype(np.int64)
    bucket_block = boff if nlist else np.array([0, nb], np.int64)
    store = DeviceStore(tiles, tile_ids, to_device(block_tile, torch.int64),
                        to_device(bm, torch.int32), to_device(bucket_block, torch.int64), d, group)
    tf = None if transform is None else OrthogonalTransform(matrix=transform,
                                                            seed=int(info.transform_seed))
    if nlist:
        obj = IvfIndex(nlist, cent[:nlist], store, to_device(bmeans[:nlist], torch.float64),
                       int(info.training_seed), info.block_size)
    else:
        obj = FlatPartitioning(store=store, global_means=means, partition_size=info.block_size)
    obj.transform = tf
    obj.global_means = means
    obj.block_mpad = bmp
    return obj


def _global_means(index) -> np.ndarray:
    """compute_means of the stored vectors in store order (cli.py:56-57)."""
    gm = getattr(index, "global_means", None)
    if gm is not None:
        return np.asarray(gm, np.float64)
    from .store import segment_means_rows
    data = getattr(index, "_host_data", None)
    if data is None:
        raise ValueError("index keeps no host data; pass global_means")
    order = index._order if getattr(index, "_order", None) is not None else None
    return segment_means_rows(data, rows=order)


def save_index(index, path, transform=None, global_means=None):
    """Write an HBM index (IvfIndex or FlatPartitioning) as a .pdx file
    (pdx_file_save), byte-compatible with the reference's write_pdx."""
    import torch
    from .index import IvfIndex
    st = index.store
    tf = transform if transform is not None else getattr(index, "transform", None)
    gm = np.ascontiguousarray(global_means if global_means is not None else _global_means(index),
                              dtype=np.float64)
    mpad = getattr(index, "block_mpad", None)
    if isinstance(index, IvfIndex):
        bs = index.block_size
        if mpad is None:  # to_blocks(pad=True): every block pads to block_size
            mpad = np.full(st.nblocks, bs, np.int32)
        boff = st.bucket_block.cpu().numpy().astype(np.int64)
        nlist, seed = index.nlist, int(index.training_seed)
        cent = np.ascontiguousarray(index.centroids, np.float32)
        bmeans = np.ascontiguousarray(index.means_dev.cpu().numpy(), np.float64)
    else:
        bs = index.partition_size
        nlist, seed, cent, boff, bmeans = 0, 0, None, None, None
    mpad = None if mpad is None else np.ascontiguousarray(mpad, np.int32)
    mat = None if tf is None else np.ascontiguousarray(tf.matrix, np.float32)
    torch.cuda.synchronize()
    _lib.check(_lib.lib().pdx_file_save(str(path).encode(), st.ref, int(bs), _lib.ptr(mpad),
                                        _lib.ptr(gm), _lib.ptr(mat),
                                        int(tf.seed) if tf is not None else 0, int(nlist), seed,
                                        _lib.ptr(cent), _lib.ptr(boff), _lib.ptr(bmeans),
                                        _lib.stream_handle()))
