"""HBM tile store: the reference's block lists (layout.py:93-110) and IVF
bucket chains (index.py:98-106) packed for the sm_100a scan.

Layout (include/pdx_b200.h): float32 tiles ``[ntiles][d_pad/G][64][G]``,
int64 ids ``[ntiles][64]`` (-1 = padding), a logical-block table
(first tile, vector count) and a bucket table (first block per bucket).
``G = 8`` keeps a vector's 8 consecutive dims in one 32-byte sector (best
for sequential visit orders: ADS, none, BOND-sequential); ``G = 1`` is the
plain PDX row layout (best when BOND visits dims in a query-dependent
permutation).  Packing runs on the GPU (kernel K1); no CPU path exists.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

TILE = _lib.TILE


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2503_04422_b200 needs a CUDA device (B200); "
                           "there is no CPU fallback")
    return torch


def device():
    torch = _torch()
    return torch.device("cuda", torch.cuda.current_device())


def to_device(x, dtype=None):
    """numpy / torch → contiguous CUDA tensor."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x.to(device=device(), dtype=dtype) if dtype is not None else x.to(device())
    else:
        t = torch.from_numpy(np.ascontiguousarray(x)).to(device())
        if dtype is not None:
            t = t.to(dtype)
    return t.contiguous()


def segment_means_rows(data, rows=None, seg_off=None):
    """float64 means of row segments (pdx_segment_means).  With no segments,
    the mean of all rows (compute_means of a collection)."""
    torch = _torch()
    x = to_device(data, torch.float32)
    n, d = x.shape
    single = seg_off is None
    if single:
        seg_off = torch.tensor([0, n], dtype=torch.int64, device=x.device)
    else:
        seg_off = to_device(seg_off, torch.int64)
    nseg = seg_off.numel() - 1
    rows_t = None if rows is None else to_device(rows, torch.int64)
    out = torch.zeros((nseg, d), dtype=torch.float64, device=x.device)
    _lib.check(_lib.lib().pdx_segment_means(_lib.ptr(x), d, _lib.ptr(rows_t), _lib.ptr(seg_off),
                                            nseg, _lib.ptr(out), _lib.stream_handle()))
    return out[0].cpu().numpy() if single else out


class DeviceStore:
    """A packed store in HBM plus the ``pdx_store`` ABI view of it."""

    def __init__(self, tiles, tile_ids, block_tile, block_m, bucket_block, d, group,
                 tile_block=None):
        """block_tile: int64 [nblocks+1] tile prefix; bucket_block: int64
        [nbuckets+1] block prefix; tile_block: int32 [ntiles] (derived when
        omitted)."""
        torch = _torch()
        self.tiles = tiles
        self.tile_ids = tile_ids
        self.block_tile = block_tile
        self.block_m = block_m
        self.bucket_block = bucket_block
        self.d = int(d)
        self.group = int(group)
        self.d_pad = (self.d + 7) // 8 * 8 if self.group == 8 else self.d
        self.nblocks = int(block_m.numel())
        self.nbuckets = int(bucket_block.numel()) - 1
        self.ntiles = int(block_tile[-1].item()) if self.nblocks else 0
        if tile_block is None:
            ntl = block_tile[1:] - block_tile[:-1]
            tile_block = torch.repeat_interleave(
                torch.arange(self.nblocks, dtype=torch.int32, device=tiles.device), ntl)
        self.tile_block = tile_block.to(torch.int32).contiguous()
        nbk = bucket_block[1:] - bucket_block[:-1]
        ntk = block_tile[bucket_block[1:]] - block_tile[bucket_block[:-1]]
        self.max_bucket_blocks = int(nbk.max().item()) if nbk.numel() else 0
        self.max_bucket_tiles = int(ntk.max().item()) if ntk.numel() else 0
        self.c = _lib.PdxStore(self.d, self.d_pad, self.group, self.nbuckets, self.ntiles,
                               self.nblocks, _lib.ptr(tiles), _lib.ptr(tile_ids),
                               _lib.ptr(block_tile), _lib.ptr(block_m), _lib.ptr(bucket_block),
                               self.max_bucket_blocks, self.max_bucket_tiles,
                               _lib.ptr(self.tile_block))

    @property
    def ref(self):
        return C.byref(self.c)

    def ensure_bsa_residuals(self, initial_step: int):
        """Residual energies for the BSA pruner (pdx_bsa_residuals), computed
        once per step schedule and attached to the ABI view."""
        torch = _torch()
        cache = self.__dict__.setdefault("_resid", {})
        if initial_step not in cache:
            n = C.c_int32(0)
            _lib.check(_lib.lib().pdx_bsa_residuals(self.ref, int(initial_step), None,
                                                   C.byref(n), _lib.stream_handle()))
            buf = torch.empty((max(1, self.ntiles), n.value, 64), dtype=torch.float32,
                              device=self.tiles.device)
            _lib.check(_lib.lib().pdx_bsa_residuals(self.ref, int(initial_step), _lib.ptr(buf),
                                                   C.byref(n), _lib.stream_handle()))
            cache[initial_step] = (buf, n.value)
        buf, n = cache[initial_step]
        self.c.d_resid = _lib.ptr(buf)
        self.c.resid_steps = n
        self.c.resid_initial_step = int(initial_step)
        return buf

    @property
    def nbytes(self) -> int:
        return self.tiles.numel() * 4 + self.tile_ids.numel() * 8

    def with_buckets(self, bucket_block) -> "DeviceStore":
        """Same tiles, another grouping of logical blocks into buckets."""
        torch = _torch()
        bb = to_device(bucket_block, torch.int64)
        return DeviceStore(self.tiles, self.tile_ids, self.block_tile, self.block_m, bb,
                           self.d, self.group, self.tile_block)

    def per_block_buckets(self) -> "DeviceStore":
        torch = _torch()
        return self.with_buckets(torch.arange(self.nblocks + 1, dtype=torch.int64,
                                              device=self.tiles.device))

    # -------------------------------------------------------------- builders
    @classmethod
    def pack(cls, x, order, block_m, bucket_nblocks, ids=None, group=8) -> "DeviceStore":
        """Pack rows of ``x`` (device, n x d, float32) into tiles.

        ``order``: int64 row index of each stored vector, in storage order
        (blocks back to back).  ``block_m``: vectors per logical block, in
        storage order.  ``bucket_nblocks``: logical blocks per bucket.
        ``ids``: external id per row of x (None = row index)."""
        torch = _torch()
        if group not in (1, 8):
            raise ValueError("group must be 1 or 8")
        dev = x.device
        n, d = x.shape
        order = to_device(order, torch.int64)
        block_m = to_device(block_m, torch.int64)
        bucket_nblocks = to_device(bucket_nblocks, torch.int64)
        nb = block_m.numel()
        ntiles_b = (block_m + TILE - 1) // TILE
        block_tile = torch.zeros(nb + 1, dtype=torch.int64, device=dev)
        if nb:
            block_tile[1:] = torch.cumsum(ntiles_b, 0)
        ntiles = int(block_tile[-1].item()) if nb else 0
        # storage position -> slot index: block b's i-th vector goes to
        # slot block_tile[b]*64 + i
        slot_src = torch.full((max(ntiles, 1) * TILE,), -1, dtype=torch.int64, device=dev)
        if nb and order.numel():
            pos_start = torch.zeros(nb, dtype=torch.int64, device=dev)
            pos_start[1:] = torch.cumsum(block_m, 0)[:-1]
            blk_of = torch.repeat_interleave(torch.arange(nb, device=dev), block_m)
            within = torch.arange(order.numel(), device=dev) - pos_start[blk_of]
            slot_src[block_tile[blk_of] * TILE + within] = order
        d_pad = (d + 7) // 8 * 8 if group == 8 else d
        tiles = torch.empty((max(ntiles, 1), d_pad // group, TILE, group), dtype=torch.float32,
                            device=dev)
        tile_ids = torch.empty((max(ntiles, 1), TILE), dtype=torch.int64, device=dev)
        ids_t = None if ids is None else to_device(ids, torch.int64)
        xc = x.contiguous()
        _lib.check(_lib.lib().pdx_pack_tiles(_lib.ptr(xc), n, d, _lib.ptr(slot_src), ntiles, group,
                                             _lib.ptr(ids_t), _lib.ptr(tiles), _lib.ptr(tile_ids),
                                             _lib.stream_handle()))
        bucket_block = torch.zeros(bucket_nblocks.numel() + 1, dtype=torch.int64, device=dev)
        if bucket_nblocks.numel():
            bucket_block[1:] = torch.cumsum(bucket_nblocks, 0)
        return cls(tiles, tile_ids, block_tile, block_m.to(torch.int32), bucket_block, d, group)

    @classmethod
    def from_blocks(cls, blocks, group=8, one_bucket_per_block=True) -> "DeviceStore":
        """Upload a list of host Blocks (layout.Block or the reference's)."""
        torch = _torch()
        if not blocks:
            raise ValueError("empty block list")
        d = blocks[0].data.shape[0]
        for b in blocks:
            if b.data.shape[0] != d:
                raise ValueError("blocks disagree on dimensionality")
        rows = np.concatenate([np.asarray(b.data, np.float32)[:, :b.m].T for b in blocks], axis=0)
        ids = np.concatenate([np.asarray(b.ids, np.int64) for b in blocks])
        ms = np.array([int(b.m) for b in blocks], dtype=np.int64)
        x = to_device(rows, torch.float32)
        order = torch.arange(rows.shape[0], dtype=torch.int64, device=x.device)
        per = np.ones(len(blocks), np.int64) if one_bucket_per_block else np.array([len(blocks)])
        return cls.pack(x, order, ms, per, ids=ids, group=group)
