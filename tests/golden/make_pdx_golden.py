"""Generate the .pdx golden files by running the REFERENCE writer.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_pdx_golden.py

Each file is written by the reference's own ``write_pdx`` (storage.py:115-140)
from stores built by its own ``to_blocks`` / ``ivf_build`` / cli helpers
(cli.py:35-64), so the native loader / saver (pdx_io.cu) is pinned to the
reference's bytes: load + save must reproduce every file exactly.  A JSON
sidecar records what the reference read back (n, d, block sizes, ids, a
checksum of each block's data) for the CPU-side checks.
"""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

import dimscan as ds  # noqa: E402  (the reference)
from dimscan import cli, storage  # noqa: E402

OUT = Path(__file__).resolve().parent / "pdx"


def collection(n, d, seed):
    x = np.random.default_rng(seed).standard_normal((n, d)).astype(np.float32)
    return ds.VectorCollection.from_array(x)


def describe(path):
    st = storage.read_pdx(path)
    return {
        "n": st.n, "d": st.d, "block_size": st.block_size, "nblocks": len(st.blocks),
        "transform_seed": st.transform_seed,
        "m": [int(b.m) for b in st.blocks],
        "m_padded": [int(b.data.shape[1]) for b in st.blocks],
        "ids": [[int(i) for i in b.ids] for b in st.blocks],
        "data_sha256": [hashlib.sha256(np.ascontiguousarray(b.data).tobytes()).hexdigest()
                        for b in st.blocks],
        "nlist": st.ivf.nlist if st.ivf is not None else 0,
        "bucket_offsets": ([int(v) for v in st.ivf.bucket_offsets]
                           if st.ivf is not None else None),
        "size": path.stat().st_size,
        "sha256": hashlib.sha256(path.read_bytes()).hexdigest(),
    }


def main():
    OUT.mkdir(exist_ok=True)
    cases = {}
    # flat, padded 64-blocks (cli convert path)
    c = collection(130, 8, 2)
    storage.write_pdx(cli.store_from_collection(c, 64), OUT / "flat64.pdx")
    # rotation section (cli convert --transform-seed)
    c = collection(200, 12, 3)
    storage.write_pdx(cli.store_from_collection(c, 64, transform_seed=5), OUT / "rotated.pdx")
    # padded 128-blocks: one block spans two tiles, the partial one pads to 128
    c = collection(300, 20, 4)
    storage.write_pdx(cli.store_from_collection(c, 128), OUT / "flat128.pdx")
    # unpadded wide partitions (flat_build's layout, index.py:171-179)
    c = collection(260, 16, 5)
    st = storage.BlockStore(blocks=ds.to_blocks(c, 100, pad=False),
                            global_means=ds.compute_means(c).means, block_size=100)
    storage.write_pdx(st, OUT / "wide.pdx")
    # IVF section (cli build path), with an empty bucket possible
    c = collection(700, 10, 6)
    index = ds.ivf_build(c, nlist=12, seed=1)
    storage.write_pdx(cli.store_from_ivf(index, 64), OUT / "ivf.pdx")
    for p in sorted(OUT.glob("*.pdx")):
        cases[p.name] = describe(p)
    (OUT / "pdx_golden.json").write_text(json.dumps(cases, indent=1) + "\n")
    print("wrote", ", ".join(sorted(cases)))


if __name__ == "__main__":
    main()
