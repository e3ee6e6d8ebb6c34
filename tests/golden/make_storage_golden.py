"""Golden outputs of the reference's storage / decode / distortion functions
(vqkit imported from /root/reference/pkg/src; build container only).  Inputs
come from tests/golden/cases.py (seeded); only reference OUTPUTS are stored,
in tests/golden/storage.npz.

Usage: python tests/golden/make_storage_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import vqkit  # noqa: E402  (the reference)
from vqkit import storage  # noqa: E402

import cases  # noqa: E402


def main():
    out = {}
    for i, (px, b) in enumerate(cases.image_cases()):
        vectors, grid = storage.pixels_to_blocks(px, b)
        out[f"img{i}_blocks"] = vectors
        out[f"img{i}_grid"] = np.array([grid.width, grid.height, grid.block, grid.count, grid.k])
        pert = cases.raster_vectors(vectors, 100 + i)
        out[f"img{i}_pgm"] = np.frombuffer(storage.blocks_to_image(pert, grid), dtype=np.uint8)
        out[f"img{i}_pgm_identity"] = np.frombuffer(storage.blocks_to_image(vectors, grid), dtype=np.uint8)
        out[f"img{i}_pgmbytes"] = np.frombuffer(storage.pgm_bytes(px), dtype=np.uint8)
    for i, c in enumerate(cases.decode_cases()):
        cb = vqkit.Codebook(c["cb"])
        stream = vqkit.EncodedStream(cb.size, cb.k, c["idx"])
        out[f"dec{i}_rows"] = vqkit.decode(stream, cb)
        path = os.path.join("/tmp", f"vqb_golden_{i}.bin")
        for metric in ("squared_euclidean", "euclidean"):
            storage.save_codebook(cb, metric, path)
            out[f"dec{i}_vqcb_{metric}"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
        storage.save_encoded(stream, path)
        out[f"dec{i}_vqen"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
        os.remove(path)
    for i, c in enumerate(cases.distortion_cases()):
        total, mean = vqkit.reconstruction_distortion(c["a"], c["b"], c["metric"])
        out[f"dist{i}_total"] = np.float64(total)
        out[f"dist{i}_mean"] = np.float64(mean)
    path = os.path.join(HERE, "storage.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
