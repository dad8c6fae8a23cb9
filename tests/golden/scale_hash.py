"""SHA-256 of a generated BASELINE config's inputs (mesh + charges): the
scale fixtures store it instead of the mesh, and the tests regenerate the
mesh with paper_1301_5914_b200.surfaces.baseline_config and compare."""

import hashlib

import numpy as np


def input_hash(cfg) -> str:
    h = hashlib.sha256()
    for a in (cfg.mesh.vertices, cfg.mesh.normals, cfg.mesh.faces.astype(np.int64),
              cfg.charges.positions, cfg.charges.charges):
        a = np.ascontiguousarray(a)
        h.update(a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes())
    return h.hexdigest()
