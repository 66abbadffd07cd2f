"""Packing helpers for golden fixtures (scene geometry as flat arrays)."""
from __future__ import annotations

from types import SimpleNamespace

import numpy as np


def pack_bodies(prefix, bodies, out):
    """bodies: objects with rest/triangles/edges/dynamic -> flat arrays in `out`."""
    out[prefix + "v_off"] = np.cumsum([0] + [len(b.rest) for b in bodies]).astype(np.int64)
    out[prefix + "t_off"] = np.cumsum([0] + [len(b.triangles) for b in bodies]).astype(np.int64)
    out[prefix + "e_off"] = np.cumsum([0] + [len(b.edges) for b in bodies]).astype(np.int64)
    out[prefix + "rest"] = np.concatenate([b.rest for b in bodies])
    out[prefix + "tris"] = np.concatenate([b.triangles for b in bodies]).astype(np.int64)
    out[prefix + "edges"] = np.concatenate([b.edges for b in bodies]).astype(np.int64)
    out[prefix + "dynamic"] = np.array([b.dynamic for b in bodies], dtype=bool)


def unpack_meshes(prefix, g):
    """-> list of (vertices, triangles, edges, dynamic)."""
    vo, to, eo = g[prefix + "v_off"], g[prefix + "t_off"], g[prefix + "e_off"]
    res = []
    for k in range(len(vo) - 1):
        res.append((g[prefix + "rest"][vo[k]:vo[k + 1]],
                    g[prefix + "tris"][to[k]:to[k + 1]],
                    g[prefix + "edges"][eo[k]:eo[k + 1]],
                    bool(g[prefix + "dynamic"][k])))
    return res


def oracle_bodies(prefix, g):
    """Duck-typed body records for the oracle."""
    out = []
    for v, t, e, dyn in unpack_meshes(prefix, g):
        d = v[e[:, 1]] - v[e[:, 0]]
        out.append(SimpleNamespace(rest=v, triangles=t, edges=e,
                                   edge_rest_len_sq=np.einsum("ij,ij->i", d, d), dynamic=dyn))
    return out


def pack_offdict(prefix, off, out):
    keys = sorted(off.keys())
    out[prefix + "off_keys"] = np.array(keys, dtype=np.int64).reshape(-1, 2)
    out[prefix + "off_blocks"] = (np.array([off[k] for k in keys]).reshape(-1, 12, 12)
                                  if keys else np.zeros((0, 12, 12)))
