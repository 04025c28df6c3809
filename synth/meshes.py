"""Structured tetrahedral meshes: voxel masks split into 6 Kuhn tetrahedra.

Geometry only (no PM-FEM arithmetic).  A lattice of vertices
``origin + (i, j, k) * h`` is built; every kept voxel is split into the six
Kuhn (Freudenthal) tetrahedra that share the voxel's main diagonal, which
gives a conforming mesh for any voxel mask.  Interior vertices are jittered
by a seeded uniform displacement.  On axes flagged ``wrap`` the jitter table
is periodic with the voxel count, so vertices that are periodic images of
one another (the touching-PBC case) receive identical jitter and
stay exact lattice translates.  The jitter component normal
to the bounding-box faces is zero on every axis, so flat free surfaces stay flat
and a touching cell keeps its extent equal to the period.
"""
from dataclasses import dataclass, field
import numpy as np

# the six monotone lattice paths (0,0,0) -> (1,1,1)
_KUHN_PERMS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))


@dataclass
class Mesh:
    xyz: np.ndarray            # [N,3] float64, cm
    tets: np.ndarray           # [T,4] int32, positively oriented
    h: float                   # lattice spacing (cm)
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def n_nodes(self):
        return self.xyz.shape[0]

    @property
    def n_tets(self):
        return self.tets.shape[0]


def kuhn_voxel_mesh(mask, h, origin=(0.0, 0.0, 0.0), wrap=(False, False, False),
                    jitter=0.0, seed=0, name=""):
    """Mesh the kept voxels of ``mask`` ([nx,ny,nz] bool).

    jitter: amplitude as a fraction of h (uniform in [-jitter*h, +jitter*h]).
    wrap[a]: jitter table periodic along axis a with period mask.shape[a].
    """
    mask = np.asarray(mask, dtype=bool)
    nx, ny, nz = mask.shape
    V = np.array([nx + 1, ny + 1, nz + 1])
    ci, cj, ck = np.nonzero(mask)
    ci = ci.astype(np.int64); cj = cj.astype(np.int64); ck = ck.astype(np.int64)

    def lin(i, j, k):
        return (i * V[1] + j) * V[2] + k

    tets = []
    for perm in _KUHN_PERMS:
        a, b, _ = perm
        e = np.eye(3, dtype=np.int64)
        p0 = np.zeros(3, dtype=np.int64)
        p1 = e[a]
        p2 = e[a] + e[b]
        p3 = np.ones(3, dtype=np.int64)
        vs = [lin(ci + p[0], cj + p[1], ck + p[2]) for p in (p0, p1, p2, p3)]
        tets.append(np.stack(vs, axis=1))
    tets = np.concatenate(tets, axis=0)
    # interleave so that the 6 tets of one voxel are adjacent (locality only)
    nc = ci.size
    tets = tets.reshape(6, nc, 4).transpose(1, 0, 2).reshape(-1, 4)

    used = np.unique(tets)
    remap = np.full(int(V.prod()), -1, dtype=np.int64)
    remap[used] = np.arange(used.size)
    tets = remap[tets].astype(np.int32)

    I = used // (V[1] * V[2])
    J = (used // V[2]) % V[1]
    K = used % V[2]
    idx = np.stack([I, J, K], axis=1)
    xyz = np.asarray(origin, dtype=np.float64)[None, :] + idx.astype(np.float64) * h

    if jitter > 0.0:
        rng = np.random.default_rng(seed)
        shape = tuple(int(mask.shape[a]) if wrap[a] else int(V[a]) for a in range(3))
        table = rng.uniform(-jitter * h, jitter * h, size=shape + (3,))
        ii = [idx[:, a] % mask.shape[a] if wrap[a] else idx[:, a] for a in range(3)]
        jit = table[ii[0], ii[1], ii[2]]
        for a in range(3):
            # flat bounding faces stay flat (and a touching cell keeps extent D = L)
            on_face = (idx[:, a] == idx[:, a].min()) | (idx[:, a] == idx[:, a].max())
            jit[on_face, a] = 0.0
        xyz = xyz + jit

    # orientation: make every signed volume positive (swap two vertices)
    p = xyz[tets]
    vol = np.einsum('ij,ij->i', np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), p[:, 3] - p[:, 0]) / 6.0
    neg = vol < 0
    tets[neg] = tets[neg][:, [0, 2, 1, 3]]
    vol = np.abs(vol)
    if vol.min() <= 0.05 * h ** 3 / 6.0:
        raise ValueError("jitter too large: near-degenerate tetrahedron (min V/V0=%.3g)"
                         % (vol.min() / (h ** 3 / 6.0)))
    return Mesh(xyz=xyz, tets=tets, h=h, name=name,
                meta={"lattice_index": idx, "mask_shape": mask.shape})
