"""Oracle mesh layer: O1-O3 of SURVEY.md 8(c).  TEST INFRASTRUCTURE ONLY.

O1  orientation + degenerate check            (PAPER.md:80 tetrahedra)
O2  T-PBC pairs, union-find, LCA = min index  ("one of its periodic images ...
    can still be found within the 0th unit cell"; "merge these pairs to their
    lowest common ancestors (LCA) by the union-find algorithm")
O3  wrap of parent coordinates into [0, L) on periodic axes (Eq. shift_hms;
    DESIGN.md reading R16)
"""
import itertools
import numpy as np
from scipy.spatial import cKDTree


class MeshError(ValueError):
    pass


def signed_volumes(xyz, tets):
    """V_T = det[P1-P0, P2-P0, P3-P0] / 6 (plain definition)."""
    p = xyz[tets]
    a = p[:, 1] - p[:, 0]
    b = p[:, 2] - p[:, 0]
    c = p[:, 3] - p[:, 0]
    return np.einsum('ij,ij->i', np.cross(a, b), c) / 6.0


def orient(xyz, tets):
    """O1: return tets with positive orientation (swap vertices 1,2 where negative).
    Rejects |V| < 1e-12 * mean |V|."""
    tets = np.array(tets, dtype=np.int64, copy=True)
    if tets.min() < 0 or tets.max() >= xyz.shape[0]:
        raise MeshError("tet index out of range")
    v = signed_volumes(xyz, tets)
    av = np.abs(v)
    bad = np.nonzero(av < 1e-12 * av.mean())[0]
    if bad.size:
        raise MeshError("degenerate tetrahedron %d" % bad[0])
    neg = v < 0
    tets[neg] = tets[neg][:, [0, 2, 1, 3]]
    return tets


def shortest_edge(xyz, tets):
    p = xyz[tets]
    m = np.inf
    for i, j in itertools.combinations(range(4), 2):
        m = min(m, np.linalg.norm(p[:, i] - p[:, j], axis=1).min())
    return m


def _find(par, i):
    root = i
    while par[root] != root:
        root = par[root]
    while par[i] != root:
        par[i], i = root, par[i]
    return root


def image_offsets(periodic):
    """All (gamma, zeta, xi) in {-1,0,1}^3, zero on non-periodic axes, not all zero
    (PAPER.md:44 with the +-1 reading of DESIGN.md R17)."""
    rng = [(-1, 0, 1) if periodic[a] else (0,) for a in range(3)]
    return [o for o in itertools.product(*rng) if any(o)]


def detect_pbc(xyz, tets, periodic, lattice, match_tol=0.0):
    """O2.  Returns lca[N] (original indices; lca[i] = min index of i's component).

    For every node i and every image offset o, a node j with
    |r_j - (r_i + o*L)| <= match_tol is a PBC partner; partners are
    merged by union-find with the minimum index as the root.
    """
    n = xyz.shape[0]
    Lv = np.array([lattice[a] if periodic[a] else 0.0 for a in range(3)])
    if match_tol <= 0.0:
        match_tol = 1e-6 * shortest_edge(xyz, tets)
    par = list(range(n))
    if not any(periodic):
        return np.arange(n)
    tree = cKDTree(xyz)
    for o in image_offsets(periodic):
        shift = np.array(o, dtype=np.float64) * Lv
        hits = tree.query_ball_point(xyz + shift, match_tol)
        for i, js in enumerate(hits):
            js = [j for j in js if j != i]
            if len(js) > 1:
                raise MeshError("PBC ambiguous: node %d image %s matches %s" % (i, o, js[:2]))
            if js:
                ri, rj = _find(par, i), _find(par, js[0])
                if ri != rj:
                    lo, hi = min(ri, rj), max(ri, rj)
                    par[hi] = lo
    lca = np.array([_find(par, i) for i in range(n)], dtype=np.int64)
    # consistency: members are integer-period translates of the root
    d = xyz - xyz[lca]
    for a in range(3):
        if periodic[a]:
            k = np.round(d[:, a] / Lv[a])
            if np.any(np.abs(d[:, a] - k * Lv[a]) > match_tol):
                raise MeshError("PBC inconsistent component on axis %d" % a)
        elif np.any(np.abs(d[:, a]) > match_tol):
            raise MeshError("PBC inconsistent component on axis %d" % a)
    return lca


class PeriodicMesh:
    """A mesh resolved into parents (unknowns) and children.

    pid[i]      parent id in [0, N') of node i (parents numbered by increasing original index)
    parent[p]   original node index of parent p
    shift[i]    integer lattice shift with r_i = r_parent(i) + shift[i] * L (exact up to match_tol)
    """

    def __init__(self, xyz, tets, periodic, lattice, match_tol=0.0):
        self.xyz = np.asarray(xyz, dtype=np.float64)
        self.tets = orient(self.xyz, tets)
        self.periodic = tuple(int(bool(p)) for p in periodic)
        self.L = np.array([lattice[a] if self.periodic[a] else 0.0 for a in range(3)])
        lca = detect_pbc(self.xyz, self.tets, self.periodic, self.L, match_tol)
        self.lca = lca
        self.parent = np.nonzero(lca == np.arange(lca.size))[0]
        pid_of_parent = np.full(lca.size, -1, dtype=np.int64)
        pid_of_parent[self.parent] = np.arange(self.parent.size)
        self.pid = pid_of_parent[lca]
        d = self.xyz - self.xyz[lca]
        sh = np.zeros((lca.size, 3), dtype=np.int64)
        for a in range(3):
            if self.periodic[a]:
                sh[:, a] = np.round(d[:, a] / self.L[a]).astype(np.int64)
        self.shift = sh
        self.n_nodes = lca.size
        self.n_parents = self.parent.size
        self.vol = signed_volumes(self.xyz, self.tets)

    def children_of(self):
        """dict parent id -> list of node indices (all copies including the parent)."""
        out = [[] for _ in range(self.n_parents)]
        for i, p in enumerate(self.pid):
            out[p].append(i)
        return out

    def extent(self):
        return self.xyz.max(axis=0) - self.xyz.min(axis=0)

    def classify(self, match_tol=None):
        """(touching, protruding) per P:44: touching <=> PBC pairs exist;
        protruding <=> extent D_i > L_i on some periodic axis."""
        if match_tol is None:
            match_tol = 1e-6 * shortest_edge(self.xyz, self.tets)
        D = self.extent()
        touching = self.n_parents < self.n_nodes
        protruding = any(self.periodic[a] and D[a] > self.L[a] + match_tol for a in range(3))
        return touching, protruding

    def wrapped_parent_xyz(self):
        """O3: parent coordinates with periodic axes wrapped into [0, L).
        w = x - L*floor(x/L); w >= L -> w - L; w < 0 -> 0  (R16)."""
        x = self.xyz[self.parent].copy()
        for a in range(3):
            if self.periodic[a]:
                L = self.L[a]
                w = x[:, a] - L * np.floor(x[:, a] / L)
                w = np.where(w >= L, w - L, w)
                w = np.where(w < 0.0, 0.0, w)
                x[:, a] = w
        return x


def fold_manhattan(xyz, periodic, lattice, r0=None):
    """Eq. shift_hms taken literally: shift each point by integer
    multiples delta of L_i to minimise sum_i |x_i - r0_i + delta_i L_i|.
    Returns (folded xyz, delta[N,3]).  Used for the P:255 fold demo pins; the
    BAIM path uses wrapped coordinates (reading R16)."""
    xyz = np.asarray(xyz, dtype=np.float64)
    if r0 is None:
        r0 = xyz.mean(axis=0)
    delta = np.zeros(xyz.shape, dtype=np.int64)
    out = xyz.copy()
    for a in range(3):
        if periodic[a]:
            L = lattice[a]
            # the per-axis terms of the Manhattan sum are independent: minimise each
            cand = np.stack([np.floor((r0[a] - xyz[:, a]) / L) + k for k in (-1, 0, 1, 2)], axis=1)
            cost = np.abs(xyz[:, a:a + 1] - r0[a] + cand * L)
            best = cand[np.arange(xyz.shape[0]), np.argmin(cost, axis=1)]
            delta[:, a] = best.astype(np.int64)
            out[:, a] = xyz[:, a] + best * L
    return out, delta
