"""Oracle exact near-field correction Z0 (O7, E1 of SURVEY.md 8(c)).  TEST INFRASTRUCTURE ONLY.

P:173 (Eq. hms_d2b): u(r_n) = u~(r_n) + sum_{k in near(n)} w^near_kn M(r_k);
P:190: "The correction sparse matrix elements are found through exact integrals of
Eq. (hms_d2) performed over the relevant elements (tetrahedrons in our case)";
P:234: the range is "the average edge length", expanded over periodic images as Eq. new_er.

Reading R10/R12: the node-k charge piece is phi_k*rho + phi_k*sigma*delta_S.
Integrating by parts, its exact potential at r_n is the volume integral

   E_{n<-(k,img)} = int_{supp phi_k + img L} [ phi_k grad' G0(r_n - r') + G0(r_n - r') grad phi_k ] . M_h dV'
   grad' G0(r_n - r') = (r_n - r') / |r_n - r'|^3,

and  (Z0 m)_n = sum_{(k,img) in near(n)} [ E_{n<-(k,img)} - G0*(r_n - r_k - img L) q_k ],  G0*(0) := 0.
near(n) = {(n,0)} for z0_ring = 0; the periodic 1-ring (all (LCA(k), img) whose translated
support contains r_n, deduplicated -- P:142-149, Eq. dedup) for z0_ring = 1.

Quadrature: Duffy collapse + tensor Gauss-Legendre.  When r_n is a vertex of the
element the collapse is taken at that vertex, which removes the 1/R and 1/R^2
singularities analytically; otherwise plain collapsed Gauss with Bey octasection
refinement of elements close to the observer.
"""
import numpy as np
import scipy.sparse as sp

_GL = {}


def _gauss01(n):
    if n not in _GL:
        x, w = np.polynomial.legendre.leggauss(n)
        _GL[n] = (0.5 * (x + 1.0), 0.5 * w)
    return _GL[n]


def _duffy_points(n, n1=None):
    """xi in [0,1]^3 tensor Gauss (n1 points in xi1, n in xi2 and xi3), barycentrics
    lam[Q,4] of the collapsed map
    r = Q0 + xi1 (Q1-Q0) + xi1 xi2 (Q2-Q1) + xi1 xi2 xi3 (Q3-Q2),
    and jacobian factor xi1^2 xi2 (times 6V)."""
    x, w = _gauss01(n)
    x1, w1 = _gauss01(n1 or n)
    X1, X2, X3 = np.meshgrid(x1, x, x, indexing="ij")
    W = np.einsum('i,j,k->ijk', w1, w, w).ravel()
    X1 = X1.ravel(); X2 = X2.ravel(); X3 = X3.ravel()
    lam = np.stack([1 - X1, X1 * (1 - X2), X1 * X2 * (1 - X3), X1 * X2 * X3], axis=1)
    return X1, X2, X3, W, lam


# Bey refinement: children as convex combinations of parent vertices (barycentric rows)
def _bey_children():
    e = np.eye(4)
    mid = lambda i, j: 0.5 * (e[i] + e[j])
    x0, x1, x2, x3 = e
    x01, x02, x03, x12, x13, x23 = mid(0, 1), mid(0, 2), mid(0, 3), mid(1, 2), mid(1, 3), mid(2, 3)
    ch = [(x0, x01, x02, x03), (x01, x1, x12, x13), (x02, x12, x2, x23), (x03, x13, x23, x3),
          (x01, x02, x03, x13), (x01, x02, x12, x13), (x02, x03, x13, x23), (x02, x12, x13, x23)]
    return np.array([np.stack(c) for c in ch])       # [8,4(child vtx),4(parent bary)]


_BEY = _bey_children()


def _child_bary(level):
    """All children after `level` uniform Bey refinements, as [C,4,4] barycentric rows."""
    cur = np.eye(4)[None]
    for _ in range(level):
        cur = np.einsum('cij,pjk->pcik', _BEY, cur).reshape(-1, 4, 4)
    return cur


def moments_vertex(P, va, n=20):
    """Singular case: observer = vertex va of each tet.  P [B,4,3].
    Returns A [B,4] = int phi_m / R,  Bm [B,4,4,3] = int phi_k phi_m (o - r)/R^3."""
    B = P.shape[0]
    order = np.array([[a] + [i for i in range(4) if i != a] for a in range(4)])
    perm = order[va]                                   # [B,4] local index of reordered vertex
    Q = np.take_along_axis(P, perm[:, :, None], axis=1)
    V6 = np.abs(np.einsum('ij,ij->i', np.cross(Q[:, 1] - Q[:, 0], Q[:, 2] - Q[:, 0]), Q[:, 3] - Q[:, 0]))
    # after the collapse the integrands are polynomials of degree <= 2 in xi1: 3 points exact
    X1, X2, X3, W, lam = _duffy_points(n, 3)
    e1 = Q[:, 1] - Q[:, 0]; e2 = Q[:, 2] - Q[:, 1]; e3 = Q[:, 3] - Q[:, 2]
    g = e1[:, None, :] + X2[None, :, None] * (e2[:, None, :] + X3[None, :, None] * e3[:, None, :])  # [B,Q,3]
    gn = np.linalg.norm(g, axis=2)
    # A: w 6V xi1 xi2 lam / |g| ;  B: - w 6V xi2 lam lam g / |g|^3
    wa = (W * X1 * X2)[None, :] * V6[:, None] / gn
    A_r = wa @ lam
    wb = -(W * X2)[None, :, None] * V6[:, None, None] * g / gn[:, :, None] ** 3
    LL = (lam[:, :, None] * lam[:, None, :]).reshape(-1, 16)
    B_r = np.matmul(np.transpose(wb, (0, 2, 1)), LL).reshape(B, 3, 4, 4).transpose(0, 2, 3, 1)
    # un-permute: reordered local j corresponds to original perm[:, j]
    A = np.zeros_like(A_r)
    Bm = np.zeros_like(B_r)
    bi = np.arange(B)[:, None]
    A[bi, perm] = A_r
    tmp = np.zeros_like(B_r)
    tmp[bi, perm] = B_r
    Bm[bi, :, perm] = np.transpose(tmp, (0, 2, 1, 3))
    return A, Bm


def moments_regular(P, o, n=12, level=0):
    """Non-singular case (observer not a vertex): collapsed Gauss on each of the
    8^level Bey children.  P [B,4,3], o [B,3]."""
    X1, X2, X3, W, lam_c = _duffy_points(n)
    ch = _child_bary(level)                               # [C,4,4]
    lam = np.einsum('qj,cjk->cqk', lam_c, ch).reshape(-1, 4)   # parent barycentrics [C*Q,4]
    V6 = np.abs(np.einsum('ij,ij->i', np.cross(P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]), P[:, 3] - P[:, 0]))
    jac = np.tile(W * X1 ** 2 * X2, ch.shape[0]) / ch.shape[0]   # each child has V/8^level
    r = np.matmul(lam[None], P)
    R = o[:, None, :] - r
    Rn = np.sqrt(np.sum(R * R, axis=2))
    wa = jac[None, :] * V6[:, None] / Rn
    A = wa @ lam
    wb = jac[None, :, None] * V6[:, None, None] * R / Rn[:, :, None] ** 3
    LL = (lam[:, :, None] * lam[:, None, :]).reshape(-1, 16)
    Bm = np.matmul(np.transpose(wb, (0, 2, 1)), LL).reshape(P.shape[0], 3, 4, 4).transpose(0, 2, 3, 1)
    return A, Bm


def tet_moments(P, o, va, n=20, nreg=12, nclose=8, chunk=256):
    """Dispatch: va >= 0 -> singular vertex scheme; else regular scheme with one Bey
    refinement when the observer is within 1.5 element diameters of the centroid."""
    B = P.shape[0]
    A = np.zeros((B, 4))
    Bm = np.zeros((B, 4, 4, 3))
    sing = va >= 0
    idx = np.nonzero(sing)[0]
    for s in range(0, idx.size, chunk):
        j = idx[s:s + chunk]
        A[j], Bm[j] = moments_vertex(P[j], va[j], n)
    idx = np.nonzero(~sing)[0]
    if idx.size:
        cen = P[idx].mean(axis=1)
        diam = np.max(np.linalg.norm(P[idx][:, :, None, :] - P[idx][:, None, :, :], axis=3), axis=(1, 2))
        close = np.linalg.norm(o[idx] - cen, axis=1) < 1.5 * diam
        for lvl, nq, sel in ((1, nclose, close), (0, nreg, ~close)):
            jj = idx[sel]
            for s in range(0, jj.size, chunk):
                j = jj[s:s + chunk]
                A[j], Bm[j] = moments_regular(P[j], o[j], nq, lvl)
    return A, Bm


def near_structure(pm, z0_ring, rows=None):
    """Enumerate, for every parent n (or only n in `rows`), near(n) and the deduplicated tet
    images U(n).  Returns (items, near) where items = list of (n, tet, shift(3), va,
    nearmask(4)) and near = list of (n, p, ell(3))."""
    copies = [[] for _ in range(pm.n_parents)]
    for c, p in enumerate(pm.pid):
        copies[p].append(c)
    tets_of = [[] for _ in range(pm.n_nodes)]
    for t, tv in enumerate(pm.tets):
        for v in tv:
            tets_of[v].append(t)
    items, near_list = [], []
    for n in (range(pm.n_parents) if rows is None else rows):
        star = set()
        for c in copies[n]:
            s = tuple(-pm.shift[c])
            for t in tets_of[c]:
                star.add((t, s))
        if z0_ring == 0:
            near = {(n, (0, 0, 0))}
        else:
            near = set()
            for (t, s) in star:
                for v in pm.tets[t]:
                    near.add((int(pm.pid[v]), tuple(int(x) for x in pm.shift[v] + np.array(s))))
        U = set()
        for (p, ell) in near:
            for c in copies[p]:
                s = tuple(int(x) for x in np.array(ell) - pm.shift[c])
                for t in tets_of[c]:
                    U.add((t, s))
        for (t, s) in sorted(U):
            va = -1
            mask = [False] * 4
            for j, v in enumerate(pm.tets[t]):
                key = (int(pm.pid[v]), tuple(int(x) for x in pm.shift[v] + np.array(s)))
                if key in near:
                    mask[j] = True
                if key == (n, (0, 0, 0)):
                    va = j
            items.append((n, t, s, va, mask))
        for (p, ell) in sorted(near):
            near_list.append((n, p, ell))
    return items, near_list


def assemble_z0(pm, ops, Ms_tet, z0_ring=1, nquad=20, rows=None):
    """O7: Z0 as three csr [N',N'] matrices (u_loc = Zx mx + Zy my + Zz mz).  With `rows`,
    only those rows are computed (the others are empty) -- for sampled full-size checks."""
    items, near = near_structure(pm, z0_ring, rows)
    Np = pm.n_parents
    T = pm.tets.shape[0]
    Ms_tet = np.broadcast_to(np.asarray(Ms_tet, dtype=np.float64), (T,))
    n_it = np.array([it[0] for it in items], dtype=np.int64)
    t_it = np.array([it[1] for it in items], dtype=np.int64)
    s_it = np.array([it[2] for it in items], dtype=np.float64).reshape(-1, 3)
    va = np.array([it[3] for it in items], dtype=np.int64)
    mask = np.array([it[4] for it in items], dtype=bool).reshape(-1, 4)
    P = pm.xyz[pm.tets[t_it]] + (s_it * pm.L[None, :])[:, None, :]
    o = pm.xyz[pm.parent[n_it]]
    A, Bm = tet_moments(P, o, va, nquad)
    grads = ops["grads"][t_it]                         # [B,4,3]
    rows, cols, vals = [], [], [[], [], []]
    for k in range(4):
        sel = mask[:, k]
        for m in range(4):
            w = Ms_tet[t_it[sel], None] * (Bm[sel, k, m, :] + grads[sel, k, :] * A[sel, m, None])
            rows.append(n_it[sel]); cols.append(pm.pid[pm.tets[t_it[sel], m]])
            for x in range(3):
                vals[x].append(w[:, x])
    # minus the point-charge value of each near source: -G0*(d) q_k, q_k = D_k . m
    D = [ops["Dx"].tocsr(), ops["Dy"].tocsr(), ops["Dz"].tocsr()]
    xyz_p = pm.xyz[pm.parent]
    for (n, p, ell) in near:
        d = xyz_p[n] - xyz_p[p] - np.array(ell) * pm.L
        r = np.linalg.norm(d)
        if r == 0.0:
            continue
        g = 1.0 / r
        for x in range(3):
            lo, hi = D[x].indptr[p], D[x].indptr[p + 1]
            cc = D[x].indices[lo:hi]
            for y in range(3):
                # keep the three value lists aligned with one shared (rows, cols) list
                vals[y].append(-g * D[x].data[lo:hi] if y == x else np.zeros(hi - lo))
            rows.append(np.full(cc.size, n)); cols.append(cc)
    rows = np.concatenate(rows); cols = np.concatenate(cols)
    Z = [sp.coo_matrix((np.concatenate(vals[x]), (rows, cols)), shape=(Np, Np)).tocsr() for x in range(3)]
    return dict(Zx=Z[0], Zy=Z[1], Zz=Z[2], n_items=len(items), n_near=len(near))
