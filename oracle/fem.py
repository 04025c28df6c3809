"""Oracle local operators: O4-O6 and E1 of SURVEY.md 8(c).  TEST INFRASTRUCTURE ONLY.

Linear tetrahedral basis phi_n (Eq. M_phi).  All operators are assembled
over ALL N-node tetrahedra and then folded through the LCA map: each child row is
accumulated into its parent row and each child column remapped to its parent
column, duplicates summed.  This is the assemble-then-fold realisation of the
paper's Cases 1-3 (Eqs. lapl, lapl_1, shift, dedup, lapl_2); the
charge and gradient operators are "modified similarly".

Readings: R1 charge sign q_n = int grad(phi_n) . M dV (rho=-div M,
sigma = n.M); R14 lumped-mass gradient; R15 lumped-mass exchange with 2A/Ms folded in.
"""
import numpy as np
import scipy.sparse as sp


def element_gradients(xyz, tets):
    """O4: grad(phi_i)|_T for i=0..3 and V_T.  phi_i(r) = [1,x,y,z] . C[:, i] with
    C = inverse of the 4x4 matrix whose rows are [1, x_j, y_j, z_j] (plain definition)."""
    p = xyz[tets]                                  # [T,4,3]
    M = np.concatenate([np.ones(p.shape[:2] + (1,)), p], axis=2)   # [T,4,4]
    C = np.linalg.inv(M)                           # [T,4,4]; column i = coeffs of phi_i
    grads = np.transpose(C[:, 1:4, :], (0, 2, 1))  # [T,4(i),3]
    vol = np.linalg.det(M) / 6.0
    return grads, vol




def assemble(pm, Ms_tet, Aex_tet):
    """O5 + O6.  Returns dict with
       Vt   [N']      lumped nodal volume  sum_{T ∋ copy of n} V_T / 4
       S    csr       folded stiffness  sum_T c_T V_T grad(phi_n).grad(phi_m), c_T = 2 A_T / Ms_T
       Dx,Dy,Dz csr   folded charge     sum_T Ms_T (V_T/4) grad(phi_n)   (q = D . m)
       Gx,Gy,Gz csr   folded gradient   (1/Vt_n) sum_T (V_T/4) grad(phi_m)   (H = -G u)
    """
    grads, vol = element_gradients(pm.xyz, pm.tets)
    T = pm.tets.shape[0]
    Np = pm.n_parents
    Ms_tet = np.broadcast_to(np.asarray(Ms_tet, dtype=np.float64), (T,))
    Aex_tet = np.broadcast_to(np.asarray(Aex_tet, dtype=np.float64), (T,))
    pid = pm.pid[pm.tets]                          # [T,4]
    Vt = np.zeros(Np)
    np.add.at(Vt, pid.ravel(), np.repeat(vol / 4.0, 4))
    rows, cols, s_val = [], [], []
    d_val = [[], [], []]
    g_val = [[], [], []]
    coef = 2.0 * Aex_tet / Ms_tet
    for a in range(4):
        for b in range(4):
            rows.append(pid[:, a]); cols.append(pid[:, b])
            s_val.append(coef * vol * np.einsum('ij,ij->i', grads[:, a], grads[:, b]))
            for x in range(3):
                d_val[x].append(Ms_tet * vol / 4.0 * grads[:, a, x])
                g_val[x].append(vol / 4.0 * grads[:, b, x])
    rows = np.concatenate(rows); cols = np.concatenate(cols)

    def mk(v):
        return sp.coo_matrix((np.concatenate(v), (rows, cols)), shape=(Np, Np)).tocsr()

    S = mk(s_val)
    D = [mk(d_val[x]) for x in range(3)]
    Ginv = sp.diags(1.0 / Vt)
    G = [(Ginv @ mk(g_val[x])).tocsr() for x in range(3)]
    return dict(Vt=Vt, S=S, Dx=D[0], Dy=D[1], Dz=D[2], Gx=G[0], Gy=G[1], Gz=G[2],
                grads=grads, vol=vol)


def charges(ops, m):
    """E1: q_n = sum_m D_nm . m_m   (Eq. hms_d1)."""
    return ops["Dx"] @ m[:, 0] + ops["Dy"] @ m[:, 1] + ops["Dz"] @ m[:, 2]


def exchange_field(ops, m):
    """E1: H_ex,n = -(1/Vt_n) sum_m S_nm m_m   (Eqs. hex/lapl; lumped mass R15)."""
    return -(ops["S"] @ m) / ops["Vt"][:, None]


def gradient_field(ops, u):
    """E6: H_ms,n = -sum_m G_nm u_m   (Eq. hms_d3)."""
    return -np.stack([ops["Gx"] @ u, ops["Gy"] @ u, ops["Gz"] @ u], axis=1)
