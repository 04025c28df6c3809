"""The five BASELINE.json workloads as seeded synthetic inputs.

Every config is a voxel mask + Kuhn split (synth.meshes) with its lattice,
periodic flags, AIM grid and material.  ``coarsen=c`` multiplies h by c and
divides the grid by c (same geometry, ~c^3 fewer nodes): the "tiny analogues"
the oracle finishes in seconds.
Units: CGS (cm).  1 nm = 1e-7 cm.
"""
import math
import numpy as np
from .meshes import kuhn_voxel_mesh

NM = 1e-7

CONFIGS = {
    # name: description (BASELINE.json configs[i])
    "C1": "3D-periodic cube, ~1k nodes filling the cell (touching), 16^3 AIM grid",
    "C2": "2D-periodic antidot film, ~200k nodes, 128x128x8 AIM grid",
    "C3": "1D-periodic nanowire segments (non-touching), ~1M nodes, 512x64x64 AIM grid",
    "C4": "3D-periodic BCC spheres protruding beyond the cell, ~10M nodes, 256^3 AIM grid",
    "C5": "1D-periodic waveguide strip (touching), ~2M nodes, 2048x64x8 AIM grid",
    # non-periodic mode: not a BASELINE.json workload
    "N1": "non-periodic isolated cube, ~1k nodes, 16^3 AIM grid (32^3 FFT)",
    "N2": "non-periodic isolated sphere, ~30k nodes, 32^3 AIM grid (64^3 FFT)",
    # other periodic axes (parity coverage, not BASELINE workloads)
    "R1": "1D-periodic rod along z (PAPER.md:277: R = 20 nm, cell height 2R, touching), 16x16x16 AIM grid",
    "Y1": "1D-periodic strip along y with a slot (touching), 8x64x4 AIM grid",
    # NEXT-2 spin-wave check (Eq. sw_disp): a continuous 2D-periodic film
    "K1": "2D-periodic Permalloy film 200 nm x 40 nm x 10 nm (touching), 64x16x4 AIM grid",
}


def _round_cells(length, h):
    return max(1, int(round(length / h)))


def make_config(name, coarsen=1, jitter=0.15, seed=None, grid=None, cells=None):
    """Return dict(mesh, periodic, L, grid, Ms, Aex, name, desc)."""
    if seed is None:
        seed = {"C": 1000, "N": 2000, "R": 3000, "Y": 4000, "K": 5000}[name[0]] + int(name[1:])
    c = float(coarsen)
    if name == "C1":
        L = 100 * NM
        n = cells or max(2, int(round(10 / c)))
        h = L / n
        mask = np.ones((n, n, n), bool)
        mesh = kuhn_voxel_mesh(mask, h, wrap=(True, True, True), jitter=jitter, seed=seed, name=name)
        periodic = (1, 1, 1); lattice = (L, L, L)
        g = grid or (max(8, int(16 // c)),) * 3
        Ms, Aex = 637.0, 1.4e-6
    elif name == "C2":
        L = 400 * NM; t = 10 * NM; h = 2 * NM * c
        nxy = _round_cells(L, h); nz = max(1, _round_cells(t, h))
        h = L / nxy
        xc = (np.arange(nxy) + 0.5) * h
        X, Y = np.meshgrid(xc, xc, indexing="ij")
        keep = (X - L / 2) ** 2 + (Y - L / 2) ** 2 > (80 * NM) ** 2
        mask = np.repeat(keep[:, :, None], nz, axis=2)
        mesh = kuhn_voxel_mesh(mask, h, wrap=(True, True, False), jitter=jitter, seed=seed, name=name)
        periodic = (1, 1, 0); lattice = (L, L, 0.0)
        g = grid or (max(16, int(128 // c)), max(16, int(128 // c)), max(4, int(round(8 / c))))
        Ms, Aex = 637.0, 1.4e-6
    elif name == "C3":
        L = 800 * NM; h = L / max(8, int(round(456 / c)))
        nx = _round_cells(L, h)
        d = 100 * NM
        nyz = int(math.ceil(d / h))
        xc = (np.arange(nx) + 0.5) * h
        yc = (np.arange(nyz) + 0.5) * h
        keepx = (xc >= 40 * NM) & (xc <= 760 * NM)
        Y, Z = np.meshgrid(yc, yc, indexing="ij")
        keepyz = (Y - nyz * h / 2) ** 2 + (Z - nyz * h / 2) ** 2 <= (d / 2) ** 2
        mask = keepx[:, None, None] & keepyz[None, :, :]
        mesh = kuhn_voxel_mesh(mask, h, wrap=(True, False, False), jitter=jitter, seed=seed, name=name)
        periodic = (1, 0, 0); lattice = (L, 0.0, 0.0)
        g = grid or (max(16, int(512 // c)), max(8, int(64 // c)), max(8, int(64 // c)))
        Ms, Aex = 637.0, 1.4e-6
    elif name == "C4":
        L = 2650 * NM; n = max(8, int(round(265 / c))); h = L / n
        R = 0.4 * L
        lo = -int(math.ceil(R / h)) - 1
        hi = int(math.ceil((0.5 * L + R) / h)) + 1
        idx = np.arange(lo, hi)
        cc = (idx + 0.5) * h
        X, Y, Z = np.meshgrid(cc, cc, cc, indexing="ij")
        keep = (X ** 2 + Y ** 2 + Z ** 2 <= R * R) | \
               ((X - L / 2) ** 2 + (Y - L / 2) ** 2 + (Z - L / 2) ** 2 <= R * R)
        mesh = kuhn_voxel_mesh(keep, h, origin=(lo * h,) * 3, wrap=(True, True, True),
                               jitter=jitter, seed=seed, name=name)
        # wrap=True on an axis whose voxel count is not n would break image
        # consistency; the spheres are non-touching so no images exist.
        periodic = (1, 1, 1); lattice = (L, L, L)
        g = grid or (max(16, int(256 // c)),) * 3
        Ms, Aex = 200.0, 1e-6
    elif name == "C5":
        L = 6400 * NM; h = 2 * NM * c
        nx = _round_cells(L, h); h = L / nx
        ny = _round_cells(200 * NM, h); nz = max(1, _round_cells(10 * NM, h))
        mask = np.ones((nx, ny, nz), bool)
        mesh = kuhn_voxel_mesh(mask, h, wrap=(True, False, False), jitter=jitter, seed=seed, name=name)
        periodic = (1, 0, 0); lattice = (L, 0.0, 0.0)
        g = grid or (max(16, int(2048 // c)), max(8, int(64 // c)), max(4, int(round(8 / c))))
        Ms, Aex = 637.0, 1.4e-6
    elif name == "N1":
        L = 100 * NM
        n = cells or max(2, int(round(10 / c)))
        h = L / n
        mask = np.ones((n, n, n), bool)
        mesh = kuhn_voxel_mesh(mask, h, wrap=(False, False, False), jitter=jitter, seed=seed, name=name)
        periodic = (0, 0, 0); lattice = (0.0, 0.0, 0.0)
        g = grid or (max(8, int(16 // c)),) * 3
        Ms, Aex = 637.0, 1.4e-6
    elif name == "N2":
        R = 60 * NM; h = 4 * NM * c
        n = int(math.ceil(R / h))
        cc = (np.arange(-n, n) + 0.5) * h
        X, Y, Z = np.meshgrid(cc, cc, cc, indexing="ij")
        keep = X ** 2 + Y ** 2 + Z ** 2 <= R * R
        mesh = kuhn_voxel_mesh(keep, h, origin=(-n * h,) * 3, wrap=(False, False, False),
                               jitter=jitter, seed=seed, name=name)
        periodic = (0, 0, 0); lattice = (0.0, 0.0, 0.0)
        g = grid or (max(8, int(32 // c)),) * 3
        Ms, Aex = 637.0, 1.4e-6
    elif name == "R1":
        # infinitely long cylindrical rod, unit cell height 2R, T-NP-PBC along z;
        # A = 9.604e-7 erg/cm, Ms = 490 emu/cm^3
        R = 20 * NM; Lz = 2 * R; h = 2.5 * NM * c
        n = int(math.ceil(R / h))
        nz = _round_cells(Lz, h); h_z = Lz / nz
        h = h_z
        n = int(math.ceil(R / h))
        cc = (np.arange(-n, n) + 0.5) * h
        X, Y = np.meshgrid(cc, cc, indexing="ij")
        disk = X ** 2 + Y ** 2 <= R * R
        mask = np.repeat(disk[:, :, None], nz, axis=2)
        mesh = kuhn_voxel_mesh(mask, h, origin=(-n * h, -n * h, 0.0), wrap=(False, False, True),
                               jitter=jitter, seed=seed, name=name)
        periodic = (0, 0, 1); lattice = (0.0, 0.0, Lz)
        g = grid or (max(8, int(16 // c)),) * 3
        Ms, Aex = 490.0, 9.604e-7
    elif name == "Y1":
        # strip along y (touching), 100 nm period, 40 nm wide, 6 nm thick, a 20 nm slot
        Ly = 100 * NM; h = 2 * NM * c
        ny = _round_cells(Ly, h); h = Ly / ny
        nx = _round_cells(40 * NM, h); nz = max(1, _round_cells(6 * NM, h))
        xc = (np.arange(nx) + 0.5) * h
        yc = (np.arange(ny) + 0.5) * h
        X, Y = np.meshgrid(xc, yc, indexing="ij")
        keep = ~((np.abs(X - 20 * NM) < 8 * NM) & (np.abs(Y - 50 * NM) < 10 * NM))
        mask = np.repeat(keep[:, :, None], nz, axis=2)
        mesh = kuhn_voxel_mesh(mask, h, wrap=(False, True, False), jitter=jitter, seed=seed, name=name)
        periodic = (0, 1, 0); lattice = (0.0, Ly, 0.0)
        g = grid or (max(4, int(8 // c)), max(16, int(64 // c)), 4)
        Ms, Aex = 637.0, 1.4e-6
    elif name == "K1":
        # Permalloy film, Ms = 637 emu/cm^3, A = 1.4e-6 erg/cm; the cell holds one spin-wave
        # wavelength 2 pi / k = 200 nm along x
        Lx, Ly, t = 200 * NM, 40 * NM, 10 * NM
        h = 2.5 * NM * c
        nx, ny, nz = _round_cells(Lx, h), _round_cells(Ly, h), max(1, _round_cells(t, h))
        mask = np.ones((nx, ny, nz), bool)
        mesh = kuhn_voxel_mesh(mask, Lx / nx, wrap=(True, True, False), jitter=jitter, seed=seed, name=name)
        periodic = (1, 1, 0); lattice = (Lx, Ly, 0.0)
        g = grid or (max(16, int(64 // c)), max(8, int(16 // c)), 4)
        Ms, Aex = 637.0, 1.4e-6
    else:
        raise KeyError(name)
    return dict(name=name, desc=CONFIGS[name], mesh=mesh, periodic=periodic,
                lattice=lattice, grid=tuple(int(v) for v in g), Ms=Ms, Aex=Aex,
                coarsen=coarsen, seed=seed)
